// rsfg_device.cuh -- device helpers shared by the sm_100a kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "rsfg_internal.h"

// Radii with a specialised (register-window) kernel -- every sigma <= 8 (R = ceil(3 sigma) <= 24);
// larger radii take the generic runtime-tap path.
#define RSFG_RADII(X)                                                                                  \
  X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16) X(17) X(18) \
  X(19) X(20) X(21) X(22) X(23) X(24)

namespace rsfg {
namespace {

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

// Opt a kernel into `bytes` of dynamic shared memory, once per (kernel,
// device): the attribute is per device, so a process that drives several GPUs
// sets it on each (a benign race otherwise: the set is idempotent).
template <auto Kernel>
inline bool smem_optin(int bytes) {
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && done[dev]) return true;
  if (cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
  if (dev >= 0 && dev < 64) done[dev] = true;
  return true;
}

__device__ __forceinline__ size_t vidx(const Geom& g, int x, int y, int z) {
  return (size_t)(z - g.zb) * (size_t)g.plane + (size_t)y * (size_t)g.nx + (size_t)x;
}

// Packed two-lane FP32 FMA (sm_100 FFMA2): acc + w * v on both lanes.
__device__ __forceinline__ float2 ffma2(float w, float2 v, float2 acc) {
  float2 d;
  asm("{\n\t.reg .b64 wv, vv, av, dv;\n\t"
      "mov.b64 wv, {%2, %2};\n\t"
      "mov.b64 vv, {%3, %4};\n\t"
      "mov.b64 av, {%5, %6};\n\t"
      "fma.rn.f32x2 dv, wv, vv, av;\n\t"
      "mov.b64 {%0, %1}, dv;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(w), "f"(v.x), "f"(v.y), "f"(acc.x), "f"(acc.y));
  return d;
}

// Packed two-lane FP32 multiply (sm_100 FMUL2): w * v on both lanes; the
// first tap of every pass (same bits as two scalar FMULs, half the issues).
__device__ __forceinline__ float2 fmul2(float w, float2 v) {
  float2 d;
  asm("{\n\t.reg .b64 wv, vv, dv;\n\t"
      "mov.b64 wv, {%2, %2};\n\t"
      "mov.b64 vv, {%3, %4};\n\t"
      "mul.rn.f32x2 dv, wv, vv;\n\t"
      "mov.b64 {%0, %1}, dv;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(w), "f"(v.x), "f"(v.y));
  return d;
}

// atan(q)/pi for q in [0, 1]: q * P(q^2), degree-8 fit; max relative error
// 1.9e-7 in fp32 (CUDA's atanf is 2 ulp); 9 FMAs, no branches.
__device__ __forceinline__ float atan_over_pi(float q) {
  const float x = q * q;
  float p = 0.000906360219232738f;
  p = fmaf(p, x, -0.00511184660717845f);
  p = fmaf(p, x, 0.013584661297500134f);
  p = fmaf(p, x, -0.023883428424596786f);
  p = fmaf(p, x, 0.0338696613907814f);
  p = fmaf(p, x, -0.04521126672625542f);
  p = fmaf(p, x, 0.06363844871520996f);
  p = fmaf(p, x, -0.10610246658325195f);
  p = fmaf(p, x, 0.31830987334251404f);
  return p * q;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Smoothed step H+ = 1/2 [1 + (2/pi) atan(phi/eps)] and H- = 1 - H+
// (rsf.cpp:22-25, 89-90), as 1/2 -+ sign(u) A with A = atan(|u|)/pi from the
// polynomial on q = min(|u|, 1/|u|): A = a (|u| <= 1) or 1/2 - a.  The small
// side on |u| > 1 is 1/2 - (1/2 - a), off a by one rounding (3e-8 absolute),
// where delta(phi) <= 1/(pi u^2) makes it negligible.  Same bits as the packed
// heaviside2 (rsfg_xy2.cuh).
__device__ __forceinline__ void heaviside_pair(float phi, float inv_eps, float& hm, float& hp) {
  const float u = phi * inv_eps;
  const float t = fabsf(u);
  const float a = atan_over_pi(fminf(t, rcp_approx(t)));
  const float A = t > 1.0f ? 0.5f - a : a;
  const float sA = copysignf(A, u);
  hm = 0.5f - sA;
  hp = 0.5f + sA;
}

__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 a,b,d; mov.b64 a,{%2,%3}; mov.b64 b,{%4,%5}; add.rn.f32x2 d,a,b; mov.b64 {%0,%1},d;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 a,b,d; mov.b64 a,{%2,%3}; mov.b64 b,{%4,%5}; mul.rn.f32x2 d,a,b; mov.b64 {%0,%1},d;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 a,b,c,d; mov.b64 a,{%2,%3}; mov.b64 b,{%4,%5}; mov.b64 c,{%6,%7}; fma.rn.f32x2 d,a,b,c; "
      "mov.b64 {%0,%1},d;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 f2s(float s) { return make_float2(s, s); }

// Heaviside pair of two voxels, packed: hm = H-(phi), hp = H+(phi) with
// H+ = 1/2 [1 + (2/pi) atan(phi/eps)] (rsf.cpp:22-25, 89-90).  Same
// evaluation as heaviside_pair (rsfg_device.cuh), bit for bit: atan(q)/pi on
// q = min(t, 1/t) in [0, 1].
template <bool WANT_HP>
__device__ __forceinline__ void heaviside2(float2 phi, float inv_eps, float2& hm, float2& hp) {
  const float2 u = f2mul(phi, f2s(inv_eps));
  const float tx = fabsf(u.x), ty = fabsf(u.y);
  const float2 q = make_float2(fminf(tx, rcp_approx(tx)), fminf(ty, rcp_approx(ty)));
  const float2 x = f2mul(q, q);
  float2 p = f2fma(f2s(0.000906360219232738f), x, f2s(-0.00511184660717845f));
  p = f2fma(p, x, f2s(0.013584661297500134f));
  p = f2fma(p, x, f2s(-0.023883428424596786f));
  p = f2fma(p, x, f2s(0.0338696613907814f));
  p = f2fma(p, x, f2s(-0.04521126672625542f));
  p = f2fma(p, x, f2s(0.06363844871520996f));
  p = f2fma(p, x, f2s(-0.10610246658325195f));
  p = f2fma(p, x, f2s(0.31830987334251404f));
  const float2 a = f2mul(p, q);  // atan(q)/pi in [0, 1/4]
  // A = atan(t)/pi = far ? 1/2 - a : a; H- = 1/2 - sign(u) A, H+ = 1/2 + sign(u) A.
  // On the far side the small H is 1/2 - (1/2 - a): exact but for one rounding
  // of 1/2 - a (3e-8 absolute), where delta(phi) <= 1/(pi t^2) is negligible.
  const float2 am = f2add(f2s(0.5f), make_float2(-a.x, -a.y));
  const float2 A = make_float2(tx > 1.0f ? am.x : a.x, ty > 1.0f ? am.y : a.y);
  const float2 sA = make_float2(copysignf(A.x, u.x), copysignf(A.y, u.y));
  hm = f2add(f2s(0.5f), make_float2(-sA.x, -sA.y));
  if constexpr (WANT_HP) hp = f2add(f2s(0.5f), sA);
}

// ---- TMA (cp.async.bulk.tensor) + mbarrier, sm_90+/sm_100a PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
#ifdef RSFG_BOUNDED_WAIT
// Debug builds (make debug): a wait that outlives ~2^30 polls -- a lost TMA
// transaction -- traps instead of hanging the caller's process.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  for (uint32_t polls = 0; !done; ++polls) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (polls == (1u << 30)) __trap();
  }
}
#else
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra.uni WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
#endif
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace
}  // namespace rsfg
