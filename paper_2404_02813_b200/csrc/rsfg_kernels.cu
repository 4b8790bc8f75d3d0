// rsfg_kernels.cu -- sm_100a kernels of the RSF level-set evolution step.
//
// One step (reference compute_energy + evolve_step, rsf.cpp:172-224,324-357)
// is two kernels:
//
//   xy  : per z-plane tile (TX x TY outputs, (TX+2R) x (TY+2R) input halo):
//         Heaviside fields (rsf.cpp:75-94) computed once per loaded voxel,
//         x pass and y pass of the separable Gaussian (ops.cpp:74-160) in
//         shared memory with register-blocked sliding windows and packed
//         FFMA2 (two fields per instruction).  Writes P = K_xy * fields.
//   zst : per column block (TX x TY columns x TZ planes): z pass from P with
//         a register window (ops.cpp:109-160 along z), region averages and
//         the force (rsf.cpp:130-148), delta (rsf.cpp:96-107), the 25-point
//         curvature stencil grad -> normalize -> divergence and the 7-point
//         Laplacian (ops.cpp:199-316, rsf.cpp:110-127) from a shared-memory
//         phi block, the combine (rsf.cpp:151-168) and the explicit update
//         with sign-change count and first-non-finite index (rsf.cpp:337-352).
//
// All neighbour indices clamp in GLOBAL coordinates (Geom.zb offsets a
// slab's buffers), so the same code runs the monolithic volume and z-slabs.
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "rsfg_internal.h"

namespace rsfg {

namespace {

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

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

__device__ __forceinline__ float2 fmul2(float w, float2 v) { return make_float2(w * v.x, w * v.y); }

// Smoothed step H+ = 1/2 [1 + (2/pi) atan(phi/eps)] and H- = 1 - H+
// (rsf.cpp:22-25, 89-90).  The side that is small is always evaluated
// directly (atan(1/t)/pi for t > 1) so both values keep full relative
// precision in fp32, as the reference's f64 evaluation does.
__device__ __forceinline__ void heaviside_pair(float phi, float inv_eps, float& hm, float& hp) {
  const float u = phi * inv_eps;
  const float t = fabsf(u);
  float small, big;
  if (t > 1.0f) {
    small = atanf(__frcp_rn(t)) * (float)(1.0 / CUDART_PI);
    big = 1.0f - small;
  } else {
    const float a = atanf(t) * (float)(1.0 / CUDART_PI);
    small = 0.5f - a;
    big = 0.5f + a;
  }
  if (u >= 0.0f) {
    hm = small;
    hp = big;
  } else {
    hm = big;
    hp = small;
  }
}

// ---------------------------------------------------------------- kernel 1
// NP = number of float2 field pairs (1: fields=2, 2: fields=4).
template <int R, int NP, int TX, int TY, int BX, int BY>
struct XYCfg {
  static constexpr int WX = TX + 2 * R;
  static constexpr int WY = TY + 2 * R;
  static constexpr int PX = WX | 1;  // odd pitch (float2): conflict-free row-strided LDS.64
  static constexpr int QX = TX | 1;
  static constexpr int kSmemF2 = NP * WY * (PX + QX);
  static constexpr size_t kSmem = kSmemF2 * sizeof(float2);
};

template <int R, int NP, int TX, int TY, int BX, int BY>
__global__ void __launch_bounds__(256) xy_kernel(Geom g, Taps taps, float inv_eps,
                                                 const float* __restrict__ phi,
                                                 const float* __restrict__ image,
                                                 float2* __restrict__ P0, float2* __restrict__ P1,
                                                 int z_begin) {
  using C = XYCfg<R, NP, TX, TY, BX, BY>;
  extern __shared__ float2 smem[];
  float2* Hs = smem;                      // [NP][WY][PX]
  float2* Xs = smem + NP * C::WY * C::PX;  // [NP][WY][QX]
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY, z = z_begin + blockIdx.z;

  // Phase A: clamped halo load + Heaviside fields (each input voxel once).
  for (int e = threadIdx.x; e < C::WX * C::WY; e += blockDim.x) {
    const int ey = e / C::WX, ex = e - ey * C::WX;
    const int gx = clampi(x0 - R + ex, 0, g.nx - 1), gy = clampi(y0 - R + ey, 0, g.ny - 1);
    const size_t i = vidx(g, gx, gy, z);
    const float p = __ldg(phi + i), im = __ldg(image + i);
    float hm, hp;
    heaviside_pair(p, inv_eps, hm, hp);
    Hs[ey * C::PX + ex] = make_float2(hm, hm * im);
    if (NP == 2) Hs[C::WY * C::PX + ey * C::PX + ex] = make_float2(hp, hp * im);
  }
  __syncthreads();

  // Phase B: x pass, BX consecutive outputs per item; lanes walk rows so a
  // half-warp reads 16 rows of the odd-pitched tile (no bank conflicts).
  constexpr int SEGX = TX / BX;
  for (int it = threadIdx.x; it < NP * C::WY * SEGX; it += blockDim.x) {
    const int np = it / (C::WY * SEGX);
    const int rem = it - np * C::WY * SEGX;
    const int sx = rem / C::WY, ry = rem - sx * C::WY;
    const float2* src = Hs + np * C::WY * C::PX + ry * C::PX + sx * BX;
    float2 v[BX + 2 * R];
#pragma unroll
    for (int k = 0; k < BX + 2 * R; ++k) v[k] = src[k];
    float2* dst = Xs + np * C::WY * C::QX + ry * C::QX + sx * BX;
#pragma unroll
    for (int b = 0; b < BX; ++b) {
      float2 acc = fmul2(taps.w[0], v[b]);
#pragma unroll
      for (int j = 1; j <= 2 * R; ++j) acc = ffma2(taps.w[j], v[b + j], acc);
      dst[b] = acc;
    }
  }
  __syncthreads();

  // Phase C: y pass, BY consecutive outputs down a column; lanes walk x.
  constexpr int SEGY = TY / BY;
  for (int it = threadIdx.x; it < NP * TX * SEGY; it += blockDim.x) {
    const int np = it / (TX * SEGY);
    const int rem = it - np * TX * SEGY;
    const int sy = rem / TX, cx = rem - sy * TX;
    const float2* src = Xs + np * C::WY * C::QX + (sy * BY) * C::QX + cx;
    float2 v[BY + 2 * R];
#pragma unroll
    for (int k = 0; k < BY + 2 * R; ++k) v[k] = src[k * C::QX];
    const int gx = x0 + cx;
    float2* P = np ? P1 : P0;
#pragma unroll
    for (int b = 0; b < BY; ++b) {
      float2 acc = fmul2(taps.w[0], v[b]);
#pragma unroll
      for (int j = 1; j <= 2 * R; ++j) acc = ffma2(taps.w[j], v[b + j], acc);
      const int gy = y0 + sy * BY + b;
      if (gx < g.nx && gy < g.ny) P[vidx(g, gx, gy, z)] = acc;
    }
  }
}

// ---------------------------------------------------------------- kernel 2
template <int R, int NP, int TX, int TY, int TZ>
struct ZCfg {
  static constexpr int FX = TX + 4, FY = TY + 4, FZ = TZ + 4;  // phi block, halo 2
  static constexpr int NXr = TX + 2, NYr = TY + 2;              // normal planes, halo 1
  static constexpr int kPhi = FX * FY * FZ;
  static constexpr int kRing = 3 * 3 * NXr * NYr;
  static constexpr int kKH = NP * TZ * TX * TY * 2;  // floats
  static constexpr size_t kSmem = (size_t)(kPhi + kRing + kKH) * sizeof(float);
};

template <int R, int NP, int TX, int TY, int TZ>
__global__ void __launch_bounds__(TX* TY, 2)
    zst_kernel(Geom g, Taps taps, StepConsts c, StepBuffers b, int z_begin, int z_end, int mode) {
  using C = ZCfg<R, NP, TX, TY, TZ>;
  extern __shared__ float smemf[];
  float* Phi = smemf;                // [FZ][FY][FX]
  float* Ring = Phi + C::kPhi;       // [3 slots][3 comps][NYr][NXr]
  float2* KH = reinterpret_cast<float2*>(Ring + C::kRing);  // [NP][TZ][TY][TX]
  __shared__ unsigned int s_count;

  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int z0 = z_begin + blockIdx.x * TZ;  // z tile fastest: consecutive CTAs share P halos in L2
  const int x0 = blockIdx.y * TX, y0 = blockIdx.z * TY;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  if (threadIdx.x == 0) s_count = 0;

  // Phase 0: phi block with halo 2 (clamped global coordinates).
  for (int e = threadIdx.x; e < C::kPhi; e += blockDim.x) {
    const int ex = e % C::FX, t = e / C::FX;
    const int ey = t % C::FY, ez = t / C::FY;
    const int gx = clampi(x0 - 2 + ex, 0, nx - 1), gy = clampi(y0 - 2 + ey, 0, ny - 1);
    const int gz = clampi(z0 - 2 + ez, g.zb, g.ze - 1);
    Phi[e] = __ldg(b.phi + vidx(g, gx, gy, gz));
  }

  // Phase 1: z pass of P for this thread's column; the reference rounds its
  // z pass to f32 after every tap in ascending order (ops.cpp:150-155), which
  // is exactly an fp32 FMA chain.
  {
    const int gx = min(x0 + tx, nx - 1), gy = min(y0 + ty, ny - 1);
#pragma unroll
    for (int np = 0; np < NP; ++np) {
      const float2* P = b.P[np];
      float2 pv[TZ + 2 * R];
#pragma unroll
      for (int k = 0; k < TZ + 2 * R; ++k)
        pv[k] = __ldg(P + vidx(g, gx, gy, clampi(z0 - R + k, g.zb, g.ze - 1)));
#pragma unroll
      for (int t = 0; t < TZ; ++t) {
        float2 acc = fmul2(taps.w[0], pv[t]);
#pragma unroll
        for (int j = 1; j <= 2 * R; ++j) acc = ffma2(taps.w[j], pv[t + j], acc);
        KH[(np * TZ + t) * TX * TY + threadIdx.x] = acc;
      }
    }
  }
  __syncthreads();

  // Normalized gradient n = grad phi / max(|grad phi|, floor) on one plane of
  // (TX+2) x (TY+2) positions; positions outside the volume take the value
  // of their clamped neighbour, which is what divergence's clamped indices
  // read (ops.cpp:294-310).  Gradient: central inside, one-sided on faces.
  auto phi_at = [&](int gx, int gy, int gz) -> float {
    return Phi[((gz - (z0 - 2)) * C::FY + (gy - (y0 - 2))) * C::FX + (gx - (x0 - 2))];
  };
  auto normal_plane = [&](int slot, int zz) {
    const int gz = clampi(zz, 0, nz - 1);
    const int zm = max(gz - 1, 0), zp = min(gz + 1, nz - 1);
    const float invz = (zp - zm) == 2 ? 0.5f : 1.0f;
    float* rs = Ring + slot * 3 * C::NXr * C::NYr;
    for (int e = threadIdx.x; e < C::NXr * C::NYr; e += blockDim.x) {
      const int i = e % C::NXr, j = e / C::NXr;
      const int gx = clampi(x0 - 1 + i, 0, nx - 1), gy = clampi(y0 - 1 + j, 0, ny - 1);
      const int xm = max(gx - 1, 0), xp = min(gx + 1, nx - 1);
      const int ym = max(gy - 1, 0), yp = min(gy + 1, ny - 1);
      const float invx = (xp - xm) == 2 ? 0.5f : 1.0f;
      const float invy = (yp - ym) == 2 ? 0.5f : 1.0f;
      const float a = (phi_at(xp, gy, gz) - phi_at(xm, gy, gz)) * invx;
      const float bb = (phi_at(gx, yp, gz) - phi_at(gx, ym, gz)) * invy;
      const float cc = (phi_at(gx, gy, zp) - phi_at(gx, gy, zm)) * invz;
      const float m = fmaxf(__fsqrt_rn(fmaf(a, a, fmaf(bb, bb, cc * cc))), c.grad_floor);
      const float inv = __frcp_rn(m);
      rs[e] = a * inv;
      rs[C::NXr * C::NYr + e] = bb * inv;
      rs[2 * C::NXr * C::NYr + e] = cc * inv;
    }
  };

  normal_plane(0, z0 - 1);
  normal_plane(1, z0);

  const int x = x0 + tx, y = y0 + ty;
  const bool col_ok = x < nx && y < ny;
  const int xm = max(x - 1, 0), xp = min(x + 1, nx - 1);
  const int ym = max(y - 1, 0), yp = min(y + 1, ny - 1);
  const float invx = (xp - xm) == 2 ? 0.5f : 1.0f;
  const float invy = (yp - ym) == 2 ? 0.5f : 1.0f;
  const int ixm = xm - (x0 - 1), ixp = xp - (x0 - 1), ic = tx + 1;
  const int jym = ym - (y0 - 1), jyp = yp - (y0 - 1), jc = ty + 1;
  const size_t col = (size_t)min(y, ny - 1) * nx + min(x, nx - 1);
  unsigned int my_count = 0;

  for (int t = 0; t < TZ; ++t) {
    const int zo = z0 + t;
    normal_plane((t + 2) % 3, zo + 1);
    __syncthreads();
    const bool active = col_ok && zo < z_end;
    if (zo < z_end) {
      const float* nm = Ring + (t % 3) * 3 * C::NXr * C::NYr;        // plane zo-1
      const float* n0 = Ring + ((t + 1) % 3) * 3 * C::NXr * C::NYr;  // plane zo
      const float* np1 = Ring + ((t + 2) % 3) * 3 * C::NXr * C::NYr; // plane zo+1
      const int zmm = max(zo - 1, 0), zpp = min(zo + 1, nz - 1);
      const float invz = (zpp - zmm) == 2 ? 0.5f : 1.0f;
      constexpr int PL = C::NXr * C::NYr;
      const float kx = (n0[jc * C::NXr + ixp] - n0[jc * C::NXr + ixm]) * invx;
      const float ky = (n0[PL + jyp * C::NXr + ic] - n0[PL + jym * C::NXr + ic]) * invy;
      const float kz = (np1[2 * PL + jc * C::NXr + ic] - nm[2 * PL + jc * C::NXr + ic]) * invz;
      const float kappa = kx + ky + kz;

      // 7-point Laplacian, clamp-to-edge (ops.cpp:258-271).
      const int sx = tx + 2, sy = ty + 2, sz = t + 2;
      const float* pc = Phi + (sz * C::FY + sy) * C::FX + sx;
      const float cphi = pc[0];
      const float lap = fmaf(-2.0f, cphi, pc[-1] + pc[1]) + fmaf(-2.0f, cphi, pc[-C::FX] + pc[C::FX]) +
                        fmaf(-2.0f, cphi, pc[-C::FX * C::FY] + pc[C::FX * C::FY]);

      // delta_eps (rsf.cpp:96-107).
      const float delta = __fdividef(c.c_delta, fmaf(cphi, cphi, c.eps2));

      // Region averages r+- and the force difference F- - F+ (rsf.cpp:130-148,164).
      const size_t vi = (size_t)(zo - g.zb) * (size_t)g.plane + col;
      const float ki = __ldg(b.ki + vi);
      float kp, kpi, km, kmi;
      const float2 h0 = KH[t * TX * TY + threadIdx.x];
      km = h0.x;
      kmi = h0.y;
      if (NP == 2) {
        const float2 h1 = KH[(TZ + t) * TX * TY + threadIdx.x];
        kp = h1.x;
        kpi = h1.y;
      } else {
        kp = 1.0f - km;
        kpi = __ldg(b.k1i + vi) - kmi;
      }
      const float rp = fminf(fmaxf(__fdiv_rn(kpi, fmaxf(kp, c.denom_floor)), c.i_min), c.i_max);
      const float rm = fminf(fmaxf(__fdiv_rn(kmi, fmaxf(km, c.denom_floor)), c.i_min), c.i_max);
      // (KI2 - 2 r- KI + r-^2) - (KI2 - 2 r+ KI + r+^2) == (r+ - r-)(2 KI - r+ - r-)
      const float dF = (rp - rm) * (fmaf(2.0f, ki, -rp) - rm);

      // Combine (rsf.cpp:151-168) and update (rsf.cpp:340-344).
      const float e = (lap - kappa) + delta * fmaf(c.alpha, kappa, c.beta * dF);
      if (active) {
        if (mode == kUpdate) {
          const float f = (float)((double)cphi + c.dt * (double)e);
          b.out[vi] = f;
          my_count += ((cphi < 0.0f) != (f < 0.0f)) ? 1u : 0u;
          if (!isfinite(f)) {
            const unsigned long long gi = (unsigned long long)zo * (unsigned long long)g.plane + col;
            atomicMin(b.counters + 1, gi);
          }
        } else {
          b.out[vi] = e;
        }
      }
    }
    __syncthreads();
  }

  if (mode == kUpdate) {
    const unsigned int wsum = __reduce_add_sync(0xffffffffu, my_count);
    if ((threadIdx.x & 31) == 0 && wsum) atomicAdd(&s_count, wsum);
    __syncthreads();
    if (threadIdx.x == 0 && s_count) atomicAdd(b.counters, (unsigned long long)s_count);
  }
}

// ---------------------------------------------------------- generic passes
__global__ void heaviside_fields_kernel(Geom g, float inv_eps, const float* __restrict__ phi,
                                        const float* __restrict__ image, float2* __restrict__ S0,
                                        float2* __restrict__ S1, int z_begin, int z_end) {
  const long long n = (long long)(z_end - z_begin) * g.plane;
  const size_t base = (size_t)(z_begin - g.zb) * (size_t)g.plane;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float p = phi[base + i], im = image[base + i];
    float hm, hp;
    heaviside_pair(p, inv_eps, hm, hp);
    S0[base + i] = make_float2(hm, hm * im);
    if (S1) S1[base + i] = make_float2(hp, hp * im);
  }
}

template <typename T>
__device__ __forceinline__ T tap(float w, T v);
template <>
__device__ __forceinline__ float tap<float>(float w, float v) { return w * v; }
template <>
__device__ __forceinline__ float2 tap<float2>(float w, float2 v) { return fmul2(w, v); }
__device__ __forceinline__ float fma_t(float w, float v, float a) { return fmaf(w, v, a); }
__device__ __forceinline__ float2 fma_t(float w, float2 v, float2 a) { return ffma2(w, v, a); }

// One separable pass along `axis` (0 x, 1 y, 2 z) with runtime taps over
// planes [z_begin, z_end); clamp-to-edge in global coordinates.
template <typename T>
__global__ void conv_axis_kernel(Geom g, Taps taps, int axis, const T* __restrict__ src,
                                 T* __restrict__ dst, int z_begin, int z_end) {
  const long long n = (long long)(z_end - z_begin) * g.plane;
  const int r = taps.r;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % g.nx);
    const int y = (int)((i / g.nx) % g.ny);
    const int z = z_begin + (int)(i / g.plane);
    const int pos = axis == 0 ? x : (axis == 1 ? y : z);
    const int n_ax = axis == 0 ? g.nx : (axis == 1 ? g.ny : g.nz);
    T acc;
    const int lo = axis == 2 ? g.zb : 0, hi = axis == 2 ? g.ze - 1 : n_ax - 1;
    for (int j = 0; j <= 2 * r; ++j) {
      const int q = clampi(clampi(pos - r + j, 0, n_ax - 1), lo, hi);
      const size_t s = axis == 0 ? vidx(g, q, y, z) : (axis == 1 ? vidx(g, x, q, z) : vidx(g, x, y, q));
      const T v = src[s];
      acc = j == 0 ? tap<T>(taps.w[0], v) : fma_t(taps.w[j], v, acc);
    }
    dst[vidx(g, x, y, z)] = acc;
  }
}

__global__ void minmax_kernel(Geom g, const float* __restrict__ v, int z_begin, int z_end,
                              unsigned int* mm) {
  const long long n = (long long)(z_end - z_begin) * g.plane;
  const size_t base = (size_t)(z_begin - g.zb) * (size_t)g.plane;
  float lo = CUDART_INF_F, hi = -CUDART_INF_F;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float f = v[base + i];
    lo = fminf(lo, f);
    hi = fmaxf(hi, f);
  }
  for (int o = 16; o; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    const unsigned int ulo = __float_as_uint(lo), uhi = __float_as_uint(hi);
    atomicMin(mm, (ulo & 0x80000000u) ? ~ulo : (ulo | 0x80000000u));
    atomicMax(mm + 1, (uhi & 0x80000000u) ? ~uhi : (uhi | 0x80000000u));
  }
}

__global__ void mask_kernel(const float* __restrict__ phi, float* __restrict__ mask, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    mask[i] = phi[i] < 0.0f ? 1.0f : 0.0f;
}

int grid_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  const long long cap = 148LL * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

// ------------------------------------------------------------ dispatchers
constexpr int kXYTX = 64, kXYTY = 32, kBX = 8, kBY = 8;
constexpr int kZTX = 32, kZTY = 8, kZTZ = 16;

template <int R, int NP>
int xy_launch(const Geom& g, const Taps& t, float inv_eps, const float* phi, const float* image,
              float2* P0, float2* P1, int z_begin, int z_end, cudaStream_t st) {
  using C = XYCfg<R, NP, kXYTX, kXYTY, kBX, kBY>;
  auto k = xy_kernel<R, NP, kXYTX, kXYTY, kBX, kBY>;
  static bool attr = false;  // benign race: idempotent attribute set
  if (!attr) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
    attr = true;
  }
  if (z_end <= z_begin) return 0;
  dim3 grid((g.nx + kXYTX - 1) / kXYTX, (g.ny + kXYTY - 1) / kXYTY, z_end - z_begin);
  k<<<grid, 256, C::kSmem, st>>>(g, t, inv_eps, phi, image, P0, P1, z_begin);
  return 1;
}

template <int R, int NP>
int zst_launch(const Geom& g, const Taps& t, const StepConsts& c, const StepBuffers& b, int z_begin,
               int z_end, int mode, cudaStream_t st) {
  using C = ZCfg<R, NP, kZTX, kZTY, kZTZ>;
  auto k = zst_kernel<R, NP, kZTX, kZTY, kZTZ>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
    attr = true;
  }
  if (z_end <= z_begin) return 0;
  dim3 grid((z_end - z_begin + kZTZ - 1) / kZTZ, (g.nx + kZTX - 1) / kZTX, (g.ny + kZTY - 1) / kZTY);
  k<<<grid, kZTX * kZTY, C::kSmem, st>>>(g, t, c, b, z_begin, z_end, mode);
  return 1;
}

#define RSFG_RADII(X) X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(15) X(18)

}  // namespace

bool has_fast_radius(int r) {
  switch (r) {
#define CASE(R) case R:
    RSFG_RADII(CASE)
#undef CASE
    return true;
    default:
      return false;
  }
}

int launch_xy(const Geom& g, int fields, const Taps& t1, float inv_eps, const float* phi,
              const float* image, float2* P0, float2* P1, int z_begin, int z_end, cudaStream_t st) {
  switch (t1.r) {
#define CASE(R)                                                                                \
  case R:                                                                                      \
    return fields == 4 ? xy_launch<R, 2>(g, t1, inv_eps, phi, image, P0, P1, z_begin, z_end, st) \
                       : xy_launch<R, 1>(g, t1, inv_eps, phi, image, P0, P1, z_begin, z_end, st);
    RSFG_RADII(CASE)
#undef CASE
    default:
      return -1;
  }
}

int launch_zst(const Geom& g, int fields, const Taps& t1, const StepConsts& c, const StepBuffers& b,
               int z_begin, int z_end, StepMode mode, cudaStream_t st) {
  switch (t1.r) {
#define CASE(R)                                                                       \
  case R:                                                                             \
    return fields == 4 ? zst_launch<R, 2>(g, t1, c, b, z_begin, z_end, (int)mode, st) \
                       : zst_launch<R, 1>(g, t1, c, b, z_begin, z_end, (int)mode, st);
    RSFG_RADII(CASE)
#undef CASE
    default:
      return -1;
  }
}

int launch_generic_conv(const Geom& g, int fields, const Taps& t1, float inv_eps, const float* phi,
                        const float* image, float2* const P[2], float2* scratch, int zk_begin,
                        int zk_end, int z_begin, int z_end, cudaStream_t st) {
  const int np = fields == 4 ? 2 : 1;
  const size_t held = (size_t)(g.ze - g.zb) * (size_t)g.plane;
  float2* S[2] = {scratch, scratch + held};
  float2* T[2] = {scratch + np * held, scratch + (np + 1) * held};
  const long long n_k = (long long)(zk_end - zk_begin) * g.plane;
  const long long n_z = (long long)(z_end - z_begin) * g.plane;
  int launches = 0;
  if (n_k > 0) {
    heaviside_fields_kernel<<<grid_for(n_k, 256), 256, 0, st>>>(g, inv_eps, phi, image, S[0],
                                                                np == 2 ? S[1] : nullptr, zk_begin,
                                                                zk_end);
    ++launches;
    for (int f = 0; f < np; ++f) {
      conv_axis_kernel<float2><<<grid_for(n_k, 256), 256, 0, st>>>(g, t1, 0, S[f], T[f], zk_begin, zk_end);
      conv_axis_kernel<float2><<<grid_for(n_k, 256), 256, 0, st>>>(g, t1, 1, T[f], S[f], zk_begin, zk_end);
      launches += 2;
    }
  }
  if (n_z > 0) {
    for (int f = 0; f < np; ++f) {
      conv_axis_kernel<float2><<<grid_for(n_z, 256), 256, 0, st>>>(g, t1, 2, S[f], P[f], z_begin, z_end);
      ++launches;
    }
  }
  return cudaPeekAtLastError() == cudaSuccess ? launches : -1;
}

int launch_convolve(const Geom& g, const Taps& t, const float* src, float* dst, float* tmp0,
                    float* tmp1, int z_begin, int z_end, cudaStream_t st) {
  if (t.r == 0) {
    const size_t off = (size_t)(z_begin - g.zb) * (size_t)g.plane;
    cudaMemcpyAsync(dst + off, src + off, (size_t)(z_end - z_begin) * g.plane * sizeof(float),
                    cudaMemcpyDeviceToDevice, st);
    return 0;
  }
  // x and y passes on every plane the z pass reads, then z on [z_begin, z_end).
  const int za = max(z_begin - t.r, g.zb), zb2 = min(z_end + t.r, g.nz);
  const long long n_xy = (long long)(zb2 - za) * g.plane, n_z = (long long)(z_end - z_begin) * g.plane;
  conv_axis_kernel<float><<<grid_for(n_xy, 256), 256, 0, st>>>(g, t, 0, src, tmp0, za, zb2);
  conv_axis_kernel<float><<<grid_for(n_xy, 256), 256, 0, st>>>(g, t, 1, tmp0, tmp1, za, zb2);
  conv_axis_kernel<float><<<grid_for(n_z, 256), 256, 0, st>>>(g, t, 2, tmp1, dst, z_begin, z_end);
  return 3;
}

int launch_minmax(const Geom& g, const float* v, int z_begin, int z_end, unsigned int* mm,
                  cudaStream_t st) {
  const long long n = (long long)(z_end - z_begin) * g.plane;
  minmax_kernel<<<grid_for(n, 256), 256, 0, st>>>(g, v, z_begin, z_end, mm);
  return 1;
}

unsigned int encode_ordered(float f) {
  unsigned int u;
  memcpy(&u, &f, 4);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

float decode_ordered(unsigned int u) {
  const unsigned int b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
  float f;
  memcpy(&f, &b, 4);
  return f;
}

int launch_mask(const float* phi, float* mask, long long n, cudaStream_t st) {
  mask_kernel<<<grid_for(n, 256), 256, 0, st>>>(phi, mask, n);
  return 1;
}

}  // namespace rsfg
