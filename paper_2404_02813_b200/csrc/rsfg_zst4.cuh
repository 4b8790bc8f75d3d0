// rsfg_zst4.cu -- kernel 2 of the RSF step, TMA-fed z-streaming variant:
// z pass, region averages and force, curvature / Laplacian stencil, combine
// and explicit update (reference rsf.cpp:96-168, 324-352; ops.cpp:109-160,
// 199-316).  Same arithmetic as rsfg_zst.cu's kernel; what changes is how the
// data reaches the threads:
//
//  * phi planes stream through an 8-slot shared ring filled by TMA (one
//    elected thread, one mbarrier per slot, four planes of prefetch), so no
//    thread spends instructions staging phi;
//  * the z-pass input window (8 + 2R planes of the kernel-1 pairs P for the
//    CTA's 32 x 8 columns) arrives as ONE 3-D TMA box per 8-plane group,
//    issued a whole group ahead into a single buffer;
//  * the plane loop is unrolled by 8 (the phi-ring period; the 4-slot normal
//    ring divides it), so every ring access is a base register plus an
//    immediate: no per-voxel address arithmetic;
//  * interior tiles away from the volume faces run a variant with constant
//    neighbour offsets and the 1/2 central-difference factors folded into a
//    doubled-gradient convention (n = 2g / max(|2g|, 2 floor) == g / max(|g|,
//    floor) exactly); tiles or plane groups that touch a face run the general
//    variant with per-thread clamped offsets and per-plane face factors.
#pragma once
#include <type_traits>

#include "rsfg_device.cuh"

namespace rsfg {
namespace {

template <int R, int NP>
struct Z4 {
  static constexpr int TX = 32, TY = 8, NT = TX * TY;
  static constexpr int BX = 40, BY = 12, SLOT = BX * BY;  // phi TMA box (floats): x0-4.., y0-2..
  static constexpr int NXr = TX + 2, NYr = TY + 2, NPL = NXr * NYr;  // normal plane, halo 1
  static constexpr int kHalo = NPL - NT;
  static constexpr int G = 8;             // planes per group (z-pass chunk, ring period)
  static constexpr int TZ = 64;           // planes per CTA
  static constexpr int NW = G + 2 * R;    // z-pass window (planes)
  static constexpr int PPL = TX * TY;     // float2 per P plane of the box
  static constexpr size_t kPBytes = (size_t)NP * NW * PPL * sizeof(float2);
  static constexpr size_t kPhiBytes = (size_t)8 * SLOT * sizeof(float);
  static constexpr size_t kNrBytes = (size_t)4 * 3 * NPL * sizeof(float);
  static constexpr size_t kSmem = kPBytes + kPhiBytes + kNrBytes + 16 * sizeof(uint64_t);
};

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// One normal-plane position: phi-ring offset of its centre, neighbour deltas
// and doubled-convention factors (1 central, 2 one-sided), normal-plane slot.
struct NPos {
  int s, dxm, dxp, dym, dyp, n;
  float fx, fy;
};

template <int R, int NP, bool GEN>
struct Z4Body {
  using C = Z4<R, NP>;

  // n at one position of global plane q from ring slots (om, o0, op); fz =
  // doubled-convention z factor.  dst = normal plane slot base.
  static __device__ __forceinline__ void normal(const float* __restrict__ Phi, const NPos& p, int om, int o0,
                                               int op, float fz, float inv2floor, float* __restrict__ dst) {
    const float* c0 = Phi + o0 + p.s;
    float a, bb, cc;
    if constexpr (GEN) {
      a = (c0[p.dxp] - c0[p.dxm]) * p.fx;
      bb = (c0[p.dyp] - c0[p.dym]) * p.fy;
      cc = (Phi[op + p.s] - Phi[om + p.s]) * fz;
    } else {
      a = c0[1] - c0[-1];
      bb = c0[C::BX] - c0[-C::BX];
      cc = Phi[op + p.s] - Phi[om + p.s];
    }
    const float inv = fminf(rsqrt_approx(fmaf(a, a, fmaf(bb, bb, cc * cc))), inv2floor);
    float* d = dst + p.n;
    d[0] = a * inv;
    d[C::NPL] = bb * inv;
    d[2 * C::NPL] = cc * inv;
  }
};

template <int R, int NP>
__global__ void __launch_bounds__(256, 2)
    zst4_kernel(Geom g, Taps taps, StepConsts c, StepBuffers b, int z_begin, int z_end,
                const __grid_constant__ CUtensorMap map_phi, const __grid_constant__ CUtensorMap map_p0,
                const __grid_constant__ CUtensorMap map_p1);

// --------------------------------------------------------------------------
// The CTA program, templated on the xy variant (GX: general offsets).  The
// z variant (faces, partial groups) is chosen per group at run time.
template <int R, int NP, bool GX>
__device__ __forceinline__ void zst4_cta(const Geom& g, const Taps& taps, const StepConsts& c, const StepBuffers& b,
                                         int z0, int z_stop, int x0, int y0, int bx0, int by0,
                                         const CUtensorMap* map_phi, const CUtensorMap* map_p0,
                                         const CUtensorMap* map_p1, unsigned char* smem, unsigned int& my_count) {
  using C = Z4<R, NP>;
  float2* Pb = reinterpret_cast<float2*>(smem);                               // [NP][NW][TY][TX]
  float* Phi = reinterpret_cast<float*>(smem + C::kPBytes);                   // [8][BY][BX]
  float* Nr = Phi + 8 * C::SLOT;                                              // [4][3][NYr][NXr]
  uint64_t* bars = reinterpret_cast<uint64_t*>(Nr + 4 * 3 * C::NPL);          // [8] phi slots, [8] P buffer
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long plane = g.plane;
  const float inv2floor = 0.5f * c.inv_grad_floor;

  // ---- positions.  Ring offset of global (gx, gy): (gy - by0) * BX + (gx - bx0).
  auto make_pos = [&](int i, int j) {  // normal-plane position (i, j) <-> global (x0-1+i, y0-1+j)
    NPos p;
    const int gx = clampi(x0 - 1 + i, 0, nx - 1), gy = clampi(y0 - 1 + j, 0, ny - 1);
    const int xm = max(gx - 1, 0), xp = min(gx + 1, nx - 1), ym = max(gy - 1, 0), yp = min(gy + 1, ny - 1);
    p.s = (gy - by0) * C::BX + (gx - bx0);
    p.dxm = xm - gx;
    p.dxp = xp - gx;
    p.dym = (ym - gy) * C::BX;
    p.dyp = (yp - gy) * C::BX;
    p.fx = (xp - xm) == 2 ? 1.0f : 2.0f;
    p.fy = (yp - ym) == 2 ? 1.0f : 2.0f;
    p.n = j * C::NXr + i;
    return p;
  };
  const NPos own = make_pos(tx + 1, ty + 1);
  const bool has_halo = tid < C::kHalo;
  NPos hal = own;
  if (has_halo) {
    int i, j;
    if (tid < C::NXr) {
      i = tid, j = 0;
    } else if (tid < 2 * C::NXr) {
      i = tid - C::NXr, j = C::NYr - 1;
    } else {
      const int k = tid - 2 * C::NXr;
      i = (k & 1) ? C::NXr - 1 : 0;
      j = 1 + (k >> 1);
    }
    hal = make_pos(i, j);
  }
  // output voxel: kappa deltas in the normal plane and factors
  const int x = x0 + tx, y = y0 + ty;
  const bool col_ok = x < nx && y < ny;
  const int gxc = min(x, nx - 1), gyc = min(y, ny - 1);
  const int kxm = max(gxc - 1, 0) - gxc, kxp = min(gxc + 1, nx - 1) - gxc;
  const int kym = (max(gyc - 1, 0) - gyc) * C::NXr, kyp = (min(gyc + 1, ny - 1) - gyc) * C::NXr;
  const float kfx = (kxp - kxm) == 2 ? 1.0f : 2.0f;
  const float kfy = (kyp - kym) == 2 * C::NXr ? 1.0f : 2.0f;
  const size_t col = (size_t)gyc * nx + gxc;

  // ---- TMA helpers (thread 0 only)
  auto zc_of = [&](int q) { return clampi(q, g.zb, g.ze - 1) - g.zb; };
  auto issue_phi = [&](int q) {  // plane q -> slot (q - z0 + 2) & 7
    const int sl = (q - z0 + 2) & 7;
    mbar_expect_tx(bars + sl, (uint32_t)(C::SLOT * sizeof(float)));
    tma_load_3d(Phi + sl * C::SLOT, map_phi, bars + sl, bx0, by0, zc_of(q));
  };
  // P window of the group starting at zc: TMA when it lies inside the held
  // planes (no clamping needed), else threads load it with clamped LDG.
  auto p_tma_ok = [&](int zc) { return zc - R >= g.zb && zc + C::G + R <= g.ze; };
  auto issue_p = [&](int zc) {
    mbar_expect_tx(bars + 8, (uint32_t)C::kPBytes);
    tma_load_3d(Pb, map_p0, bars + 8, 2 * x0, y0, zc - R - g.zb);
    if (NP == 2) tma_load_3d(Pb + C::NW * C::PPL, map_p1, bars + 8, 2 * x0, y0, zc - R - g.zb);
  };

  if (tid == 0) {
    for (int i = 0; i < 9; ++i) mbar_init(bars + i, 1);
    const int last = min(z0 + 5, z_stop + 1);
    for (int q = z0 - 2; q <= last; ++q) issue_phi(q);
    if (p_tma_ok(z0)) issue_p(z0);
  }
  __syncthreads();

  // ---- prologue: normal planes z0-1 and z0 (normal slots 0 and 1)
  for (int sl = 0; sl < 4; ++sl) mbar_wait(bars + sl, 0);
  {
    auto fzq = [&](int q) { return (q == 0 || q == nz - 1) ? 2.0f : 1.0f; };
    // plane z0-1 from ring slots (0,1,2); plane z0 from (1,2,3)
    Z4Body<R, NP, true>::normal(Phi, own, 0, C::SLOT, 2 * C::SLOT, fzq(z0 - 1), inv2floor, Nr);
    if (has_halo) Z4Body<R, NP, true>::normal(Phi, hal, 0, C::SLOT, 2 * C::SLOT, fzq(z0 - 1), inv2floor, Nr);
    Z4Body<R, NP, true>::normal(Phi, own, C::SLOT, 2 * C::SLOT, 3 * C::SLOT, fzq(z0), inv2floor, Nr + 3 * C::NPL);
    if (has_halo)
      Z4Body<R, NP, true>::normal(Phi, hal, C::SLOT, 2 * C::SLOT, 3 * C::SLOT, fzq(z0), inv2floor,
                                  Nr + 3 * C::NPL);
  }

  // ring base pointers (per thread), all accesses below add immediates
  float* const Nown = Nr + own.n;

  uint32_t pphase = 0;
  float kib[8], k1ib[8];
  // static-field prefetch two planes ahead (planes z0, z0+1)
  {
    const float* kip = b.ki + (size_t)(z0 - g.zb) * plane + col;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      kib[k] = (z0 + k < z_stop) ? __ldg(kip + (size_t)k * plane) : 0.0f;
      if (NP == 1) k1ib[k] = (z0 + k < z_stop) ? __ldg(b.k1i + (size_t)(z0 + k - g.zb) * plane + col) : 0.0f;
    }
  }

#pragma unroll 1
  for (int zc = z0, grp = 0; zc < z_stop; zc += C::G, ++grp) {
    // ---- z pass for planes zc .. zc+7 (fp32 FMA per tap, ascending order,
    // like the reference's f32-rounded z pass, ops.cpp:150-155)
    float2 kh[NP][C::G];
    if (p_tma_ok(zc)) {
      mbar_wait(bars + 8, pphase);
      pphase ^= 1;
      const float2* src = Pb + ty * C::TX + tx;
#pragma unroll
      for (int np = 0; np < NP; ++np) {
        float2 w[C::NW];
#pragma unroll
        for (int k = 0; k < C::NW; ++k) w[k] = src[(np * C::NW + k) * C::PPL];
#pragma unroll
        for (int t = 0; t < C::G; ++t) {
          float2 acc = fmul2(taps.w[0], w[t]);
#pragma unroll
          for (int j = 1; j <= 2 * R; ++j) acc = ffma2(taps.w[j], w[t + j], acc);
          kh[np][t] = acc;
        }
      }
    } else {
#pragma unroll
      for (int np = 0; np < NP; ++np) {
        const float2* P = b.P[np] + col;
        float2 w[C::NW];
#pragma unroll
        for (int k = 0; k < C::NW; ++k)
          w[k] = __ldg(P + (size_t)(clampi(zc - R + k, g.zb, g.ze - 1) - g.zb) * (size_t)plane);
#pragma unroll
        for (int t = 0; t < C::G; ++t) {
          float2 acc = fmul2(taps.w[0], w[t]);
#pragma unroll
          for (int j = 1; j <= 2 * R; ++j) acc = ffma2(taps.w[j], w[t + j], acc);
          kh[np][t] = acc;
        }
      }
    }

    const bool zfast = !GX && zc >= 1 && zc + C::G <= nz - 2 && zc + C::G <= z_stop;
    float* out = b.out + (size_t)(zc - g.zb) * plane + col;
    const float* kip = b.ki + (size_t)(zc - g.zb) * plane + col;
    const float* k1ip = b.k1i + (size_t)(zc - g.zb) * plane + col;

    auto step = [&](auto kc, auto genc) {
      constexpr int k = decltype(kc)::value;
      constexpr bool GEN = decltype(genc)::value;
      using B = Z4Body<R, NP, GEN>;
      const int zo = zc + k;
      if (GEN && zo >= z_stop) return;  // partial last group (uniform)
      // prefetch static fields two planes ahead
      if (!GEN || zo + 2 < z_stop) {
        kib[(k + 2) & 7] = __ldg(kip + (size_t)(k + 2) * plane);
        if (NP == 1) k1ib[(k + 2) & 7] = __ldg(k1ip + (size_t)(k + 2) * plane);
      }
      // phi plane zo+2 (slot (k+4)&7) has landed?
      mbar_wait(bars + ((k + 4) & 7), (uint32_t)((grp + (k >= 4 ? 1 : 0)) & 1));
      // normal plane zo+1 into normal slot (k+2)&3 from phi slots of zo, zo+1, zo+2
      {
        constexpr int om = ((k + 2) & 7) * C::SLOT, o0 = ((k + 3) & 7) * C::SLOT, op = ((k + 4) & 7) * C::SLOT;
        float* dst = Nr + ((k + 2) & 3) * 3 * C::NPL;
        const float fz = GEN ? ((zo + 1 == 0 || zo + 1 == nz - 1) ? 2.0f : 1.0f) : 1.0f;
        B::normal(Phi, own, om, o0, op, fz, inv2floor, dst);
        if (has_halo) B::normal(Phi, hal, om, o0, op, fz, inv2floor, dst);
      }
      __syncthreads();
      if (tid == 0) {
        // slot of plane zo-2 is free (last read in step zo-1): refill with zo+6
        if (zo + 6 <= z_stop + 1) {
          fence_proxy_async();
          issue_phi(zo + 6);
        }
        // the z pass of this group is done (all threads passed the barrier):
        // prefetch the next group's P window into the single buffer
        if (k == 0 && zc + C::G < z_stop && p_tma_ok(zc + C::G)) {
          fence_proxy_async();
          issue_p(zc + C::G);
        }
      }
      // ---- output voxel (x, y, zo)
      constexpr int s_m = ((k + 1) & 7) * C::SLOT, s_0 = ((k + 2) & 7) * C::SLOT, s_p = ((k + 3) & 7) * C::SLOT;
      constexpr int n_m = ((k + 0) & 3) * 3 * C::NPL, n_0 = ((k + 1) & 3) * 3 * C::NPL,
                    n_p = ((k + 2) & 3) * 3 * C::NPL;
      const float* pc = Phi + s_0 + own.s;
      const float cphi = pc[0];
      float kappa, lap;
      if constexpr (!GEN) {
        // kappa = div n (ops.cpp:281-316), doubled convention: 0.5 * sum of central differences
        const float dx = Nown[n_0 + 1] - Nown[n_0 - 1];
        const float dy = Nown[n_0 + C::NPL + C::NXr] - Nown[n_0 + C::NPL - C::NXr];
        const float dz = Nown[n_p + 2 * C::NPL] - Nown[n_m + 2 * C::NPL];
        kappa = 0.5f * ((dx + dy) + dz);
        // 7-point Laplacian (ops.cpp:249-277)
        lap = fmaf(-6.0f, cphi, ((pc[-1] + pc[1]) + (pc[-C::BX] + pc[C::BX])) + (Phi[s_m + own.s] + Phi[s_p + own.s]));
      } else {
        const float dx = (Nown[n_0 + kxp] - Nown[n_0 + kxm]) * kfx;
        const float dy = (Nown[n_0 + C::NPL + kyp] - Nown[n_0 + C::NPL + kym]) * kfy;
        // z face rule: zo == 0 -> n(1) - n(0); zo == nz-1 -> n(nz-1) - n(nz-2); factor 2
        const int nzp = zo + 1 <= nz - 1 ? n_p : n_0;
        const int nzm = zo - 1 >= 0 ? n_m : n_0;
        const float fz = (zo + 1 <= nz - 1 && zo - 1 >= 0) ? 1.0f : 2.0f;
        const float dz = (Nown[nzp + 2 * C::NPL] - Nown[nzm + 2 * C::NPL]) * fz;
        kappa = 0.5f * ((dx + dy) + dz);
        // clamped neighbours (the ring holds clamped planes in z)
        lap = fmaf(-6.0f, cphi, ((pc[own.dxm] + pc[own.dxp]) + (pc[own.dym] + pc[own.dyp])) +
                                    (Phi[s_m + own.s] + Phi[s_p + own.s]));
      }
      // delta_eps (rsf.cpp:96-107)
      const float delta = c.c_delta * rcp_approx(fmaf(cphi, cphi, c.eps2));
      // region averages r+- and F- - F+ (rsf.cpp:130-148, 164)
      const float km = kh[0][k].x, kmi = kh[0][k].y;
      float kp, kpi;
      if constexpr (NP == 2) {
        kp = kh[NP - 1][k].x;
        kpi = kh[NP - 1][k].y;
      } else {
        kp = 1.0f - km;
        kpi = k1ib[k & 7] - kmi;
      }
      const float ki = kib[k & 7];
      // the floored denominators are >= denom_floor > FLT_MIN: plain rcp.approx
      const float rp = fminf(fmaxf(kpi * rcp_approx(fmaxf(kp, c.denom_floor)), c.i_min), c.i_max);
      const float rm = fminf(fmaxf(kmi * rcp_approx(fmaxf(km, c.denom_floor)), c.i_min), c.i_max);
      const float dF = (rp - rm) * (fmaf(2.0f, ki, -rp) - rm);
      // combine (rsf.cpp:151-168) and explicit update (rsf.cpp:340-344)
      const float e = (lap - kappa) + delta * fmaf(c.alpha, kappa, c.beta * dF);
      const float f = fmaf(c.dt_f, e, cphi);
      if (col_ok) {
        out[(size_t)k * plane] = f;
        my_count += ((cphi < 0.0f) != (f < 0.0f)) ? 1u : 0u;
        if (!(fabsf(f) <= 3.402823466e38f))
          atomicMin(b.counters + 1, (unsigned long long)zo * (unsigned long long)plane + col);
      }
    };
    using F = std::false_type;
    using T = std::true_type;
    if (zfast) {
      step(std::integral_constant<int, 0>{}, F{});
      step(std::integral_constant<int, 1>{}, F{});
      step(std::integral_constant<int, 2>{}, F{});
      step(std::integral_constant<int, 3>{}, F{});
      step(std::integral_constant<int, 4>{}, F{});
      step(std::integral_constant<int, 5>{}, F{});
      step(std::integral_constant<int, 6>{}, F{});
      step(std::integral_constant<int, 7>{}, F{});
    } else {
      step(std::integral_constant<int, 0>{}, T{});
      step(std::integral_constant<int, 1>{}, T{});
      step(std::integral_constant<int, 2>{}, T{});
      step(std::integral_constant<int, 3>{}, T{});
      step(std::integral_constant<int, 4>{}, T{});
      step(std::integral_constant<int, 5>{}, T{});
      step(std::integral_constant<int, 6>{}, T{});
      step(std::integral_constant<int, 7>{}, T{});
    }
  }
}

template <int R, int NP>
__global__ void __launch_bounds__(256, 2)
    zst4_kernel(Geom g, Taps taps, StepConsts c, StepBuffers b, int z_begin, int z_end,
                const __grid_constant__ CUtensorMap map_phi, const __grid_constant__ CUtensorMap map_p0,
                const __grid_constant__ CUtensorMap map_p1) {
  using C = Z4<R, NP>;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned int s_count;
  const int z0 = z_begin + blockIdx.x * C::TZ;
  const int z_stop = min(z0 + C::TZ, z_end);
  const int x0 = blockIdx.y * C::TX, y0 = blockIdx.z * C::TY;
  const int bx0 = max(x0 - 4, 0), by0 = max(y0 - 2, 0);
  if (threadIdx.x == 0) s_count = 0;
  unsigned int my_count = 0;
  const bool interior = x0 >= 2 && x0 + C::TX + 2 <= g.nx && y0 >= 2 && y0 + C::TY + 2 <= g.ny;
  if (interior)
    zst4_cta<R, NP, false>(g, taps, c, b, z0, z_stop, x0, y0, bx0, by0, &map_phi, &map_p0, &map_p1, smem,
                           my_count);
  else
    zst4_cta<R, NP, true>(g, taps, c, b, z0, z_stop, x0, y0, bx0, by0, &map_phi, &map_p0, &map_p1, smem,
                          my_count);
  const unsigned int wsum = __reduce_add_sync(0xffffffffu, my_count);
  if ((threadIdx.x & 31) == 0 && wsum) atomicAdd(&s_count, wsum);
  __syncthreads();
  if (threadIdx.x == 0 && s_count) atomicAdd(b.counters, (unsigned long long)s_count);
}

template <int R, int NP>
int zst4_launch(const Geom& g, const Taps& t, const StepConsts& c, const StepBuffers& b, int z_begin, int z_end,
                const ZMaps& m, cudaStream_t st) {
  using C = Z4<R, NP>;
  if (C::kSmem > 227 * 1024) return -1;
  auto k = zst4_kernel<R, NP>;
  static bool attr = false;  // benign race: idempotent attribute set
  if (!attr) {
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem) != cudaSuccess)
      return -1;
    attr = true;
  }
  if (z_end <= z_begin) return 0;
  dim3 grid((z_end - z_begin + C::TZ - 1) / C::TZ, (g.nx + C::TX - 1) / C::TX, (g.ny + C::TY - 1) / C::TY);
  k<<<grid, C::NT, C::kSmem, st>>>(g, t, c, b, z_begin, z_end, m.phi, m.p[0], NP == 2 ? m.p[1] : m.p[0]);
  return 1;
}

}  // namespace

// Per-radius-group entry points (rsfg_zst4_g*.cu): -2 when r is not in the group.
#define RSFG_ZST4_GROUPS(X) X(0) X(1) X(2) X(3) X(4) X(5)
#define RSFG_ZST4_DECL(N)                                                                              \
  int zst4_group_##N(int r, const Geom& g, int fields, const Taps& t1, const StepConsts& c,             \
                     const StepBuffers& b, int z_begin, int z_end, const ZMaps& m, cudaStream_t st);    \
  int zst4_group_box_##N(int r, int fields, int* pbox_z);
RSFG_ZST4_GROUPS(RSFG_ZST4_DECL)
#undef RSFG_ZST4_DECL

}  // namespace rsfg
