// rsfg_zst4.cuh -- kernel 2 of the RSF step, TMA-fed z-streaming variant:
// z pass, region averages and force, curvature / Laplacian stencil, combine
// and explicit update (reference rsf.cpp:96-168, 324-352; ops.cpp:109-160,
// 199-316).  Same arithmetic as rsfg_zst.cu's kernel; what changes is how the
// data reaches the threads:
//
//  * phi planes, and the static fields K2*I (== I when sigma2 = 0) and K1*I
//    of the same plane, stream through an 8-slot shared ring filled by TMA
//    (one elected thread, one mbarrier per slot, four planes of prefetch), so
//    no thread spends instructions or registers staging them;
//  * the z-pass input window (8 + 2R planes of the kernel-1 pairs P for the
//    CTA's 32 x 8 columns) arrives as ONE 3-D TMA box per 8-plane group,
//    issued a whole group ahead into a single buffer;
//  * the plane loop is unrolled by 8 (the ring period), so every shared
//    access is a base register plus an immediate;
//  * a thread keeps its own column's phi (planes q-1..q+2), the four in-plane
//    phi neighbours of plane q and n_z (planes q-1..q+1) in registers: the
//    shared normal ring holds only n_x, n_y of two planes, and one barrier per
//    plane separates "normal of plane q+1" from "output of plane q", which run
//    interleaved in the same step (independent work for the scheduler);
//  * interior tiles away from the volume faces run a variant with constant
//    neighbour offsets and the 1/2 central-difference factors folded into a
//    doubled-gradient convention (n = 2g / max(|2g|, 2 floor) == g / max(|g|,
//    floor) exactly); tiles or plane groups that touch a face run the general
//    variant with clamped offsets and face factors (bitwise identical on
//    interior voxels: the factors there are exact 1s).
#pragma once
#include <type_traits>

#include "rsfg_device.cuh"

namespace rsfg {
namespace {

#ifndef RSFG_Z4_TALL_TY
#define RSFG_Z4_TALL_TY 8
#endif
// column-tile height for R <= 9, fields=2: 32 x 16 (one 512-thread CTA/SM,
// halo = 3 full warps) measured slower than 32 x 8 (zst 1.044 vs 0.962 ms)
constexpr int kZ4TallTY = RSFG_Z4_TALL_TY;

// Shared memory of a 32 x ty zst4 CTA at radius r (the Z4 layout below).
constexpr size_t z4_smem(int r, int np, int ty) {
  return (size_t)np * (8 + 2 * r) * 32 * ty * 8 + (size_t)8 * ((40 * (ty + 4) + 31) & ~31) * 4 +
         (size_t)8 * (np == 1 ? 2 : 1) * 32 * ty * 4 + (size_t)2 * 2 * 34 * (ty + 2) * 4 + 128;
}
// Column-tile height.  fields = 2: 32 x 8, or 32 x 6 where the 8-row z-pass
// window (8 + 2R planes of P) would leave one CTA per SM (R >= 16), or 32 x 4.
// fields = 4: 32 x 8, 32 x 4 from R = 17.
constexpr int z4_ty(int r, int np) {
  if (np == 2) return r >= 17 ? 4 : 8;
  if (r <= 9) return kZ4TallTY;
  if (z4_smem(r, np, 8) + 1024 <= 114 * 1024) return 8;
  if (z4_smem(r, np, 6) + 1024 <= 114 * 1024) return 6;
  return 4;
}

template <int R, int NP>
struct Z4 {
  static constexpr int TX = 32, TY = z4_ty(R, NP), NT = TX * TY;
  // phi TMA box (floats): x0-4.., y0-2..; ring slots padded to 128 bytes
  // (cp.async.bulk.tensor destinations must be 128-byte aligned)
  static constexpr int BX = 40, BY = TY + 4, BOXF = BX * BY, SLOT = (BOXF + 31) & ~31;
  static constexpr int NXr = TX + 2, NYr = TY + 2, NPL = NXr * NYr;  // normal plane, halo 1
  static constexpr int kHalo = 2 * TX + 2 * TY;           // halo positions kappa reads (no corners)
  static constexpr int kProducer = 3 * 32;                // TMA-issuing thread (warp 3, no halo work)
  static_assert(kHalo > 2 * 32 && kHalo <= 3 * 32 && NT >= 4 * 32, "halo slots: warps 0, 1 and part of warp 2");
  static constexpr int G = 8;                             // planes per group (z-pass chunk, ring period)
  static constexpr int TZ = 128;                          // planes per CTA
  static constexpr int NW = G + 2 * R;                    // z-pass window (planes)
  static constexpr int PPL = TX * TY;                     // float2 per P plane of the box
  static constexpr int NK = NP == 1 ? 2 : 1;              // static fields per plane: K2*I (+ K1*I)
  static constexpr size_t kPBytes = (size_t)NP * NW * PPL * sizeof(float2);
  static constexpr size_t kPhiBytes = (size_t)8 * SLOT * sizeof(float);
  static constexpr size_t kKBytes = (size_t)8 * NK * NT * sizeof(float);
  static constexpr size_t kNrBytes = (size_t)2 * 2 * NPL * sizeof(float);
  static constexpr size_t kSmem = kPBytes + kPhiBytes + kKBytes + kNrBytes + 16 * sizeof(uint64_t);
  // CTAs per SM the register budget is sized for: three 32 x 4 CTAs where their
  // shared memory allows it, else two (one for 32 x 16 tiles)
  static constexpr int kMinBlocks = TY == 16 ? 1 : (NP == 1 && 3 * (kSmem + 1024) <= 228 * 1024 ? 3 : 2);
  static constexpr uint32_t kSlotTx = (uint32_t)((BOXF + NK * NT) * sizeof(float));
};

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// One normal-plane position: phi-ring offset of its centre, in-plane
// neighbour deltas (clamped), doubled-convention factors (1 central, 2
// one-sided) and its offset in a normal-plane slot.
struct NPos {
  int s, dxm, dxp, dym, dyp, n;
  float fx, fy;
};

template <int R, int NP, bool GX, bool HH>
__device__ __forceinline__ void zst4_cta(const Geom& g, const Taps& taps, const StepConsts& c, const StepBuffers& b,
                                         int z0, int z_stop, int x0, int y0, int bx0, int by0,
                                         const CUtensorMap* map_phi, const CUtensorMap* map_ki,
                                         const CUtensorMap* map_k1i, const CUtensorMap* map_p0,
                                         const CUtensorMap* map_p1, unsigned char* smem, unsigned int& my_count) {
  using C = Z4<R, NP>;
  float2* Pb = reinterpret_cast<float2*>(smem);                       // [NP][NW][TY][TX]
  float* Phi = reinterpret_cast<float*>(smem + C::kPBytes);           // [8][BY][BX]
  float* Kr = Phi + 8 * C::SLOT;                                      // [8][NK][TY][TX]
  float* Nr = Kr + 8 * C::NK * C::NT;                                 // [2][2][NYr][NXr]  (n_x, n_y)
  uint64_t* bars = reinterpret_cast<uint64_t*>(Nr + 2 * 2 * C::NPL);  // [8] plane slots, [8] P buffer
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5, lane = tid & 31;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long plane = g.plane;
  const float inv2floor = 0.5f * c.inv_grad_floor;
  const bool producer_warp = __any_sync(0xffffffffu, tid == C::kProducer);  // warp-uniform
  bool any_bad = false;  // a non-finite phi' in this thread's outputs (rare; rescanned at the end)

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
  // halo: rows y0-1 and y0+TY (warps 0, 1), columns x0-1 and x0+TX (warp 2,
  // lanes 0..15); the TMA producer is warp 3 (kProducer), so no warp carries
  // two of the extra jobs into the per-plane barrier.
  // Warps 0..2 all take the halo branch (warp-uniform: no reconvergence
  // bookkeeping); warp 2's lanes past the last halo slot repeat its first
  // ones (same values to the same addresses).
  const bool has_halo = __any_sync(0xffffffffu, tid < C::kHalo);
  NPos hal = own;
  if (has_halo) {
    int i, j;
    const int h = tid < C::kHalo ? tid : 2 * C::TX + (tid - 2 * C::TX) % (C::kHalo - 2 * C::TX);
    if (h < C::TX) {
      i = h + 1, j = 0;
    } else if (h < 2 * C::TX) {
      i = h - C::TX + 1, j = C::NYr - 1;
    } else if (h < 2 * C::TX + C::TY) {
      i = 0, j = h - 2 * C::TX + 1;
    } else {
      i = C::NXr - 1, j = h - 2 * C::TX - C::TY + 1;
    }
    hal = make_pos(i, j);
  }
  // output voxel: kappa deltas in the normal plane, factors
  const int x = x0 + tx, y = y0 + ty;
  const bool col_ok = x < nx && y < ny;
  const int gxc = min(x, nx - 1), gyc = min(y, ny - 1);
  const int kxm = max(gxc - 1, 0) - gxc, kxp = min(gxc + 1, nx - 1) - gxc;
  const int kym = (max(gyc - 1, 0) - gyc) * C::NXr, kyp = (min(gyc + 1, ny - 1) - gyc) * C::NXr;
  const float kfx = (kxp - kxm) == 2 ? 1.0f : 2.0f;
  const float kfy = (kyp - kym) == 2 * C::NXr ? 1.0f : 2.0f;
  const size_t col = (size_t)gyc * nx + gxc;

  // ---- TMA producer (thread kProducer)
  auto zc_of = [&](int q) { return clampi(q, g.zb, g.ze - 1) - g.zb; };
  auto issue_plane = [&](int q) {  // phi, K2*I (, K1*I) of plane q -> slot (q - z0 + 2) & 7
    const int sl = (q - z0 + 2) & 7;
    mbar_expect_tx(bars + sl, C::kSlotTx);
    tma_load_3d(Phi + sl * C::SLOT, map_phi, bars + sl, bx0, by0, zc_of(q));
    tma_load_3d(Kr + sl * C::NK * C::NT, map_ki, bars + sl, x0, y0, zc_of(q));
    if (NP == 1) tma_load_3d(Kr + (sl * C::NK + 1) * C::NT, map_k1i, bars + sl, x0, y0, zc_of(q));
  };
  // P window of the group starting at zc: TMA when it lies inside the held
  // planes (no clamping needed), else threads load it with clamped LDG.
  auto p_tma_ok = [&](int zc) { return zc - R >= g.zb && zc + C::G + R <= g.ze; };
  auto issue_p = [&](int zc) {
    mbar_expect_tx(bars + 8, (uint32_t)C::kPBytes);
    tma_load_3d(Pb, map_p0, bars + 8, 2 * x0, y0, zc - R - g.zb);
    if (NP == 2) tma_load_3d(Pb + C::NW * C::PPL, map_p1, bars + 8, 2 * x0, y0, zc - R - g.zb);
  };

  if (tid == C::kProducer) {
    for (int i = 0; i < 9; ++i) mbar_init(bars + i, 1);
    const int last = min(z0 + 5, z_stop + 1);
    for (int q = z0 - 2; q <= last; ++q) issue_plane(q);
    if (p_tma_ok(z0)) issue_p(z0);
  }
  __syncthreads();

  // normal at a halo position of plane q (ring slots om, o0, op of q-1, q, q+1)
  auto halo_normal = [&](auto genc, int om, int o0, int op, float fz, float* dst) {
    constexpr bool GEN = decltype(genc)::value;
    const float* c0 = Phi + o0 + hal.s;
    float a, bb, cc;
    if constexpr (GEN) {
      a = (c0[hal.dxp] - c0[hal.dxm]) * hal.fx;
      bb = (c0[hal.dyp] - c0[hal.dym]) * hal.fy;
      cc = (Phi[op + hal.s] - Phi[om + hal.s]) * fz;
    } else {
      a = c0[1] - c0[-1];
      bb = c0[C::BX] - c0[-C::BX];
      cc = Phi[op + hal.s] - Phi[om + hal.s];
    }
    const float inv = fminf(rsqrt_approx(fmaf(a, a, fmaf(bb, bb, cc * cc))), inv2floor);
    dst[hal.n] = a * inv;
    dst[C::NPL + hal.n] = bb * inv;
  };
  auto fzq = [&](int q) { return (q == 0 || q == nz - 1) ? 2.0f : 1.0f; };

  // ---- prologue: planes z0-2 .. z0+1 in slots 0..3
  for (int sl = 0; sl < 4; ++sl) mbar_wait(bars + sl, 0);
  const float* Pown = Phi + own.s;
  float cm1 = Pown[1 * C::SLOT], c0 = Pown[2 * C::SLOT], cp1 = Pown[3 * C::SLOT];  // own phi z0-1, z0, z0+1
  float nzm1, nz0;                                                                   // own n_z at z0-1, z0
  float xm0, xp0, ym0, yp0;  // phi(z0) at the clamped in-plane neighbours
  {
    // n_z at (x, y, z0-1): needs the full gradient there
    const float* p = Pown + 1 * C::SLOT;
    const float a = (p[own.dxp] - p[own.dxm]) * own.fx, bb = (p[own.dyp] - p[own.dym]) * own.fy;
    const float cc = (c0 - Pown[0]) * fzq(z0 - 1);
    nzm1 = cc * fminf(rsqrt_approx(fmaf(a, a, fmaf(bb, bb, cc * cc))), inv2floor);
  }
  {
    const float* p = Pown + 2 * C::SLOT;
    xm0 = p[own.dxm], xp0 = p[own.dxp], ym0 = p[own.dym], yp0 = p[own.dyp];
    const float a = (xp0 - xm0) * own.fx, bb = (yp0 - ym0) * own.fy, cc = (cp1 - cm1) * fzq(z0);
    const float inv = fminf(rsqrt_approx(fmaf(a, a, fmaf(bb, bb, cc * cc))), inv2floor);
    Nr[own.n] = a * inv;  // normal slot 0 <-> plane z0
    Nr[C::NPL + own.n] = bb * inv;
    nz0 = cc * inv;
    if (has_halo) halo_normal(std::true_type{}, 1 * C::SLOT, 2 * C::SLOT, 3 * C::SLOT, fzq(z0), Nr);
  }

  uint32_t pphase = 0;
#pragma unroll 1
  for (int zc = z0, grp = 0; zc < z_stop; zc += C::G, ++grp) {
    // ---- z pass for planes zc .. zc+7 (fp32 FMA per tap, ascending tap
    // order like the reference's f32-rounded z pass, ops.cpp:150-155),
    // scattered from one window plane at a time into 8 accumulators.
    float2 kh[NP][C::G];
    auto zpass = [&](auto load) {
#pragma unroll
      for (int np = 0; np < NP; ++np) {
#pragma unroll
        for (int kk = 0; kk < C::NW; ++kk) {
          const float2 v = load(np, kk);
#pragma unroll
          for (int t = 0; t < C::G; ++t) {
            const int j = kk - t;
            if (j == 0) kh[np][t] = fmul2(taps.w[0], v);
            else if (j > 0 && j <= 2 * R) kh[np][t] = ffma2(taps.w[j], v, kh[np][t]);
          }
        }
      }
    };
    if (p_tma_ok(zc)) {
      mbar_wait(bars + 8, pphase);
      pphase ^= 1;
      const float2* src = Pb + tid;
      zpass([&](int np, int kk) { return src[(np * C::NW + kk) * C::PPL]; });
    } else {
      zpass([&](int np, int kk) {
        return __ldg(b.P[np] + col + (size_t)(clampi(zc - R + kk, g.zb, g.ze - 1) - g.zb) * (size_t)plane);
      });
    }

    const bool zfast = !GX && zc >= 1 && zc + C::G <= nz - 2 && zc + C::G <= z_stop;
    float* out = b.out + (size_t)(zc - g.zb) * plane + col;
    float2* hh_out = HH ? b.hh + (size_t)(zc - g.zb) * plane + col : nullptr;
    float f_prev = 0.0f, ki_prev = 0.0f;  // fast path: Heaviside pairs of planes (q-1, q), packed

    auto step = [&](auto kc, auto genc) {
      constexpr int k = decltype(kc)::value;
      constexpr bool GEN = decltype(genc)::value;
      const int q = zc + k;
      if (GEN && q >= z_stop) return;  // partial last group (uniform)
      constexpr int o0 = ((k + 2) & 7) * C::SLOT, o1 = ((k + 3) & 7) * C::SLOT, o2 = ((k + 4) & 7) * C::SLOT;
      constexpr int nq = (k & 1) * 2 * C::NPL, nq1 = ((k + 1) & 1) * 2 * C::NPL;
      // normals of plane q (written in step q-1) complete; everybody is done
      // with step q-1, so the ring slot of plane q-2 is free
      __syncthreads();
      if (producer_warp && lane == 0) {
        if (q + 6 <= z_stop + 1) {
          fence_proxy_async();
          issue_plane(q + 6);
        }
        // the z pass of this group is done: next group's P window
        if (k == 0 && zc + C::G < z_stop && p_tma_ok(zc + C::G)) {
          fence_proxy_async();
          issue_p(zc + C::G);
        }
      }
      // plane q+2 (slot (k+4)&7) landed?  Issued for step q-4 / the prologue.
      mbar_wait(bars + ((k + 4) & 7), (uint32_t)((grp + (k >= 4 ? 1 : 0)) & 1));

      // Shared loads first: the output's normals of plane q and static
      // fields, then the phi of plane q+1 -- ahead of this step's normal
      // stores, which the compiler must otherwise keep them behind.
      const float* N0 = Nr + nq + own.n;
      float nxm, nxp, nym, nyp;
      if constexpr (!GEN) {
        nxm = N0[-1], nxp = N0[1], nym = N0[C::NPL - C::NXr], nyp = N0[C::NPL + C::NXr];
      } else {
        nxm = N0[kxm], nxp = N0[kxp], nym = N0[C::NPL + kym], nyp = N0[C::NPL + kyp];
      }
      const float* K = Kr + ((k + 2) & 7) * C::NK * C::NT + tid;
      const float ki = K[0];
      [[maybe_unused]] const float k1i = NP == 1 ? K[C::NT] : 0.0f;
      const float* p1 = Pown + o1;
      float xm1, xp1, ym1, yp1;
      if constexpr (GEN) {
        xm1 = p1[own.dxm], xp1 = p1[own.dxp], ym1 = p1[own.dym], yp1 = p1[own.dyp];
      } else {
        xm1 = p1[-1], xp1 = p1[1], ym1 = p1[-C::BX], yp1 = p1[C::BX];
      }
      const float cp2 = Pown[o2];

      // ---- A: own normal at plane q+1 (n_x, n_y -> shared; n_z stays here)
      float a = xp1 - xm1, bb = yp1 - ym1, cc = cp2 - c0;
      if constexpr (GEN) {
        a *= own.fx;
        bb *= own.fy;
        cc *= fzq(q + 1);
      }
      const float inv = fminf(rsqrt_approx(fmaf(a, a, fmaf(bb, bb, cc * cc))), inv2floor);
      const float nzp1 = cc * inv;
      if (has_halo) halo_normal(genc, o0, o1, o2, GEN ? fzq(q + 1) : 1.0f, Nr + nq1);
      Nr[nq1 + own.n] = a * inv;
      Nr[nq1 + C::NPL + own.n] = bb * inv;

      // ---- B: output voxel (x, y, q)
      float kappa;
      if constexpr (!GEN) {
        // kappa = div n (ops.cpp:281-316), doubled convention: 0.5 * sum of central differences
        kappa = 0.5f * (((nxp - nxm) + (nyp - nym)) + (nzp1 - nzm1));
      } else {
        const float dx = (nxp - nxm) * kfx;
        const float dy = (nyp - nym) * kfy;
        // z face rule: q == 0 -> n(1) - n(0); q == nz-1 -> n(nz-1) - n(nz-2); factor 2
        const float zp = q + 1 <= nz - 1 ? nzp1 : nz0;
        const float zm = q - 1 >= 0 ? nzm1 : nz0;
        const float fz = (q + 1 <= nz - 1 && q - 1 >= 0) ? 1.0f : 2.0f;
        kappa = 0.5f * ((dx + dy) + (zp - zm) * fz);
      }
      // 7-point Laplacian, clamp-to-edge (ops.cpp:249-277; the ring holds clamped planes)
      const float lap = fmaf(-6.0f, c0, ((xm0 + xp0) + (ym0 + yp0)) + (cm1 + cp1));
      // delta_eps (rsf.cpp:96-107)
      const float delta = c.c_delta * rcp_approx(fmaf(c0, c0, c.eps2));
      // region averages r+- and F- - F+ (rsf.cpp:130-148, 164)
      const float km = kh[0][k].x, kmi = kh[0][k].y;
      float kp, kpi;
      if constexpr (NP == 2) {
        kp = kh[NP - 1][k].x;
        kpi = kh[NP - 1][k].y;
      } else {
        kp = 1.0f - km;
        kpi = k1i - kmi;
      }
      // the floored denominators are >= denom_floor > FLT_MIN: plain rcp.approx
      const float rp = fminf(fmaxf(kpi * rcp_approx(fmaxf(kp, c.denom_floor)), c.i_min), c.i_max);
      const float rm = fminf(fmaxf(kmi * rcp_approx(fmaxf(km, c.denom_floor)), c.i_min), c.i_max);
      const float dF = (rp - rm) * (fmaf(2.0f, ki, -rp) - rm);
      // combine (rsf.cpp:151-168) and explicit update (rsf.cpp:340-344)
      const float e = (lap - kappa) + delta * fmaf(c.alpha, kappa, c.beta * dF);
      const float f = fmaf(c.dt_f, e, c0);
      if (!GX || col_ok) {
        out[(size_t)k * plane] = f;
        if constexpr (HH) {  // stored-Heaviside mode: kernel 1 of the next step reads (H-, H- I) of phi'
          if constexpr (!GEN) {
            // full 8-plane group: evaluate planes (q-1, q) as one packed pair
            // (same bits as the scalar heaviside_pair)
            if constexpr ((k & 1) == 0) {
              f_prev = f;
              ki_prev = ki;
            } else {
              float2 hm2, hp2;
              heaviside2<false>(make_float2(f_prev, f), c.inv_eps, hm2, hp2);
              const float2 hmi = f2mul(hm2, make_float2(ki_prev, ki));
              hh_out[(size_t)(k - 1) * plane] = make_float2(hm2.x, hmi.x);
              hh_out[(size_t)k * plane] = make_float2(hm2.y, hmi.y);
            }
          } else {
            float hm, hp;
            heaviside_pair(f, c.inv_eps, hm, hp);
            hh_out[(size_t)k * plane] = make_float2(hm, hm * ki);
          }
        }
        my_count += ((c0 < 0.0f) != (f < 0.0f)) ? 1u : 0u;
        any_bad |= !(fabsf(f) <= 3.402823466e38f);
      }
      // ---- rotate the register windows to plane q+1
      cm1 = c0;
      c0 = cp1;
      cp1 = cp2;
      xm0 = xm1, xp0 = xp1, ym0 = ym1, yp0 = yp1;
      nzm1 = nz0;
      nz0 = nzp1;
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
  // Rare path (evolve_step's blowup report, rsf.cpp:324-352): some thread saw a
  // non-finite phi'.  Rescan this thread's column of the CTA's planes for the
  // first one (the CTA's own stores, visible to the thread that made them).
  if (__any_sync(0xffffffffu, any_bad) && any_bad) {
    for (int q = z0; q < z_stop; ++q) {
      const float f = b.out[(size_t)(q - g.zb) * plane + col];
      if (!(fabsf(f) <= 3.402823466e38f)) {
        atomicMin(b.counters + 1, (unsigned long long)q * (unsigned long long)plane + col);
        break;
      }
    }
  }
}

template <int R, int NP, bool HH>
__global__ void __launch_bounds__(Z4<R, NP>::NT, Z4<R, NP>::kMinBlocks)
    zst4_kernel(Geom g, Taps taps, StepConsts c, StepBuffers b, int z_begin, int z_end,
                const __grid_constant__ CUtensorMap map_phi, const __grid_constant__ CUtensorMap map_ki,
                const __grid_constant__ CUtensorMap map_k1i, const __grid_constant__ CUtensorMap map_p0,
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
    zst4_cta<R, NP, false, HH>(g, taps, c, b, z0, z_stop, x0, y0, bx0, by0, &map_phi, &map_ki, &map_k1i, &map_p0,
                           &map_p1, smem, my_count);
  else
    zst4_cta<R, NP, true, HH>(g, taps, c, b, z0, z_stop, x0, y0, bx0, by0, &map_phi, &map_ki, &map_k1i, &map_p0,
                          &map_p1, smem, my_count);
  const unsigned int wsum = __reduce_add_sync(0xffffffffu, my_count);
  if ((threadIdx.x & 31) == 0 && wsum) atomicAdd(&s_count, wsum);
  __syncthreads();
  if (threadIdx.x == 0 && s_count) atomicAdd(b.counters, (unsigned long long)s_count);
}

template <int R, int NP, bool HH>
int zst4_launch_v(const Geom& g, const Taps& t, const StepConsts& c, const StepBuffers& b, int z_begin, int z_end,
                  const ZMaps& m, cudaStream_t st) {
  using C = Z4<R, NP>;
  if (C::kSmem > 227 * 1024) return -1;
  auto k = zst4_kernel<R, NP, HH>;
  if (!smem_optin<zst4_kernel<R, NP, HH>>((int)C::kSmem)) return -1;
  if (z_end <= z_begin) return 0;
  dim3 grid((z_end - z_begin + C::TZ - 1) / C::TZ, (g.nx + C::TX - 1) / C::TX, (g.ny + C::TY - 1) / C::TY);
  k<<<grid, C::NT, C::kSmem, st>>>(g, t, c, b, z_begin, z_end, m.phi, m.ki, NP == 1 ? m.k1i : m.ki, m.p[0],
                                   NP == 2 ? m.p[1] : m.p[0]);
  return 1;
}

// The stored-Heaviside variant exists for the radii where the mode pays
// (R <= kHHMaxR, rsfg_api.cu make_xy2_maps); elsewhere b.hh is never set.
template <int R, int NP>
int zst4_launch(const Geom& g, const Taps& t, const StepConsts& c, const StepBuffers& b, int z_begin, int z_end,
                const ZMaps& m, cudaStream_t st) {
  if constexpr (NP == 1 && R <= kHHMaxR) {
    if (b.hh) return zst4_launch_v<R, NP, true>(g, t, c, b, z_begin, z_end, m, st);
  }
  if (b.hh) return -1;
  return zst4_launch_v<R, NP, false>(g, t, c, b, z_begin, z_end, m, st);
}

}  // namespace

// Per-radius-group entry points (rsfg_zst4_g*.cu): -2 when r is not in the group.
#define RSFG_ZST4_GROUPS(X) X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13)
#define RSFG_ZST4_DECL(N)                                                                              \
  int zst4_group_##N(int r, const Geom& g, int fields, const Taps& t1, const StepConsts& c,             \
                     const StepBuffers& b, int z_begin, int z_end, const ZMaps& m, cudaStream_t st);    \
  int zst4_group_box_##N(int r, int fields, int* pbox_z, int* ty);
RSFG_ZST4_GROUPS(RSFG_ZST4_DECL)
#undef RSFG_ZST4_DECL

// Body of one radius-group translation unit (rsfg_zst4_g*.cu): the P-window
// box (rows = the launched kernel's tile) and the launch of every radius in RADII.
#define RSFG_ZST4_BOX_CASE(R)                                                   \
  case R:                                                                       \
    *pbox_z = Z4<R, 1>::NW;                                                     \
    *ty = fields == 4 ? Z4<R, 2>::TY : Z4<R, 1>::TY;                            \
    return (fields == 4 ? Z4<R, 2>::kSmem : Z4<R, 1>::kSmem) <= 227 * 1024;
#define RSFG_ZST4_LAUNCH_CASE(R)                                                \
  case R:                                                                       \
    return fields == 4 ? zst4_launch<R, 2>(g, t1, c, b, z_begin, z_end, m, st)  \
                       : zst4_launch<R, 1>(g, t1, c, b, z_begin, z_end, m, st);
#define RSFG_ZST4_GROUP(N, RADII)                                                                            \
  int zst4_group_box_##N(int r, int fields, int* pbox_z, int* ty) {                                        \
    switch (r) {                                                                                           \
      RADII(RSFG_ZST4_BOX_CASE)                                                                            \
      default:                                                                                             \
        return -2;                                                                                         \
    }                                                                                                      \
  }                                                                                                        \
  int zst4_group_##N(int r, const Geom& g, int fields, const Taps& t1, const StepConsts& c,                 \
                     const StepBuffers& b, int z_begin, int z_end, const ZMaps& m, cudaStream_t st) {      \
    switch (r) {                                                                                           \
      RADII(RSFG_ZST4_LAUNCH_CASE)                                                                         \
      default:                                                                                             \
        return -2;                                                                                         \
    }                                                                                                      \
  }

}  // namespace rsfg
