// rsfg_xy2.cuh -- kernel 1 of the RSF step, multi-plane TMA variant:
// Heaviside fields of a haloed z-plane tile, then the x and y passes of the
// separable Gaussian (reference rsf.cpp:75-94, ops.cpp:74-160).  Same
// arithmetic and output (P pairs) as rsfg_xy.cu; what changes:
//
//  * the y pass runs first (it carries the x halo: WX/TX = 1.28 < WY/TY =
//    1.56 at R = 9), then the x pass writes a staging tile that leaves as
//    coalesced 16-byte stores;
//  * a CTA owns one 64 x TY tile for NZC consecutive planes.  The raw phi and
//    I tiles of plane z+1 are requested by TMA (one thread, one mbarrier) as
//    soon as the Heaviside phase of plane z has consumed plane z's, so the
//    load overlaps the x and y passes; no thread issues a global load;
//  * the Heaviside fields of two adjacent voxels are evaluated with packed
//    f32x2 arithmetic (FMUL2/FFMA2/FADD2: the atan polynomial runs once per
//    pair), reading both voxels' phi and I with one 64-bit shared load each;
//  * every tile loads the same box layout (origin (x0 - R) rounded down to
//    16 bytes, possibly negative); edge tiles first overwrite the positions
//    outside the volume with their clamp-to-edge values, then all tiles run
//    the same paired path.
#pragma once
#include "rsfg_device.cuh"

namespace rsfg {
namespace {

template <int R, int NP, int TY>
struct XY2 {
  static constexpr int TX = 64;
  static constexpr int NT = TY >= 64 ? 512 : 256;
  static constexpr int NZC = 8;  // planes per CTA
  static constexpr int WX = TX + 2 * R, WY = TY + 2 * R;
  // TMA box row: starts at (x0 - R) rounded down to 4 floats (16 bytes)
  static constexpr int BOXX = (WX + 3 + 3) & ~3;
  static constexpr int SHIFT = (64 * 1024 - R) & 3;  // (x0 - R) mod 4 for x0 % 64 == 0
  static constexpr int BX = 8, BY = 8;               // outputs per x-pass / y-pass item
  // interior Heaviside: pairs of raw columns [C0, C0 + 2*NPR) cover [SHIFT, SHIFT + WX)
  static constexpr int C0 = SHIFT & ~1;
  static constexpr int NPR = (SHIFT + WX - C0 + 1) / 2;
  // Hs [NP][WY][PH]: H pairs of the haloed tile, raw-column indexed; PH even so a
  // pair of voxels is one aligned 16-byte store (the y pass reads it along x).
  static constexpr int PH = (C0 + 2 * NPR + 1) & ~1;
  // Ys [NP][TY][PY]: y-pass output on the WX window columns; PY odd so the x pass
  // (lanes walk rows) hits 16 distinct bank pairs per half-warp.
  static constexpr int PY = WX | 1;
  // Os [NP][TY][PO]: x-pass output staging for coalesced 16-byte global stores;
  // PO = TX + 2 makes the row-strided 16-byte stores conflict-free.
  static constexpr int PO = TX + 2;
  static constexpr size_t kHsBytes = ((size_t)NP * WY * PH * sizeof(float2) + 127) & ~(size_t)127;
  static constexpr size_t kYsBytes = ((size_t)NP * TY * PY * sizeof(float2) + 127) & ~(size_t)127;
  static constexpr size_t kOsBytes = ((size_t)NP * TY * PO * sizeof(float2) + 127) & ~(size_t)127;
  static constexpr size_t kTile = ((size_t)BOXX * WY * sizeof(float) + 127) & ~(size_t)127;
  // Os gets its own space when two CTAs still fit an SM; otherwise it aliases
  // Hs (free after the y pass) at the cost of one more barrier per plane.
  static constexpr bool kOsAlias = kHsBytes + kYsBytes + kOsBytes + 2 * kTile + 16 > 112 * 1024 &&
                                   kOsBytes <= kHsBytes;
  static constexpr size_t kSmem = kHsBytes + kYsBytes + (kOsAlias ? 0 : kOsBytes) + 2 * kTile + 16;
  // stored-Heaviside variant (xy2_cta_hh): two (H-, H- I) tile buffers, Ys, Os
  static constexpr size_t kTileHH = ((size_t)BOXX * WY * sizeof(float2) + 127) & ~(size_t)127;
  // Two (H-, H- I) tile buffers (plane z+1 lands while plane z is filtered)
  // while that still leaves two CTAs per SM; past that (R >= 11 at 64 x 32)
  // one buffer, refilled as soon as the y pass has consumed it.
  static constexpr bool kHHDouble = 2 * kTileHH + kYsBytes + kOsBytes + 16 <= 113 * 1024;
  static constexpr int kHHBufs = kHHDouble ? 2 : 1;
  static constexpr size_t kSmemHH = kHHBufs * kTileHH + kYsBytes + kOsBytes + 16;
  static constexpr int RG = NT / NPR;                     // row groups of phase A
  static constexpr int RITER = (WY + RG - 1) / RG;        // rows per phase-A thread
  static constexpr int YIT = (NP * WX * (TY / BY) + NT - 1) / NT;  // y-pass items per thread
  static constexpr int XIT = (NP * TY * (TX / BX) + NT - 1) / NT;  // x-pass items per thread
  static constexpr int OIT = (NP * TY * TX / 2 + NT - 1) / NT;     // copy-out float4 per thread
  // Stored-Heaviside variant's y pass: the WX window columns x NSEGH row
  // segments of BYH outputs, sized so the items fill the CTA once (64 x 32,
  // R = 9: 82 x 3 = 246 items of 11 rows, where 8-row segments gave 328 items
  // = 1.28 rounds with 72 threads busy in the second).  The last segment ends
  // at row TY and may overlap its neighbour; it skips the rows already stored.
  // Segment count for np field pairs: least work on the busiest thread
  // (rounds x (FFMA2 + 2 x LDS.64 per item); shared loads weigh double, the
  // pass is LSU-heavy), register window BY + 2R <= 52 pairs unless the plain
  // 8-row split (always a candidate) is already wider.
  static constexpr long seg_cost(int np, int s) {
    const int by = (TY + s - 1) / s;
    return (long)((np * WX * s + NT - 1) / NT) * (by * (2 * R + 1) + 2 * (by + 2 * R));
  }
  static constexpr int nseg(int np) {
    int best = TY / BY;
    long best_cost = seg_cost(np, best);
    for (int s = 1; s <= TY; ++s) {
      const int by = (TY + s - 1) / s;
      if (by + 2 * R > 52) continue;
      if (seg_cost(np, s) < best_cost) best_cost = seg_cost(np, s), best = s;
    }
    return best;
  }
  static constexpr int NSEGH = nseg(1);
  static constexpr int BYH = (TY + NSEGH - 1) / NSEGH;
  static constexpr int YITH = (WX * NSEGH + NT - 1) / NT;
  // The Heaviside-computing variant keeps 8-row segments: the cost model's
  // picks for it (R = 12: 8 x 4 rows; R >= 15: 5 x 13 rows) measured slower or
  // equal (sigma 4: 1.87 vs 1.81 ms/step) -- its Hs tile traffic dominates.
  static constexpr int NSEG = TY / BY;
  static constexpr int BYS = (TY + NSEG - 1) / NSEG;
  static constexpr int YITS = (NP * WX * NSEG + NT - 1) / NT;
};

template <int R, int NP, int TY, bool EDGE>
__device__ __forceinline__ void xy2_cta(const Geom& g, const Taps& taps, float inv_eps, float2* __restrict__ P0,
                                        float2* __restrict__ P1, int z_first, int z_last, int x0, int y0,
                                        const CUtensorMap* map_phi, const CUtensorMap* map_img,
                                        unsigned char* smem) {
  using C = XY2<R, NP, TY>;
  // Hs, Ys and Os are disjoint (Os == Hs only under kOsAlias, whose phases a
  // barrier separates): restrict lets loads of one item pass stores of another.
  float2* __restrict__ Hs = reinterpret_cast<float2*>(smem);                            // [NP][WY][PH]
  float2* __restrict__ Ys = reinterpret_cast<float2*>(smem + C::kHsBytes);              // [NP][TY][PY]
  float2* __restrict__ Os =
      C::kOsAlias ? Hs : reinterpret_cast<float2*>(smem + C::kHsBytes + C::kYsBytes);  // [NP][TY][PO]
  float* Tphi =
      reinterpret_cast<float*>(smem + C::kHsBytes + C::kYsBytes + (C::kOsAlias ? 0 : C::kOsBytes));  // [WY][BOXX]
  float* Timg = Tphi + C::kTile / sizeof(float);
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(Tphi) + 2 * C::kTile);
  const int tid = threadIdx.x;
  // Box origin: (x0 - R) rounded down to 16 bytes, y0 - R.  Starts may be
  // negative (TMA zero-fills outside the volume; only a non-16-byte-aligned x
  // start faults, tools/microbench/tma_neg.cu); edge tiles then overwrite the
  // outside positions with their clamp-to-edge values (ops.cpp:48-70) so
  // every tile runs the same paired Heaviside path.
  const int bx0 = x0 - R - C::SHIFT, by0 = y0 - R;

  // ---- per-thread work descriptors (constant across the CTA's planes)
  // phase A: pair column pc of row group rg
  const int a_pc = tid % C::NPR, a_rg = tid / C::NPR;
  const bool a_on = a_rg < C::RG;
  const bool a_last = a_rg + (C::RITER - 1) * C::RG < C::WY;
  const float* Ta = Tphi + a_rg * C::BOXX + C::C0 + 2 * a_pc;
  float2* Ha = Hs + a_rg * C::PH + C::C0 + 2 * a_pc;
  // phase B (y pass): lanes walk the window columns cx;
  // y-pass items (np, segment, column): NSEG row segments of BYS outputs, the
  // last ending at row TY (rows its neighbour wrote are not stored twice)
  int ysrc[C::YITS], ydst[C::YITS], yskip[C::YITS];
#pragma unroll
  for (int i = 0; i < C::YITS; ++i) {
    const int it = min(tid + i * C::NT, NP * C::WX * C::NSEG - 1);
    const int np = it / (C::WX * C::NSEG);
    const int rem = it - np * C::WX * C::NSEG;
    const int sy = rem / C::WX, cx = rem - sy * C::WX;
    const int r0 = sy < C::NSEG - 1 ? sy * C::BYS : TY - C::BYS;
    ysrc[i] = np * C::WY * C::PH + r0 * C::PH + C::SHIFT + cx;
    ydst[i] = np * TY * C::PY + r0 * C::PY + cx;
    yskip[i] = sy < C::NSEG - 1 ? 0 : (C::NSEG - 1) * C::BYS - r0;
  }
  const bool y_last = tid + (C::YITS - 1) * C::NT < NP * C::WX * C::NSEG;
  // phase C (x pass) items -> (np, sx, row): lanes walk rows
  int xsrc[C::XIT], xdst[C::XIT];
  constexpr int SEGX = C::TX / C::BX;
#pragma unroll
  for (int i = 0; i < C::XIT; ++i) {
    const int it = min(tid + i * C::NT, NP * TY * SEGX - 1);
    const int np = it / (TY * SEGX);
    const int rem = it - np * TY * SEGX;
    const int sx = rem / TY, row = rem - sx * TY;
    xsrc[i] = np * TY * C::PY + row * C::PY + sx * C::BX;
    xdst[i] = np * TY * C::PO + row * C::PO + sx * C::BX;
  }
  const bool x_last = tid + (C::XIT - 1) * C::NT < NP * TY * SEGX;
  // phase D (copy-out) float4 items -> (np, row, column pair)
  int osrc[C::OIT];
  size_t odst[C::OIT];
  bool o_np[C::OIT], o_ok[C::OIT];
#pragma unroll
  for (int i = 0; i < C::OIT; ++i) {
    const int it = min(tid + i * C::NT, NP * TY * C::TX / 2 - 1);
    const int np = it / (TY * C::TX / 2);
    const int rem = it - np * TY * C::TX / 2;
    const int row = rem / (C::TX / 2), cp = rem - row * (C::TX / 2);
    osrc[i] = np * TY * C::PO + row * C::PO + 2 * cp;
    const int gx = x0 + 2 * cp, gy = y0 + row;
    o_np[i] = np != 0;
    o_ok[i] = tid + i * C::NT < NP * TY * C::TX / 2 && (!EDGE || (gx < g.nx && gy < g.ny));
    odst[i] = (size_t)min(gy, g.ny - 1) * g.nx + min(gx, g.nx - 2);
  }

  auto issue = [&](int z) {
    mbar_expect_tx(bar, (uint32_t)(2 * C::BOXX * C::WY * sizeof(float)));
    tma_load_3d(Tphi, map_phi, bar, bx0, by0, z - g.zb);
    tma_load_3d(Timg, map_img, bar, bx0, by0, z - g.zb);
  };
  if (tid == 0) {
    mbar_init(bar, 1);
    issue(z_first);
  }
  __syncthreads();

#pragma unroll 1
  for (int z = z_first, ph = 0; z < z_last; ++z, ph ^= 1) {
    mbar_wait(bar, (uint32_t)ph);
    if constexpr (EDGE) {
      // raw columns [0, lo) lie left of x = 0, [hi, BOXX) right of nx - 1
      const int lo = max(0, -bx0), hi = min(C::BOXX, g.nx - bx0);
      const int nfix = lo + (C::BOXX - hi);
      for (int e = tid; e < C::WY * nfix; e += C::NT) {
        const int ry = e / nfix, k = e - ry * nfix;
        const int cdst = k < lo ? k : hi + (k - lo);
        const int csrc = k < lo ? lo : hi - 1;
        Tphi[ry * C::BOXX + cdst] = Tphi[ry * C::BOXX + csrc];
        Timg[ry * C::BOXX + cdst] = Timg[ry * C::BOXX + csrc];
      }
      __syncthreads();
      // rows [0, ylo) above y = 0, [yhi, WY) below ny - 1 (whole rows, after the column fix)
      const int ylo = max(0, -by0), yhi = min(C::WY, g.ny - by0);
      const int nrow = ylo + (C::WY - yhi);
      for (int e = tid; e < nrow * C::BOXX; e += C::NT) {
        const int k = e / C::BOXX, cx = e - k * C::BOXX;
        const int rdst = k < ylo ? k : yhi + (k - ylo);
        const int rsrc = k < ylo ? ylo : yhi - 1;
        Tphi[rdst * C::BOXX + cx] = Tphi[rsrc * C::BOXX + cx];
        Timg[rdst * C::BOXX + cx] = Timg[rsrc * C::BOXX + cx];
      }
      __syncthreads();
    }
    // ---- Phase A: Heaviside fields of the haloed tile -> Hs.  Pairs of raw
    // columns (c, c+1), c even: one LDS.64 of phi and of I each, one 16-byte
    // store.  Thread (rg, pc) owns pair column pc of rows rg, rg + RG, ...
    if (a_on) {
      // all of this thread's loads first (the stores below may alias them as
      // far as the compiler knows), then the packed Heaviside and the stores
      float2 pv[C::RITER], iv[C::RITER];
#pragma unroll
      for (int i = 0; i < C::RITER; ++i) {
        if (i < C::RITER - 1 || a_last) {
          pv[i] = *reinterpret_cast<const float2*>(Ta + i * C::RG * C::BOXX);
          iv[i] = *reinterpret_cast<const float2*>(Ta + C::kTile / sizeof(float) + i * C::RG * C::BOXX);
        }
      }
#pragma unroll
      for (int i = 0; i < C::RITER; ++i) {
        if (i < C::RITER - 1 || a_last) {
          const int ro = i * C::RG;
          float2 hm, hp;
          heaviside2<NP == 2>(pv[i], inv_eps, hm, hp);
          const float2 hmi = f2mul(hm, iv[i]);
          *reinterpret_cast<float4*>(Ha + ro * C::PH) = make_float4(hm.x, hmi.x, hm.y, hmi.y);
          if (NP == 2) {
            const float2 hpi = f2mul(hp, iv[i]);
            *reinterpret_cast<float4*>(Ha + C::WY * C::PH + ro * C::PH) = make_float4(hp.x, hpi.x, hp.y, hpi.y);
          }
        }
      }
    }
    __syncthreads();
    // raw tiles consumed: fetch the next plane while the passes run
    if (tid == 0 && z + 1 < z_last) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(z + 1);
    }

    // ---- Phase B: y pass on the WX window columns (the first pass carries the
    // x halo: WX/TX < WY/TY).  BY outputs down a column, lanes walk x.
#pragma unroll
    for (int i = 0; i < C::YITS; ++i) {
      if (i < C::YITS - 1 || y_last) {
        const float2* src = Hs + ysrc[i];
        float2 v[C::BYS + 2 * R];
#pragma unroll
        for (int k = 0; k < C::BYS + 2 * R; ++k) v[k] = src[k * C::PH];
        float2* dst = Ys + ydst[i];
#pragma unroll
        for (int b = 0; b < C::BYS; ++b) {
          float2 acc = fmul2(taps.w[0], v[b]);
#pragma unroll
          for (int j = 1; j <= 2 * R; ++j) acc = ffma2(taps.w[j], v[b + j], acc);
          if (b >= yskip[i]) dst[b * C::PY] = acc;
        }
      }
    }
    __syncthreads();

    // ---- Phase C: x pass, BX consecutive outputs per item; lanes walk rows of
    // the odd-pitched Ys.  Outputs to the staging tile Os.
#pragma unroll
    for (int i = 0; i < C::XIT; ++i) {
      if (i < C::XIT - 1 || x_last) {
        const float2* src = Ys + xsrc[i];
        float2 v[C::BX + 2 * R];
#pragma unroll
        for (int k = 0; k < C::BX + 2 * R; ++k) v[k] = src[k];
        float2 o[C::BX];
#pragma unroll
        for (int b = 0; b < C::BX; ++b) {
          float2 acc = fmul2(taps.w[0], v[b]);
#pragma unroll
          for (int j = 1; j <= 2 * R; ++j) acc = ffma2(taps.w[j], v[b + j], acc);
          o[b] = acc;
        }
        float4* dst = reinterpret_cast<float4*>(Os + xdst[i]);
#pragma unroll
        for (int b = 0; b < C::BX / 2; ++b) dst[b] = make_float4(o[2 * b].x, o[2 * b].y, o[2 * b + 1].x, o[2 * b + 1].y);
      }
    }
    __syncthreads();

    // ---- Phase D: coalesced 16-byte stores of P (two voxels per store)
    {
      float2* Pz0 = P0 + (size_t)(z - g.zb) * (size_t)g.plane;
      float2* Pz1 = NP == 2 ? P1 + (size_t)(z - g.zb) * (size_t)g.plane : nullptr;
#pragma unroll
      for (int i = 0; i < C::OIT; ++i) {
        if (o_ok[i]) {
          const float4 v = *reinterpret_cast<const float4*>(Os + osrc[i]);
          float2* Pz = (NP == 2 && o_np[i]) ? Pz1 : Pz0;
          *reinterpret_cast<float4*>(Pz + odst[i]) = v;
        }
      }
    }
    if (C::kOsAlias) __syncthreads();  // Os == Hs: copy-out done before phase A
    // Next plane: phase A rewrites Hs (last read in phase B, two barriers
    // ago), phase B rewrites Ys (last read in phase C, before the barrier
    // above) after phase A's barrier, and phase C rewrites Os only after
    // phase B's barrier, which every thread reaches after its phase D.
  }
}

// Stored-Heaviside variant (fields=2, sigma2 = 0): kernel 2 of the previous
// step wrote (H-, H- I) of phi, so the tile arrives ready for the y pass --
// no Heaviside phase and no halo recomputation.  Two tile buffers: plane z+1
// is requested as soon as plane z's wait returns (its buffer held plane z-1,
// whose y pass ended two barriers earlier).
template <int R, int TY, bool EDGE>
__device__ __forceinline__ void xy2_cta_hh(const Geom& g, const Taps& taps, float2* __restrict__ P0, int z_first,
                                           int z_last, int x0, int y0, const CUtensorMap* map_hh,
                                           unsigned char* smem) {
  using C = XY2<R, 1, TY>;
  float2* __restrict__ Ys = reinterpret_cast<float2*>(smem + C::kHHBufs * C::kTileHH);                 // [TY][PY]
  float2* __restrict__ Os = reinterpret_cast<float2*>(smem + C::kHHBufs * C::kTileHH + C::kYsBytes);  // [TY][PO]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kSmemHH - 16);
  const int tid = threadIdx.x;
  const int bx0 = x0 - R - C::SHIFT, by0 = y0 - R;

  int ysrc[C::YITH], ydst[C::YITH], yskip[C::YITH];
#pragma unroll
  for (int i = 0; i < C::YITH; ++i) {
    const int it = min(tid + i * C::NT, C::WX * C::NSEGH - 1);
    const int sy = it / C::WX, cx = it - sy * C::WX;
    const int r0 = sy < C::NSEGH - 1 ? sy * C::BYH : TY - C::BYH;
    ysrc[i] = r0 * C::BOXX + C::SHIFT + cx;
    ydst[i] = r0 * C::PY + cx;
    yskip[i] = sy < C::NSEGH - 1 ? 0 : (C::NSEGH - 1) * C::BYH - r0;  // rows the previous segment wrote
  }
  const bool y_last = tid + (C::YITH - 1) * C::NT < C::WX * C::NSEGH;
  int xsrc[C::XIT], xdst[C::XIT];
  constexpr int SEGX = C::TX / C::BX;
#pragma unroll
  for (int i = 0; i < C::XIT; ++i) {
    const int it = min(tid + i * C::NT, TY * SEGX - 1);
    const int sx = it / TY, row = it - sx * TY;
    xsrc[i] = row * C::PY + sx * C::BX;
    xdst[i] = row * C::PO + sx * C::BX;
  }
  const bool x_last = tid + (C::XIT - 1) * C::NT < TY * SEGX;
  int osrc[C::OIT];
  size_t odst[C::OIT];
  bool o_ok[C::OIT];
#pragma unroll
  for (int i = 0; i < C::OIT; ++i) {
    const int it = min(tid + i * C::NT, TY * C::TX / 2 - 1);
    const int row = it / (C::TX / 2), cp = it - row * (C::TX / 2);
    osrc[i] = row * C::PO + 2 * cp;
    const int gx = x0 + 2 * cp, gy = y0 + row;
    o_ok[i] = tid + i * C::NT < TY * C::TX / 2 && (!EDGE || (gx < g.nx && gy < g.ny));
    odst[i] = (size_t)min(gy, g.ny - 1) * g.nx + min(gx, g.nx - 2);
  }

  auto issue = [&](int z, int buf) {
    mbar_expect_tx(bars + buf, (uint32_t)(C::BOXX * C::WY * sizeof(float2)));
    tma_load_3d(smem + buf * C::kTileHH, map_hh, bars + buf, 2 * bx0, by0, z - g.zb);
  };
  if (tid == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    issue(z_first, 0);
  }
  __syncthreads();

#pragma unroll 1
  for (int z = z_first; z < z_last; ++z) {
    const int xb = C::kHHDouble ? (z - z_first) & 1 : 0;
    float2* T = reinterpret_cast<float2*>(smem + xb * C::kTileHH);  // [WY][BOXX] (H-, H- I)
    mbar_wait(bars + xb, (uint32_t)((C::kHHDouble ? (z - z_first) >> 1 : z - z_first) & 1));
    if (C::kHHDouble && tid == 0 && z + 1 < z_last) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(z + 1, xb ^ 1);
    }
    if constexpr (EDGE) {  // clamp-to-edge fix-up of the pairs outside the volume
      const int lo = max(0, -bx0), hi = min(C::BOXX, g.nx - bx0);
      const int nfix = lo + (C::BOXX - hi);
      for (int e = tid; e < C::WY * nfix; e += C::NT) {
        const int ry = e / nfix, k = e - ry * nfix;
        const int cdst = k < lo ? k : hi + (k - lo);
        const int csrc = k < lo ? lo : hi - 1;
        T[ry * C::BOXX + cdst] = T[ry * C::BOXX + csrc];
      }
      __syncthreads();
      const int ylo = max(0, -by0), yhi = min(C::WY, g.ny - by0);
      const int nrow = ylo + (C::WY - yhi);
      for (int e = tid; e < nrow * C::BOXX; e += C::NT) {
        const int k = e / C::BOXX, cx = e - k * C::BOXX;
        const int rdst = k < ylo ? k : yhi + (k - ylo);
        const int rsrc = k < ylo ? ylo : yhi - 1;
        T[rdst * C::BOXX + cx] = T[rsrc * C::BOXX + cx];
      }
      __syncthreads();
    }
    // ---- y pass straight from the tile (lanes walk x: consecutive pairs)
#pragma unroll
    for (int i = 0; i < C::YITH; ++i) {
      if (i < C::YITH - 1 || y_last) {
        const float2* src = T + ysrc[i];
        float2 v[C::BYH + 2 * R];
#pragma unroll
        for (int k = 0; k < C::BYH + 2 * R; ++k) v[k] = src[k * C::BOXX];
        float2* dst = Ys + ydst[i];
#pragma unroll
        for (int b = 0; b < C::BYH; ++b) {
          float2 acc = fmul2(taps.w[0], v[b]);
#pragma unroll
          for (int j = 1; j <= 2 * R; ++j) acc = ffma2(taps.w[j], v[b + j], acc);
          if (b >= yskip[i]) dst[b * C::PY] = acc;
        }
      }
    }
    __syncthreads();
    if (!C::kHHDouble && tid == 0 && z + 1 < z_last) {  // one buffer: the y pass has consumed it
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(z + 1, 0);
    }
    // ---- x pass (lanes walk rows of the odd-pitched Ys) into the staging tile
#pragma unroll
    for (int i = 0; i < C::XIT; ++i) {
      if (i < C::XIT - 1 || x_last) {
        const float2* src = Ys + xsrc[i];
        float2 v[C::BX + 2 * R];
#pragma unroll
        for (int k = 0; k < C::BX + 2 * R; ++k) v[k] = src[k];
        float2 o[C::BX];
#pragma unroll
        for (int b = 0; b < C::BX; ++b) {
          float2 acc = fmul2(taps.w[0], v[b]);
#pragma unroll
          for (int j = 1; j <= 2 * R; ++j) acc = ffma2(taps.w[j], v[b + j], acc);
          o[b] = acc;
        }
        float4* dst = reinterpret_cast<float4*>(Os + xdst[i]);
#pragma unroll
        for (int b = 0; b < C::BX / 2; ++b) dst[b] = make_float4(o[2 * b].x, o[2 * b].y, o[2 * b + 1].x, o[2 * b + 1].y);
      }
    }
    __syncthreads();
    // ---- coalesced 16-byte stores of P
    float2* Pz = P0 + (size_t)(z - g.zb) * (size_t)g.plane;
#pragma unroll
    for (int i = 0; i < C::OIT; ++i)
      if (o_ok[i]) *reinterpret_cast<float4*>(Pz + odst[i]) = *reinterpret_cast<const float4*>(Os + osrc[i]);
    // next plane: the y pass rewrites Ys after this plane's x pass (barrier
    // above); the x pass rewrites Os after the next y-pass barrier, which
    // every thread reaches after this copy-out.
  }
}

template <int R, int TY>
__global__ void __launch_bounds__(XY2<R, 1, TY>::NT, XY2<R, 1, TY>::NT == 256 ? 2 : 1)
    xy2_hh_kernel(Geom g, Taps taps, float2* __restrict__ P0, int z_begin, int z_end,
                  const __grid_constant__ CUtensorMap map_hh) {
  using C = XY2<R, 1, TY>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int x0 = blockIdx.x * C::TX, y0 = blockIdx.y * TY;
  const int z_first = z_begin + blockIdx.z * C::NZC;
  const int z_last = min(z_first + C::NZC, z_end);
  const bool edge = x0 - R < 0 || y0 - R < 0 || x0 - R + C::WX > g.nx || y0 - R + C::WY > g.ny;
  if (edge)
    xy2_cta_hh<R, TY, true>(g, taps, P0, z_first, z_last, x0, y0, &map_hh, smem);
  else
    xy2_cta_hh<R, TY, false>(g, taps, P0, z_first, z_last, x0, y0, &map_hh, smem);
}

template <int R, int NP, int TY>
__global__ void __launch_bounds__(XY2<R, NP, TY>::NT, XY2<R, NP, TY>::NT == 256 ? 2 : 1)
    xy2_kernel(Geom g, Taps taps, float inv_eps, float2* __restrict__ P0, float2* __restrict__ P1, int z_begin,
               int z_end, const __grid_constant__ CUtensorMap map_phi, const __grid_constant__ CUtensorMap map_img) {
  using C = XY2<R, NP, TY>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int x0 = blockIdx.x * C::TX, y0 = blockIdx.y * TY;
  const int z_first = z_begin + blockIdx.z * C::NZC;
  const int z_last = min(z_first + C::NZC, z_end);
  const bool edge = x0 - R < 0 || y0 - R < 0 || x0 - R + C::WX > g.nx || y0 - R + C::WY > g.ny;
  if (edge)
    xy2_cta<R, NP, TY, true>(g, taps, inv_eps, P0, P1, z_first, z_last, x0, y0, &map_phi, &map_img, smem);
  else
    xy2_cta<R, NP, TY, false>(g, taps, inv_eps, P0, P1, z_first, z_last, x0, y0, &map_phi, &map_img, smem);
}

template <int R, int TY>
int xy2_hh_launch(const Geom& g, const Taps& t, float2* P0, int z_begin, int z_end, const XYMaps& m,
                  cudaStream_t st) {
  using C = XY2<R, 1, TY>;
  static_assert(C::kSmemHH <= 227 * 1024, "stored-Heaviside tile exceeds shared memory");
  auto k = xy2_hh_kernel<R, TY>;
  if (!smem_optin<xy2_hh_kernel<R, TY>>((int)C::kSmemHH)) return -1;
  if (z_end <= z_begin) return 0;
  dim3 grid((g.nx + C::TX - 1) / C::TX, (g.ny + TY - 1) / TY, (z_end - z_begin + C::NZC - 1) / C::NZC);
  k<<<grid, C::NT, C::kSmemHH, st>>>(g, t, P0, z_begin, z_end, m.hh);
  return 1;
}

template <int R, int NP, int TY>
int xy2_launch(const Geom& g, const Taps& t, float inv_eps, float2* P0, float2* P1, int z_begin, int z_end,
               const XYMaps& m, cudaStream_t st) {
  // the stored-Heaviside variant exists where the mode is used (R <= kHHMaxR,
  // 64 x 32 tiles; rsfg_api.cu make_xy2_maps)
  if constexpr (NP == 1 && R <= kHHMaxR && TY == 32) {
    if (m.use_hh) return xy2_hh_launch<R, TY>(g, t, P0, z_begin, z_end, m, st);
  }
  if (m.use_hh && NP == 1) return -1;
  using C = XY2<R, NP, TY>;
  // variants that cannot fit shared memory (or that setup never selects:
  // 64-row tiles past R = 18) are not instantiated
  if constexpr (C::kSmem > 227 * 1024 || (TY == 64 && R > 18)) {
    return -1;
  } else {
    auto k = xy2_kernel<R, NP, TY>;
    if (!smem_optin<xy2_kernel<R, NP, TY>>((int)C::kSmem)) return -1;
    if (z_end <= z_begin) return 0;
    dim3 grid((g.nx + C::TX - 1) / C::TX, (g.ny + TY - 1) / TY, (z_end - z_begin + C::NZC - 1) / C::NZC);
    k<<<grid, C::NT, C::kSmem, st>>>(g, t, inv_eps, P0, P1, z_begin, z_end, m.phi, m.img);
    return 1;
  }
}

}  // namespace

// kernel 1 tile height used by xy2 (RSFG_XY2_TY overrides: 32 or 64)
constexpr int kXY2DefaultTY = 32;

#define RSFG_XY2_GROUPS(X) X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11)
#define RSFG_XY2_DECL(N)                                                                                  \
  int xy2_group_##N(int r, int ty, const Geom& g, int fields, const Taps& t1, float inv_eps, float2* P0,   \
                    float2* P1, int z_begin, int z_end, const XYMaps& m, cudaStream_t st);                 \
  int xy2_group_box_##N(int r, int ty, int* bx, int* by);
RSFG_XY2_GROUPS(RSFG_XY2_DECL)
#undef RSFG_XY2_DECL

// Body of one radius-group translation unit (rsfg_xy2_g*.cu): the TMA box and
// the launch of every radius in RADII (64 x 64 tiles: fields=2 only, the
// fields=4 tile exceeds shared memory).
#define RSFG_XY2_BOX_CASE(R)                                       \
  case R:                                                          \
    *bx = ty == 64 ? XY2<R, 1, 64>::BOXX : XY2<R, 1, 32>::BOXX;    \
    *by = ty == 64 ? XY2<R, 1, 64>::WY : XY2<R, 1, 32>::WY;        \
    return 1;
#define RSFG_XY2_LAUNCH_CASE(R)                                                                       \
  case R:                                                                                             \
    if (ty == 64) return fields == 4 ? -1 : xy2_launch<R, 1, 64>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st); \
    return fields == 4 ? xy2_launch<R, 2, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st)                  \
                       : xy2_launch<R, 1, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
#define RSFG_XY2_GROUP(N, RADII)                                                                              \
  int xy2_group_box_##N(int r, int ty, int* bx, int* by) {                                                  \
    switch (r) {                                                                                            \
      RADII(RSFG_XY2_BOX_CASE)                                                                              \
      default:                                                                                              \
        return -2;                                                                                          \
    }                                                                                                       \
  }                                                                                                         \
  int xy2_group_##N(int r, int ty, const Geom& g, int fields, const Taps& t1, float inv_eps, float2* P0,     \
                    float2* P1, int z_begin, int z_end, const XYMaps& m, cudaStream_t st) {                 \
    switch (r) {                                                                                            \
      RADII(RSFG_XY2_LAUNCH_CASE)                                                                           \
      default:                                                                                              \
        return -2;                                                                                          \
    }                                                                                                       \
  }

}  // namespace rsfg
