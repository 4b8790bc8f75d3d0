// rsfg_zst.cu -- kernel 2 of the RSF step: z pass, region averages and
// force, curvature / Laplacian stencil, combine and explicit update
// (reference rsf.cpp:96-168, 324-352; ops.cpp:109-160, 199-316).
#include "rsfg_device.cuh"

namespace rsfg {
namespace {

// ---------------------------------------------------------------- kernel 2
// One CTA = TX x TY columns x (TZC * NCH) planes, streamed in z.  Shared
// memory holds a 7-plane ring of phi (halo 2 in x/y), a 4-plane ring of the
// normalized gradient (halo 1) and the z-pass results of one TZC chunk.  The
// ring depths let one barrier per plane order every ring access.
template <int R, int NP, int TX, int TY, int TZC, int NCH>
struct ZCfg {
  static constexpr int FX = TX + 4, FY = TY + 4, FPL = FX * FY;  // phi plane with halo 2
  static constexpr int NXr = TX + 2, NYr = TY + 2, NPL = NXr * NYr;  // normal plane, halo 1
  static constexpr int kThreads = TX * TY;
  static constexpr int kHalo = NPL - TX * TY;  // normal-plane halo positions
  static constexpr int kPhiPer = (FPL + kThreads - 1) / kThreads;
  static constexpr int TZ = TZC * NCH;
  static constexpr size_t kSmem =
      (size_t)(7 * FPL + 4 * 3 * NPL) * sizeof(float) + (size_t)NP * TZC * TX * TY * sizeof(float2);
};

template <int R, int NP, int TX, int TY, int TZC, int NCH>
__global__ void __launch_bounds__(TX* TY, 2)
    zst_kernel(Geom g, Taps taps, StepConsts c, StepBuffers b, int z_begin, int z_end, int mode) {
  using C = ZCfg<R, NP, TX, TY, TZC, NCH>;
  extern __shared__ float smemf[];
  float* Phi = smemf;                   // [7][FY][FX] ring, slot = (q - (z0-2)) % 7
  float* Nr = Phi + 7 * C::FPL;         // [4 slots][3 comps][NYr][NXr]
  float2* KH = reinterpret_cast<float2*>(Nr + 12 * C::NPL);  // [NP][TZC][TY*TX]
  __shared__ unsigned int s_count;

  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  const int z0 = z_begin + blockIdx.x * C::TZ;  // z tile fastest: neighbours share P halos in L2
  const int x0 = blockIdx.y * TX, y0 = blockIdx.z * TY;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long plane = g.plane;
  if (tid == 0) s_count = 0;

  // ---- per-thread constants
  // phi-plane load slots: element e = tid + k*threads of the FX x FY window
  int phi_g[C::kPhiPer], phi_s[C::kPhiPer];
#pragma unroll
  for (int k = 0; k < C::kPhiPer; ++k) {
    const int e = tid + k * C::kThreads;
    phi_s[k] = e < C::FPL ? e : -1;
    const int ex = e % C::FX, ey = e / C::FX;
    phi_g[k] = clampi(y0 - 2 + ey, 0, ny - 1) * nx + clampi(x0 - 2 + ex, 0, nx - 1);
  }
  auto plane_ptr = [&](int q) { return b.phi + (size_t)(clampi(q, g.zb, g.ze - 1) - g.zb) * (size_t)plane; };
  // ring slot of global plane q (used outside the steady-state loop only)
  auto slot_of = [&](int q) { return ((q - (z0 - 2)) % 7) * C::FPL; };

  // normal positions: own column (i = tx+1, j = ty+1) and, for tid < kHalo,
  // one halo position of the (TX+2) x (TY+2) ring.
  struct NPos {
    int s, sxm, sxp, sym, syp, n;  // phi offsets (in-plane) and normal-plane offset
    float invx, invy;
  };
  auto make_pos = [&](int i, int j) {
    NPos p;
    const int gx = clampi(x0 - 1 + i, 0, nx - 1), gy = clampi(y0 - 1 + j, 0, ny - 1);
    const int xm = max(gx - 1, 0), xp = min(gx + 1, nx - 1), ym = max(gy - 1, 0), yp = min(gy + 1, ny - 1);
    const int cx = gx - (x0 - 2), cy = gy - (y0 - 2);
    p.s = cy * C::FX + cx;
    p.sxm = cy * C::FX + (xm - (x0 - 2));
    p.sxp = cy * C::FX + (xp - (x0 - 2));
    p.sym = (ym - (y0 - 2)) * C::FX + cx;
    p.syp = (yp - (y0 - 2)) * C::FX + cx;
    p.invx = (xp - xm) == 2 ? 0.5f : 1.0f;
    p.invy = (yp - ym) == 2 ? 0.5f : 1.0f;
    p.n = j * C::NXr + i;
    return p;
  };
  const NPos own = make_pos(tx + 1, ty + 1);
  NPos hal = own;
  const bool has_halo = tid < C::kHalo;
  if (has_halo) {
    int i, j;
    if (tid < C::NXr) {
      i = tid, j = 0;
    } else if (tid < 2 * C::NXr) {
      i = tid - C::NXr, j = C::NYr - 1;
    } else {
      const int k = tid - 2 * C::NXr;  // 2 * TY side positions
      i = (k & 1) ? C::NXr - 1 : 0;
      j = 1 + (k >> 1);
    }
    hal = make_pos(i, j);
  }
  // n = grad phi / max(|grad phi|, floor) at p from phi planes (zm, gz, zp)
  // given as ring offsets (rsf.cpp:110-123; ops.cpp:199-232 face rule).
  auto normal_at = [&](const NPos& p, int om, int o0, int op, float invz, float* dst) {
    const float a = (Phi[o0 + p.sxp] - Phi[o0 + p.sxm]) * p.invx;
    const float bb = (Phi[o0 + p.syp] - Phi[o0 + p.sym]) * p.invy;
    const float cc = (Phi[op + p.s] - Phi[om + p.s]) * invz;
    const float inv = fminf(rsqrt_approx(fmaf(a, a, fmaf(bb, bb, cc * cc))), c.inv_grad_floor);
    dst[p.n] = a * inv;
    dst[C::NPL + p.n] = bb * inv;
    dst[2 * C::NPL + p.n] = cc * inv;
  };
  auto normal_plane = [&](float* dst, int om, int o0, int op, float invz) {
    normal_at(own, om, o0, op, invz, dst);
    if (has_halo) normal_at(hal, om, o0, op, invz, dst);
  };
  auto normal_plane_slow = [&](float* dst, int zz) {
    const int gz = clampi(zz, 0, nz - 1);
    const int zm = max(gz - 1, 0), zp = min(gz + 1, nz - 1);
    normal_plane(dst, slot_of(zm), slot_of(gz), slot_of(zp), (zp - zm) == 2 ? 0.5f : 1.0f);
  };

  // output-voxel constants
  const int x = x0 + tx, y = y0 + ty;
  const bool col_ok = x < nx && y < ny;
  const int xm = max(x - 1, 0), xp = min(x + 1, nx - 1), ym = max(y - 1, 0), yp = min(y + 1, ny - 1);
  const float invx = (xp - xm) == 2 ? 0.5f : 1.0f;
  const float invy = (yp - ym) == 2 ? 0.5f : 1.0f;
  const int n_c = (ty + 1) * C::NXr + (tx + 1);
  const int n_xm = (ty + 1) * C::NXr + (xm - (x0 - 1)), n_xp = (ty + 1) * C::NXr + (xp - (x0 - 1));
  const int n_ym = (ym - (y0 - 1)) * C::NXr + (tx + 1), n_yp = (yp - (y0 - 1)) * C::NXr + (tx + 1);
  const int s_c = (ty + 2) * C::FX + (tx + 2);
  const int col = min(y, ny - 1) * nx + min(x, nx - 1);
  unsigned int my_count = 0;

  // ---- prologue: phi planes z0-2 .. z0+4 into ring slots 0..6
#pragma unroll 1
  for (int q = z0 - 2; q <= z0 + 4; ++q) {
    const float* src = plane_ptr(q);
    float* dst = Phi + slot_of(q);
#pragma unroll
    for (int k = 0; k < C::kPhiPer; ++k)
      if (phi_s[k] >= 0) dst[phi_s[k]] = __ldg(src + phi_g[k]);
  }
  // Rotating ring offsets, phi planes zo-2 .. zo+4 and normal planes
  // zo-2 / zo-1 / zo / free.  Per step: write normal plane zo+1 into the free
  // slot (read by nobody still in step zo-1), barrier, read, refill phi
  // plane zo+5 into zo-2's slot (no longer read by anyone past the barrier;
  // first read three steps later).
  int o_m2 = 0, o_m1 = C::FPL, o_0 = 2 * C::FPL, o_p1 = 3 * C::FPL, o_p2 = 4 * C::FPL, o_p3 = 5 * C::FPL,
      o_p4 = 6 * C::FPL;
  int n_m2 = 9 * C::NPL, n_m = 0, n_0 = 3 * C::NPL, n_f = 6 * C::NPL;
  // phi refill sources: plane zo+5 of this thread's load slots, advanced per step
  const float* pf[C::kPhiPer];
#pragma unroll
  for (int k = 0; k < C::kPhiPer; ++k) pf[k] = plane_ptr(z0 + 5) + phi_g[k];
  __syncthreads();
  normal_plane_slow(Nr + n_m, z0 - 1);
  normal_plane_slow(Nr + n_0, z0);

  const int z_stop = min(z0 + C::TZ, z_end);
  // static fields of the first output plane (then prefetched one plane ahead)
  size_t vi = (size_t)(z0 - g.zb) * (size_t)plane + col;
  float ki_n = __ldg(b.ki + vi);
  float k1i_n = NP == 1 ? __ldg(b.k1i + vi) : 0.0f;
#pragma unroll 1
  for (int zc = z0; zc < z_stop; zc += TZC) {
    // ---- z pass of one chunk: TZC outputs per column from a (TZC + 2R)
    // register window; fp32 FMA per tap in ascending order, like the
    // reference's f32-rounded z pass (ops.cpp:150-155).
    __syncthreads();  // previous chunk's KH reads are done
    {
      const int gx = min(x, nx - 1), gy = min(y, ny - 1);
      const bool interior = zc - R >= g.zb && zc + TZC + R <= g.ze;
#pragma unroll
      for (int np = 0; np < NP; ++np) {
        const float2* P = b.P[np] + (size_t)gy * nx + gx;
        float2 pv[TZC + 2 * R];
        if (interior) {
          const float2* Pz = P + (size_t)(zc - R - g.zb) * (size_t)plane;
#pragma unroll
          for (int k = 0; k < TZC + 2 * R; ++k) pv[k] = __ldg(Pz + (size_t)k * (size_t)plane);
        } else {
#pragma unroll
          for (int k = 0; k < TZC + 2 * R; ++k)
            pv[k] = __ldg(P + (size_t)(clampi(zc - R + k, g.zb, g.ze - 1) - g.zb) * (size_t)plane);
        }
#pragma unroll
        for (int t = 0; t < TZC; ++t) {
          float2 acc = fmul2(taps.w[0], pv[t]);
#pragma unroll
          for (int j = 1; j <= 2 * R; ++j) acc = ffma2(taps.w[j], pv[t + j], acc);
          KH[(np * TZC + t) * C::kThreads + tid] = acc;
        }
      }
    }
    __syncthreads();

    const int tend = min(TZC, z_stop - zc);
#pragma unroll 1
    for (int t = 0; t < tend; ++t) {
      const int zo = zc + t;
      // prefetch: phi plane zo+5 (ring refill) and the static fields at zo+1
      float nxt[C::kPhiPer];
#pragma unroll
      for (int k = 0; k < C::kPhiPer; ++k) nxt[k] = phi_s[k] >= 0 ? __ldg(pf[k]) : 0.0f;
      if (zo + 6 <= g.ze - 1) {  // clamped at the last held plane
#pragma unroll
        for (int k = 0; k < C::kPhiPer; ++k) pf[k] += plane;
      }
      const float ki = ki_n, k1i = k1i_n;
      const size_t vo = vi;
      vi += (size_t)plane;
      if (zo + 1 < z_stop) {
        ki_n = __ldg(b.ki + vi);
        if (NP == 1) k1i_n = __ldg(b.k1i + vi);
      }

      // normal plane zo+1 from phi planes (zo, zo+1, zo+2), face rule at z = nz-1
      if (zo + 2 <= nz - 1)
        normal_plane(Nr + n_f, o_0, o_p1, o_p2, 0.5f);
      else if (zo + 1 == nz - 1)
        normal_plane(Nr + n_f, o_0, o_p1, o_p1, 1.0f);
      else
        normal_plane(Nr + n_f, o_m1, o_0, o_0, 1.0f);
      __syncthreads();

      {
        const int zmm = max(zo - 1, 0), zpp = min(zo + 1, nz - 1);
        const float invz = (zpp - zmm) == 2 ? 0.5f : 1.0f;
        // curvature kappa = div n (ops.cpp:281-316), same face rule
        const float* N0 = Nr + n_0;
        const float kappa = (N0[n_xp] - N0[n_xm]) * invx + (N0[C::NPL + n_yp] - N0[C::NPL + n_ym]) * invy +
                            (Nr[n_f + 2 * C::NPL + n_c] - Nr[n_m + 2 * C::NPL + n_c]) * invz;
        // 7-point Laplacian, clamp-to-edge (ops.cpp:258-271)
        const float* pc = Phi + o_0 + s_c;
        const float cphi = pc[0];
        const float pzm = Phi[o_m1 + s_c], pzp = Phi[o_p1 + s_c];
        const float lap = fmaf(-2.0f, cphi, pc[-1] + pc[1]) + fmaf(-2.0f, cphi, pc[-C::FX] + pc[C::FX]) +
                          fmaf(-2.0f, cphi, pzm + pzp);
        // delta_eps (rsf.cpp:96-107)
        const float delta = c.c_delta * rcp_approx(fmaf(cphi, cphi, c.eps2));
        // region averages r+- and F- - F+ (rsf.cpp:130-148, 164)
        const float2 h0 = KH[t * C::kThreads + tid];
        const float km = h0.x, kmi = h0.y;
        float kp, kpi;
        if (NP == 2) {
          const float2 h1 = KH[(TZC + t) * C::kThreads + tid];
          kp = h1.x;
          kpi = h1.y;
        } else {
          kp = 1.0f - km;
          kpi = k1i - kmi;
        }
        const float rp = fminf(fmaxf(__fdividef(kpi, fmaxf(kp, c.denom_floor)), c.i_min), c.i_max);
        const float rm = fminf(fmaxf(__fdividef(kmi, fmaxf(km, c.denom_floor)), c.i_min), c.i_max);
        // (KI2 - 2 r- KI + r-^2) - (KI2 - 2 r+ KI + r+^2) == (r+ - r-)(2 KI - r+ - r-)
        const float dF = (rp - rm) * (fmaf(2.0f, ki, -rp) - rm);
        // combine (rsf.cpp:151-168) and explicit update (rsf.cpp:340-344)
        const float e = (lap - kappa) + delta * fmaf(c.alpha, kappa, c.beta * dF);
        if (col_ok && zo < z_end) {
          if (mode == kUpdate) {
            const float f = fmaf(c.dt_f, e, cphi);
            b.out[vo] = f;
            my_count += ((cphi < 0.0f) != (f < 0.0f)) ? 1u : 0u;
            if (!isfinite(f)) atomicMin(b.counters + 1, (unsigned long long)zo * (unsigned long long)plane + col);
          } else {
            b.out[vo] = e;
          }
        }
      }
      {
        float* dst = Phi + o_m2;  // plane zo-2: no thread past this step's barrier reads it
#pragma unroll
        for (int k = 0; k < C::kPhiPer; ++k)
          if (phi_s[k] >= 0) dst[phi_s[k]] = nxt[k];
      }
      const int ot = o_m2;
      o_m2 = o_m1;
      o_m1 = o_0;
      o_0 = o_p1;
      o_p1 = o_p2;
      o_p2 = o_p3;
      o_p3 = o_p4;
      o_p4 = ot;
      const int nt = n_m2;
      n_m2 = n_m;
      n_m = n_0;
      n_0 = n_f;
      n_f = nt;
    }
  }

  if (mode == kUpdate) {
    const unsigned int wsum = __reduce_add_sync(0xffffffffu, my_count);
    if ((tid & 31) == 0 && wsum) atomicAdd(&s_count, wsum);
    __syncthreads();
    if (tid == 0 && s_count) atomicAdd(b.counters, (unsigned long long)s_count);
  }
}

// ------------------------------------------------------------ dispatchers
constexpr int kZTX = 32, kZTY = 8, kZTZC = 16, kZNCH = 4;

template <int R, int NP>
int zst_launch(const Geom& g, const Taps& t, const StepConsts& c, const StepBuffers& b, int z_begin,
               int z_end, int mode, cudaStream_t st) {
  // z-pass register window = TZC + 2R float2: halve the chunk for large radii
  constexpr int TZC = R > 18 ? kZTZC / 4 : (R > 12 ? kZTZC / 2 : kZTZC);
  constexpr int NCH = kZTZC * kZNCH / TZC;
  using C = ZCfg<R, NP, kZTX, kZTY, TZC, NCH>;
  auto k = zst_kernel<R, NP, kZTX, kZTY, TZC, NCH>;
  smem_optin<zst_kernel<R, NP, kZTX, kZTY, TZC, NCH>>((int)C::kSmem);
  if (z_end <= z_begin) return 0;
  dim3 grid((z_end - z_begin + C::TZ - 1) / C::TZ, (g.nx + kZTX - 1) / kZTX, (g.ny + kZTY - 1) / kZTY);
  k<<<grid, kZTX * kZTY, C::kSmem, st>>>(g, t, c, b, z_begin, z_end, mode);
  return 1;
}

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

}  // namespace rsfg
