// rsfg_xy.cu -- kernel 1 of the RSF step (see rsfg_zst.cu for kernel 2):
// Heaviside fields on a haloed z-plane tile, then the x and y passes of the
// separable Gaussian (reference rsf.cpp:75-94, ops.cpp:74-160).
//
// The (TX+2R) x (TY+2R) phi and I tiles arrive by TMA (cp.async.bulk.tensor,
// one thread, mbarrier completion; edge tiles read their clamp-to-edge
// neighbours from inside the box) when the row
// pitch allows it (nx % 4 == 0), else by batched LDG.
#include "rsfg_device.cuh"

namespace rsfg {
namespace {

// NP = number of float2 field pairs (1: fields=2, 2: fields=4).
template <int R, int NP, int TX, int TY, int BX, int BY>
struct XYCfg {
  static constexpr int WX = TX + 2 * R;
  static constexpr int WY = TY + 2 * R;
  // TMA box row: starts on a 16-byte boundary (x origin rounded down to a
  // multiple of 4 floats) and spans a multiple of 16 bytes.
  static constexpr int BOXX = (WX + 3 + 3) & ~3;
  static constexpr int PX = WX | 1;  // odd pitch (float2): conflict-free row-strided LDS.64
  static constexpr int QX = TX | 1;
  static constexpr size_t kHsBytes = ((size_t)NP * WY * PX * sizeof(float2) + 127) & ~(size_t)127;
  static constexpr size_t kXsBytes = (size_t)NP * WY * QX * sizeof(float2);
  static constexpr size_t kTileBytes = ((size_t)BOXX * WY * sizeof(float) + 127) & ~(size_t)127;
  static constexpr size_t kRawBytes = 2 * kTileBytes;  // phi + I tiles (TMA dst: 128-byte aligned)
  static constexpr size_t kUnion = kXsBytes > kRawBytes ? kXsBytes : kRawBytes;
  static constexpr size_t kSmem = kHsBytes + kUnion + 16;  // + mbarrier
  static constexpr int kThreads = 256;
  static constexpr int kItems = (WX * WY + kThreads - 1) / kThreads;  // halo elements per thread
};

template <int R, int NP, int TX, int TY, int BX, int BY, bool TMA>
__global__ void __launch_bounds__(256) xy_kernel(Geom g, Taps taps, float inv_eps,
                                                 const float* __restrict__ phi,
                                                 const float* __restrict__ image,
                                                 float2* __restrict__ P0, float2* __restrict__ P1, int z_begin,
                                                 const __grid_constant__ CUtensorMap map_phi,
                                                 const __grid_constant__ CUtensorMap map_img) {
  using C = XYCfg<R, NP, TX, TY, BX, BY>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float2* Hs = reinterpret_cast<float2*>(smem_raw);                 // [NP][WY][PX]
  float2* Xs = reinterpret_cast<float2*>(smem_raw + C::kHsBytes);   // [NP][WY][QX]
  float* Tphi = reinterpret_cast<float*>(smem_raw + C::kHsBytes);   // [WY][BOXX] (aliases Xs)
  float* Timg = reinterpret_cast<float*>(smem_raw + C::kHsBytes + C::kTileBytes);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + C::kHsBytes + C::kUnion);
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY, z = z_begin + blockIdx.z;

  // Phase A: the haloed tile, then the Heaviside fields once per loaded voxel.
  if constexpr (TMA) {
    // The box starts at max(origin, 0) rounded down to 16 bytes (TMA faults on
    // negative or unaligned x starts here); positive out-of-range elements are
    // zero-filled and never read: edge tiles read their clamped neighbour.
    const int bx0 = max(x0 - R, 0) & ~3, by0 = max(y0 - R, 0);
    if (threadIdx.x == 0) {
      mbar_init(bar, 1);
      mbar_expect_tx(bar, (uint32_t)(2 * C::BOXX * C::WY * sizeof(float)));
      tma_load_3d(Tphi, &map_phi, bar, bx0, by0, z - g.zb);
      tma_load_3d(Timg, &map_img, bar, bx0, by0, z - g.zb);
    }
    __syncthreads();  // barrier initialised before anyone waits on it
    mbar_wait(bar, 0);
    const bool edge = x0 - R < 0 || y0 - R < 0 || x0 - R + C::WX > g.nx || y0 - R + C::WY > g.ny;
    const int shift = (x0 - R) - bx0;  // 0..3 on interior tiles
#pragma unroll 4
    for (int e = threadIdx.x; e < C::WX * C::WY; e += C::kThreads) {
      const int ey = e / C::WX, ex = e - ey * C::WX;
      int src = ey * C::BOXX + ex + shift;
      if (edge) {  // clamp-to-edge in global coordinates, then into the box
        const int cx = clampi(x0 - R + ex, 0, g.nx - 1) - bx0;
        const int cy = clampi(y0 - R + ey, 0, g.ny - 1) - by0;
        src = cy * C::BOXX + cx;
      }
      const float p = Tphi[src], im = Timg[src];
      float hm, hp;
      heaviside_pair(p, inv_eps, hm, hp);
      Hs[ey * C::PX + ex] = make_float2(hm, hm * im);
      if (NP == 2) Hs[C::WY * C::PX + ey * C::PX + ex] = make_float2(hp, hp * im);
    }
  } else {
    const float* phi_p = phi + (size_t)(z - g.zb) * (size_t)g.plane;
    const float* img_p = image + (size_t)(z - g.zb) * (size_t)g.plane;
    float pv[C::kItems], iv[C::kItems];
    int so[C::kItems];
#pragma unroll
    for (int k = 0; k < C::kItems; ++k) {  // all loads first (ILP), then compute
      const int e = threadIdx.x + k * C::kThreads;
      so[k] = -1;
      if (e < C::WX * C::WY) {
        const int ey = e / C::WX, ex = e - ey * C::WX;
        const int gx = clampi(x0 - R + ex, 0, g.nx - 1), gy = clampi(y0 - R + ey, 0, g.ny - 1);
        const int i = gy * g.nx + gx;
        pv[k] = __ldg(phi_p + i);
        iv[k] = __ldg(img_p + i);
        so[k] = ey * C::PX + ex;
      }
    }
#pragma unroll
    for (int k = 0; k < C::kItems; ++k) {
      if (so[k] >= 0) {
        float hm, hp;
        heaviside_pair(pv[k], inv_eps, hm, hp);
        Hs[so[k]] = make_float2(hm, hm * iv[k]);
        if (NP == 2) Hs[C::WY * C::PX + so[k]] = make_float2(hp, hp * iv[k]);
      }
    }
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
    float2* P = (np ? P1 : P0) + (size_t)(z - g.zb) * (size_t)g.plane;
#pragma unroll
    for (int b = 0; b < BY; ++b) {
      float2 acc = fmul2(taps.w[0], v[b]);
#pragma unroll
      for (int j = 1; j <= 2 * R; ++j) acc = ffma2(taps.w[j], v[b + j], acc);
      const int gy = y0 + sy * BY + b;
      if (gx < g.nx && gy < g.ny) P[gy * g.nx + gx] = acc;
    }
  }
}

constexpr int kXYTX = 64, kXYTY = 32, kBX = 8, kBY = 8;

template <int R, int NP, bool TMA>
int xy_launch(const Geom& g, const Taps& t, float inv_eps, const float* phi, const float* image, float2* P0,
              float2* P1, int z_begin, int z_end, const XYMaps* maps, cudaStream_t st) {
  using C = XYCfg<R, NP, kXYTX, kXYTY, kBX, kBY>;
  if constexpr (C::kSmem > 227 * 1024) {
    return -1;  // setup routes such (radius, fields) to the generic path (xy_fits)
  } else {
  auto k = xy_kernel<R, NP, kXYTX, kXYTY, kBX, kBY, TMA>;
  smem_optin<xy_kernel<R, NP, kXYTX, kXYTY, kBX, kBY, TMA>>((int)C::kSmem);
  if (z_end <= z_begin) return 0;
  static const CUtensorMap kNoMap{};
  const CUtensorMap& mp = TMA ? maps->phi : kNoMap;
  const CUtensorMap& mi = TMA ? maps->img : kNoMap;
  dim3 grid((g.nx + kXYTX - 1) / kXYTX, (g.ny + kXYTY - 1) / kXYTY, z_end - z_begin);
  k<<<grid, C::kThreads, C::kSmem, st>>>(g, t, inv_eps, phi, image, P0, P1, z_begin, mp, mi);
  return 1;
  }
}

template <int R, int NP>
int xy_dispatch(const Geom& g, const Taps& t, float inv_eps, const float* phi, const float* image, float2* P0,
                float2* P1, int z_begin, int z_end, const XYMaps* maps, cudaStream_t st) {
  if (maps && maps->valid)
    return xy_launch<R, NP, true>(g, t, inv_eps, phi, image, P0, P1, z_begin, z_end, maps, st);
  return xy_launch<R, NP, false>(g, t, inv_eps, phi, image, P0, P1, z_begin, z_end, maps, st);
}

}  // namespace

bool xy_fits(int r, int fields) {
  switch (r) {
#define CASE(R)                                                                                        \
  case R:                                                                                              \
    return (fields == 4 ? XYCfg<R, 2, kXYTX, kXYTY, kBX, kBY>::kSmem : XYCfg<R, 1, kXYTX, kXYTY, kBX, kBY>::kSmem) <= \
           227 * 1024;
    RSFG_RADII(CASE)
#undef CASE
    default:
      return false;
  }
}

bool xy_tma_box(int r, int* bx, int* by) {
  switch (r) {
#define CASE(R)                                                 \
  case R:                                                       \
    *bx = XYCfg<R, 1, kXYTX, kXYTY, kBX, kBY>::BOXX;            \
    *by = XYCfg<R, 1, kXYTX, kXYTY, kBX, kBY>::WY;              \
    return true;
    RSFG_RADII(CASE)
#undef CASE
    default:
      return false;
  }
}

int launch_xy(const Geom& g, int fields, const Taps& t1, float inv_eps, const float* phi, const float* image,
              float2* P0, float2* P1, int z_begin, int z_end, const XYMaps* maps, cudaStream_t st) {
  switch (t1.r) {
#define CASE(R)                                                                                          \
  case R:                                                                                                \
    return fields == 4 ? xy_dispatch<R, 2>(g, t1, inv_eps, phi, image, P0, P1, z_begin, z_end, maps, st) \
                       : xy_dispatch<R, 1>(g, t1, inv_eps, phi, image, P0, P1, z_begin, z_end, maps, st);
    RSFG_RADII(CASE)
#undef CASE
    default:
      return -1;
  }
}

}  // namespace rsfg
