// rsfg_kernels.cu -- support kernels: the generic-radius separable passes,
// static-field convolutions (init), min/max, mask.  The two hot kernels are
// xy2 (rsfg_xy2.cuh) and zst4 (rsfg_zst4.cuh); rsfg_xy.cu / rsfg_zst.cu hold
// their LDG-staged fallbacks.
#include <cstring>

#include "rsfg_device.cuh"

namespace rsfg {
namespace {

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
    if (pos - r >= max(lo, 0) && pos + r <= min(hi, n_ax - 1)) {
      // whole window inside: one base pointer, constant stride, no clamps
      const long long stride = axis == 0 ? 1 : (axis == 1 ? g.nx : g.plane);
      const T* p = src + (long long)vidx(g, x, y, z) - (long long)r * stride;
      acc = tap<T>(taps.w[0], p[0]);
      for (int j = 1; j <= 2 * r; ++j) acc = fma_t(taps.w[j], p[j * stride], acc);
    } else {
      for (int j = 0; j <= 2 * r; ++j) {
        const int q = clampi(clampi(pos - r + j, 0, n_ax - 1), lo, hi);
        const size_t sidx = axis == 0 ? vidx(g, q, y, z) : (axis == 1 ? vidx(g, x, q, z) : vidx(g, x, y, q));
        const T v = src[sidx];
        acc = j == 0 ? tap<T>(taps.w[0], v) : fma_t(taps.w[j], v, acc);
      }
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

}  // namespace

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

int launch_conv_pair(const Geom& g, const Taps& t, float2* a, float2* b, cudaStream_t st) {
  const long long n = (long long)(g.ze - g.zb) * g.plane;
  conv_axis_kernel<float2><<<grid_for(n, 256), 256, 0, st>>>(g, t, 0, a, b, g.zb, g.ze);
  conv_axis_kernel<float2><<<grid_for(n, 256), 256, 0, st>>>(g, t, 1, b, a, g.zb, g.ze);
  conv_axis_kernel<float2><<<grid_for(n, 256), 256, 0, st>>>(g, t, 2, a, b, g.zb, g.ze);
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

__global__ void hh_kernel(Geom g, float inv_eps, const float* __restrict__ phi, const float* __restrict__ image,
                          float2* __restrict__ hh, long long first, long long n) {
  for (long long i = first + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < first + n;
       i += (long long)gridDim.x * blockDim.x) {
    float hm, hp;
    heaviside_pair(phi[i], inv_eps, hm, hp);
    hh[i] = make_float2(hm, hm * image[i]);
  }
}

int launch_hh(const Geom& g, float inv_eps, const float* phi, const float* image, float2* hh, int z_begin,
              int z_end, cudaStream_t st) {
  if (z_end <= z_begin) return 0;
  const long long n = (long long)(z_end - z_begin) * g.plane;
  hh_kernel<<<grid_for(n, 256), 256, 0, st>>>(g, inv_eps, phi, image, hh, (long long)(z_begin - g.zb) * g.plane, n);
  return 1;
}

int launch_mask(const float* phi, float* mask, long long n, cudaStream_t st) {
  mask_kernel<<<grid_for(n, 256), 256, 0, st>>>(phi, mask, n);
  return 1;
}

}  // namespace rsfg

// ------------------------------------------------------------ peer halo flags
namespace rsfg {
namespace {
// Publishes "the halo planes of step v have landed" into a (possibly peer)
// flag word; the preceding copy on the same stream is complete when this runs.
__global__ void flag_store_kernel(unsigned int* flag, unsigned int v) {
  __threadfence_system();
  *reinterpret_cast<volatile unsigned int*>(flag) = v;
  __threadfence_system();
}

// Fallback wait when stream memory operations are unavailable: one thread
// polls the local flag word until it reaches v.
__global__ void flag_wait_kernel(const unsigned int* flag, unsigned int v) {
  while (*reinterpret_cast<const volatile unsigned int*>(flag) < v) __nanosleep(200);
  __threadfence_system();
}
}  // namespace

int launch_flag_store(unsigned int* flag, unsigned int v, cudaStream_t st) {
  flag_store_kernel<<<1, 1, 0, st>>>(flag, v);
  return 1;
}

int launch_flag_wait(const unsigned int* flag, unsigned int v, cudaStream_t st) {
  flag_wait_kernel<<<1, 1, 0, st>>>(flag, v);
  return 1;
}
}  // namespace rsfg
