// rsfg_phantom_gpu.cu -- device-side tube-network phantom + perturb
// (reference phantom.cpp:55-214, rng.hpp:10-60).
//
// The random-walk centerlines are serial in the RNG and cheap: they come from
// the host generator (rsfg_phantom.cpp, phantom_centerlines).  Everything
// per voxel runs here:
//  * the swept-ball signed distance is an order-independent min over samples
//    (phantom.cpp:113-137): one CTA per sample box, atomicMin on an ordered
//    integer encoding of the float distance -- exact in any order;
//  * image/ground truth from the distance, optional z-only blur (double
//    accumulation, ascending taps, clamp: phantom.cpp:140-166);
//  * perturb (phantom.cpp:186-214): SplitMix64 is a Weyl counter, so draw n of
//    the noise stream is mix(seed + (n+1) * 0x9e3779b97f4a7c15) and voxel i
//    takes Box-Muller pair floor(i/2) (draws 2p, 2p+1; cos for even i, sin for
//    odd i) -- every voxel independently.
// Differences from the host/reference generator can only come from libm
// rounding (device double log/sin/cos vs glibc) or FMA contraction order in
// the distance sum; they reach the float output in a vanishing fraction of
// voxels (tests/test_gpu_phantom.py bounds it).
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/rsfg.h"

struct rsfg_phantom_sample {
  double x, y, z, r;
};
int rsfg_phantom_samples_host(const rsfg_phantom_spec* s, std::vector<rsfg_phantom_sample>& out);

namespace {

__device__ __forceinline__ unsigned int enc(float f) {
  const unsigned int u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float dec(unsigned int u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

__global__ void fill_u32(unsigned int* p, unsigned int v, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}

// One CTA per sample: signed distance to the ball over its padded box.
__global__ void raster_kernel(const rsfg_phantom_sample* __restrict__ q, int nx, int ny, int nz, bool flat,
                              unsigned int* __restrict__ dist) {
  const rsfg_phantom_sample s = q[blockIdx.x];
  const int x0 = max(0, (int)floor(s.x - s.r - 1.5)), x1 = min(nx - 1, (int)ceil(s.x + s.r + 1.5));
  const int y0 = max(0, (int)floor(s.y - s.r - 1.5)), y1 = min(ny - 1, (int)ceil(s.y + s.r + 1.5));
  const int z0 = flat ? 0 : max(0, (int)floor(s.z - s.r - 1.5));
  const int z1 = flat ? 0 : min(nz - 1, (int)ceil(s.z + s.r + 1.5));
  const int bx = x1 - x0 + 1, by = y1 - y0 + 1, bz = z1 - z0 + 1;
  if (bx <= 0 || by <= 0 || bz <= 0) return;
  const int total = bx * by * bz;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int x = x0 + e % bx, y = y0 + (e / bx) % by, z = z0 + e / (bx * by);
    const double dx = x - s.x, dy = y - s.y, dz = z - s.z;
    const float d = (float)(sqrt(dx * dx + dy * dy + dz * dz) - s.r);
    atomicMin(dist + (size_t)x + (size_t)nx * ((size_t)y + (size_t)ny * z), enc(d));
  }
}

// image / ground truth from the distance (phantom.cpp:140-148), in place.
__global__ void compose_kernel(float* __restrict__ img, float* __restrict__ gt, size_t n, float fg, float bg) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float d = dec(__float_as_uint(img[i]));
    const float a = fminf(fmaxf(0.5f - d, 0.0f), 1.0f);
    img[i] = bg + (fg - bg) * a;
    if (gt) gt[i] = d < 0.0f ? 1.0f : 0.0f;
  }
}

// z-only Gaussian blur with clamp, double accumulation in ascending tap order.
__global__ void zblur_kernel(const float* __restrict__ in, float* __restrict__ out, int nz, size_t plane,
                             const double* __restrict__ w, int r) {
  const size_t n = plane * nz;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t xy = i % plane;
    const int z = (int)(i / plane);
    double acc = 0.0;
    for (int j = -r; j <= r; ++j) acc += w[j + r] * in[xy + plane * min(max(z + j, 0), nz - 1)];
    out[i] = (float)acc;
  }
}

__device__ __forceinline__ uint64_t splitmix(uint64_t z) {  // rng.hpp:14-19 (state already advanced)
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// perturb (phantom.cpp:186-214): Gaussian noise (Box-Muller pairs) and an
// intensity ramp along one axis, clamped to [0, 255], in place.
__global__ void perturb_kernel(float* __restrict__ img, int nx, int ny, int nz, double sigma, uint64_t seed,
                               int axis, double lo, double hi) {
  const size_t n = (size_t)nx * ny * nz;
  const uint64_t gamma = 0x9e3779b97f4a7c15ULL;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double v = img[i];
    if (sigma > 0.0) {
      const uint64_t p = i >> 1;
      const double a = (double)(splitmix(seed + (2 * p + 1) * gamma) >> 11) * 0x1.0p-53;
      const double b = (double)(splitmix(seed + (2 * p + 2) * gamma) >> 11) * 0x1.0p-53;
      const double rad = sqrt(-2.0 * log(a));
      const double ang = 2.0 * CUDART_PI * b;
      v += sigma * ((i & 1) ? rad * sin(ang) : rad * cos(ang));
    }
    double m = 1.0;
    if (axis) {
      const int x = (int)(i % nx), y = (int)((i / nx) % ny), z = (int)(i / ((size_t)nx * ny));
      const int c = axis == 1 ? x : axis == 2 ? y : z, len = axis == 1 ? nx : axis == 2 ? ny : nz;
      m = len <= 1 ? 0.5 * (lo + hi) : lo + (hi - lo) * (double)c / (len - 1);
    }
    img[i] = (float)fmin(fmax(v * m, 0.0), 255.0);
  }
}

}  // namespace

extern "C" {

// Device-side rsfg_phantom: same spec, DEVICE output buffers (d_gt may be NULL).
__attribute__((visibility("default"))) int rsfg_phantom_device(const rsfg_phantom_spec* s, float* d_image,
                                                               float* d_gt, int32_t device, int64_t* launches) {
  if (!s || !d_image) return RSFG_ERR_STATE;
  std::vector<rsfg_phantom_sample> samples;
  if (int rc = rsfg_phantom_samples_host(s, samples)) return rc;
  if (cudaSetDevice(device) != cudaSuccess) return RSFG_ERR_CUDA;
  const int nx = s->nx, ny = s->ny, nz = s->nz;
  const bool flat = nz == 1;
  const size_t n = (size_t)nx * ny * nz, plane = (size_t)nx * ny;
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return RSFG_ERR_CUDA;
  int64_t nl = 0;
  rsfg_phantom_sample* d_q = nullptr;
  float* tmp = nullptr;
  double* d_w = nullptr;
  int rc = RSFG_OK;
  const int grid = 148 * 16;
  do {
    unsigned int* dist = reinterpret_cast<unsigned int*>(d_image);  // distance first, image in place
    {
      // every voxel starts at +FLT_MAX (phantom.cpp:113), ordered-int encoded
      float fmax = 3.402823466e38f;
      unsigned int u;
      std::memcpy(&u, &fmax, 4);
      fill_u32<<<grid, 256, 0, st>>>(dist, u | 0x80000000u, n);
      ++nl;
    }
    if (!samples.empty()) {
      if (cudaMallocAsync(&d_q, samples.size() * sizeof(rsfg_phantom_sample), st) != cudaSuccess) {
        rc = RSFG_ERR_OOM;
        break;
      }
      cudaMemcpyAsync(d_q, samples.data(), samples.size() * sizeof(rsfg_phantom_sample), cudaMemcpyHostToDevice,
                      st);
      raster_kernel<<<(unsigned)samples.size(), 128, 0, st>>>(d_q, nx, ny, nz, flat, dist);
      ++nl;
    }
    compose_kernel<<<grid, 256, 0, st>>>(d_image, d_gt, n, s->foreground, s->background);
    ++nl;
    if (s->axial_blur_sigma > 0.0 && !flat) {
      const int r = (int)std::ceil(3.0 * s->axial_blur_sigma);
      std::vector<double> w(2 * r + 1);
      double sum = 0.0;
      for (int i = -r; i <= r; ++i) {
        w[i + r] = std::exp(-((double)i * i) / (2.0 * s->axial_blur_sigma * s->axial_blur_sigma));
        sum += w[i + r];
      }
      for (double& v : w) v /= sum;
      if (cudaMallocAsync(&tmp, n * sizeof(float), st) != cudaSuccess ||
          cudaMallocAsync(&d_w, w.size() * sizeof(double), st) != cudaSuccess) {
        rc = RSFG_ERR_OOM;
        break;
      }
      cudaMemcpyAsync(d_w, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice, st);
      cudaMemcpyAsync(tmp, d_image, n * sizeof(float), cudaMemcpyDeviceToDevice, st);
      zblur_kernel<<<grid, 256, 0, st>>>(tmp, d_image, nz, plane, d_w, r);
      ++nl;
    }
    perturb_kernel<<<grid, 256, 0, st>>>(d_image, nx, ny, nz, s->noise_sigma, s->noise_seed, s->contrast_axis,
                                         s->contrast_lo, s->contrast_hi);
    ++nl;
  } while (false);
  if (d_q) cudaFreeAsync(d_q, st);
  if (tmp) cudaFreeAsync(tmp, st);
  if (d_w) cudaFreeAsync(d_w, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (rc == RSFG_OK && (e != cudaSuccess || cudaGetLastError() != cudaSuccess)) rc = RSFG_ERR_CUDA;
  if (launches) *launches = nl;
  return rc;
}

}  // extern "C"
