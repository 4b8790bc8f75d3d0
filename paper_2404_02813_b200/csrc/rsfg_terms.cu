// rsfg_terms.cu -- the reference's term-level APIs on the device:
// rsf::region_intensities (rsf.hpp:39-41, rsf.cpp:235-266) and
// rsf::directional_forces (rsf.hpp:47-50, rsf.cpp:268-291).  They expose the
// same arithmetic the fused step uses (Heaviside pair, separable Gaussian,
// clamped region means, fitting-error fields) as whole fields, for
// term-level tests and callers that want the intermediate volumes.
#include <cstring>
#include <string>

#include "../../include/rsfg.h"
#include "rsfg_device.cuh"

namespace rsfg {
namespace {

int grid_n(long long n) {
  long long b = (n + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 148LL * 16 ? 148LL * 16 : b));
}

// (H+, H+ I) and (H-, H- I) of phi (stage_heaviside_image, rsf.cpp:75-94).
__global__ void heaviside_both_kernel(float inv_eps, const float* __restrict__ phi, const float* __restrict__ image,
                                      float2* __restrict__ plus, float2* __restrict__ minus, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float hm, hp;
    heaviside_pair(phi[i], inv_eps, hm, hp);
    const float im = image[i];
    plus[i] = make_float2(hp, hp * im);
    minus[i] = make_float2(hm, hm * im);
  }
}

// r = clamp(K*(H I) / max(K*H, denom_floor), i_min, i_max) (rsf.cpp:251-261).
__global__ void region_mean_kernel(const float2* __restrict__ conv, float denom_floor, const unsigned int* mm,
                                   float* __restrict__ r, long long n) {
  const unsigned int ulo = mm[0], uhi = mm[1];
  const float lo = __uint_as_float((ulo & 0x80000000u) ? (ulo & 0x7fffffffu) : ~ulo);
  const float hi = __uint_as_float((uhi & 0x80000000u) ? (uhi & 0x7fffffffu) : ~uhi);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float2 c = conv[i];
    const float q = __fdiv_rn(c.y, fmaxf(c.x, denom_floor));
    r[i] = fminf(fmaxf(q, lo), hi);
  }
}

// F = f32((KI2 - 2 r KI) + r^2) in f64 (rsf.cpp:282-287), no contraction, so
// the f64 rounding points are the reference's.
__global__ void forces_kernel(const float* __restrict__ rp, const float* __restrict__ rm,
                              const float* __restrict__ ki, const float* __restrict__ ki2, float* __restrict__ Fp,
                              float* __restrict__ Fm, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double a = ki2[i], b = ki[i], p = rp[i], m = rm[i];
    Fp[i] = (float)__dadd_rn(__dsub_rn(a, __dmul_rn(__dmul_rn(2.0, p), b)), __dmul_rn(p, p));
    Fm[i] = (float)__dadd_rn(__dsub_rn(a, __dmul_rn(__dmul_rn(2.0, m), b)), __dmul_rn(m, m));
  }
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": CUDA error: " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? RSFG_ERR_OOM : RSFG_ERR_CUDA;
}

}  // namespace
}  // namespace rsfg

using namespace rsfg;

extern "C" {

__attribute__((visibility("default"))) int rsfg_region_intensities_device(const float* d_image, const float* d_phi,
                                                                          int32_t nx, int32_t ny, int32_t nz,
                                                                          double sigma1, double epsilon,
                                                                          double denom_floor, float* d_r_plus,
                                                                          float* d_r_minus, int32_t device) {
  if (!d_image || !d_phi || !d_r_plus || !d_r_minus) {
    set_error("region_intensities: null buffer");
    return RSFG_ERR_STATE;
  }
  if (nx <= 0 || ny <= 0 || nz <= 0) {
    set_error("region_intensities: volume dims must be positive");
    return RSFG_ERR_SHAPE;
  }
  // rsf.cpp:238-239, same messages.
  if (!(epsilon > 0.0)) {
    set_error("region_intensities: epsilon must be > 0");
    return RSFG_ERR_PARAM;
  }
  if (!(denom_floor > 0.0)) {
    set_error("region_intensities: denom_floor must be > 0");
    return RSFG_ERR_PARAM;
  }
  Taps t;
  if (int rc = gaussian_taps(sigma1, t)) return rc;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "region_intensities");
  const long long n = (long long)nx * ny * nz;
  Geom g{nx, ny, nz, 0, nz, (long long)nx * ny};
  cudaStream_t st = nullptr;
  float2 *P = nullptr, *M = nullptr, *T = nullptr;
  unsigned int* mm = nullptr;
  e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMallocAsync(&P, n * sizeof(float2), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&M, n * sizeof(float2), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&T, n * sizeof(float2), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&mm, 2 * sizeof(unsigned int), st);
  if (e == cudaSuccess) {
    const unsigned int init[2] = {0xffffffffu, 0u};
    e = cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, st);
  }
  if (e == cudaSuccess) {
    launch_minmax(g, d_image, 0, nz, mm, st);  // Volume::min_max (volume.cpp:25-33)
    heaviside_both_kernel<<<grid_n(n), 256, 0, st>>>((float)(1.0 / epsilon), d_phi, d_image, P, M, n);
    launch_conv_pair(g, t, P, T, st);  // K*H+, K*(H+ I) -> T
    region_mean_kernel<<<grid_n(n), 256, 0, st>>>(T, (float)denom_floor, mm, d_r_plus, n);
    launch_conv_pair(g, t, M, P, st);  // K*H-, K*(H- I) -> P
    region_mean_kernel<<<grid_n(n), 256, 0, st>>>(P, (float)denom_floor, mm, d_r_minus, n);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (st) {
    cudaFreeAsync(P, st);
    cudaFreeAsync(M, st);
    cudaFreeAsync(T, st);
    cudaFreeAsync(mm, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  }
  return e == cudaSuccess ? RSFG_OK : cuda_fail(e, "region_intensities");
}

__attribute__((visibility("default"))) int rsfg_directional_forces_device(const float* d_r_plus, const float* d_r_minus,
                                                                          const float* d_ki, const float* d_ki2,
                                                                          int64_t n, float* d_f_plus, float* d_f_minus,
                                                                          int32_t device) {
  if (n <= 0) return RSFG_OK;
  if (!d_r_plus || !d_r_minus || !d_ki || !d_ki2 || !d_f_plus || !d_f_minus) {
    set_error("directional_forces: null buffer");
    return RSFG_ERR_STATE;
  }
  cudaError_t e = cudaSetDevice(device);
  cudaStream_t st = nullptr;
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e == cudaSuccess) {
    forces_kernel<<<grid_n(n), 256, 0, st>>>(d_r_plus, d_r_minus, d_ki, d_ki2, d_f_plus, d_f_minus, n);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (st) cudaStreamDestroy(st);
  return e == cudaSuccess ? RSFG_OK : cuda_fail(e, "directional_forces");
}

// Host-buffer forms: the inputs go up, the fields come back.
__attribute__((visibility("default"))) int rsfg_region_intensities(const float* image, const float* phi, int32_t nx,
                                                                   int32_t ny, int32_t nz, double sigma1,
                                                                   double epsilon, double denom_floor,
                                                                   float* r_plus, float* r_minus, int32_t device) {
  if (!image || !phi || !r_plus || !r_minus) {
    set_error("region_intensities: null buffer");
    return RSFG_ERR_STATE;
  }
  if (nx <= 0 || ny <= 0 || nz <= 0) {
    set_error("region_intensities: volume dims must be positive");
    return RSFG_ERR_SHAPE;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "region_intensities");
  const size_t bytes = (size_t)nx * ny * nz * sizeof(float);
  float* d = nullptr;
  e = cudaMalloc(&d, 4 * bytes);
  if (e != cudaSuccess) return cuda_fail(e, "region_intensities");
  float *dI = d, *dP = d + bytes / 4, *dRp = d + 2 * (bytes / 4), *dRm = d + 3 * (bytes / 4);
  int rc = RSFG_OK;
  e = cudaMemcpy(dI, image, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(dP, phi, bytes, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) rc = cuda_fail(e, "region_intensities");
  if (!rc) rc = rsfg_region_intensities_device(dI, dP, nx, ny, nz, sigma1, epsilon, denom_floor, dRp, dRm, device);
  if (!rc) {
    e = cudaMemcpy(r_plus, dRp, bytes, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(r_minus, dRm, bytes, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = cuda_fail(e, "region_intensities");
  }
  cudaFree(d);
  return rc;
}

__attribute__((visibility("default"))) int rsfg_directional_forces(const float* r_plus, const float* r_minus,
                                                                   const float* ki, const float* ki2, int64_t n,
                                                                   float* f_plus, float* f_minus, int32_t device) {
  if (n <= 0) return RSFG_OK;
  if (!r_plus || !r_minus || !ki || !ki2 || !f_plus || !f_minus) {
    set_error("directional_forces: null buffer");
    return RSFG_ERR_STATE;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "directional_forces");
  const size_t bytes = (size_t)n * sizeof(float);
  float* d = nullptr;
  e = cudaMalloc(&d, 6 * bytes);
  if (e != cudaSuccess) return cuda_fail(e, "directional_forces");
  float* b[6];
  for (int i = 0; i < 6; ++i) b[i] = d + (size_t)i * n;
  const float* in[4] = {r_plus, r_minus, ki, ki2};
  for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaMemcpy(b[i], in[i], bytes, cudaMemcpyHostToDevice);
  int rc = e == cudaSuccess ? RSFG_OK : cuda_fail(e, "directional_forces");
  if (!rc) rc = rsfg_directional_forces_device(b[0], b[1], b[2], b[3], n, b[4], b[5], device);
  if (!rc) {
    e = cudaMemcpy(f_plus, b[4], bytes, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(f_minus, b[5], bytes, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = cuda_fail(e, "directional_forces");
  }
  cudaFree(d);
  return rc;
}

}  // extern "C"
