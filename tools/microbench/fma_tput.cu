// Microbenchmark: FP32 FMA issue rates on sm_100a (3-reg FFMA, FFMA with a
// constant-bank operand, packed FFMA2) and a float4 copy for HBM bandwidth.
#include <cstdio>
#include <cuda_runtime.h>

__constant__ float c_w[64];

template <int CHAINS>
__global__ void ffma_reg(float* out, float a, float b, int iters) {
  float acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  float w = a + threadIdx.x * 1e-9f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = fmaf(acc[i], w, b);
  }
  float s = 0; 
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 3 distinct register operands per FMA
template <int CHAINS>
__global__ void ffma_3reg(float* out, float a, float b, int iters) {
  float acc[CHAINS], x[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { acc[i] = threadIdx.x * 1e-3f + i; x[i] = a + i * 1e-7f; }
  float w = b + threadIdx.x * 1e-9f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = fmaf(x[i], w, acc[i]);
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) x[i] = fmaf(x[i], w, acc[i]);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i] + x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// conv-like: acc = fma(c_w[j], v_j, acc) with v in registers, w from constant bank
template <int TAPS>
__global__ void ffma_const(float* out, float a, int iters) {
  float v[TAPS + 8];
#pragma unroll
  for (int i = 0; i < TAPS + 8; ++i) v[i] = a + i * 1e-3f + threadIdx.x * 1e-6f;
  float res = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      float acc = 0.f;
#pragma unroll
      for (int j = 0; j < TAPS; ++j) acc = fmaf(c_w[j], v[o + j], acc);
      v[o] = acc;
    }
  }
#pragma unroll
  for (int i = 0; i < TAPS + 8; ++i) res += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = res;
}

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long rb = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long rc = *reinterpret_cast<unsigned long long*>(&c);
  unsigned long long rd;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2*>(&rd);
}

template <int TAPS>
__global__ void ffma2_conv(float* out, float a, int iters) {
  float2 v[TAPS + 8];
#pragma unroll
  for (int i = 0; i < TAPS + 8; ++i) v[i] = make_float2(a + i * 1e-3f + threadIdx.x * 1e-6f, a - i * 1e-3f);
  float2 res = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < TAPS; ++j) { float w = c_w[j]; acc = ffma2(make_float2(w, w), v[o + j], acc); }
      v[o] = acc;
    }
  }
#pragma unroll
  for (int i = 0; i < TAPS + 8; ++i) { res.x += v[i].x; res.y += v[i].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = res.x + res.y;
}

template <int CHAINS>
__global__ void ffma2_reg(float* out, float a, float b, int iters) {
  float2 acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = make_float2(threadIdx.x * 1e-3f + i, i * 2.f);
  float2 w = make_float2(a + threadIdx.x * 1e-9f, a);
  float2 bb = make_float2(b, b + 1e-3f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = ffma2(acc[i], w, bb);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy4(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

#define TIME(label, flops_per, launch)                                              \
  {                                                                                 \
    launch; cudaDeviceSynchronize();                                                \
    cudaEventRecord(e0); launch; cudaEventRecord(e1); cudaEventSynchronize(e1);     \
    float ms; cudaEventElapsedTime(&ms, e0, e1);                                    \
    double fl = (double)(flops_per);                                                \
    printf("%-28s %8.3f ms  %8.2f TFMA/s (%.1f FMA/clk/SM @%.0f MHz)\n", label, ms,    \
           fl / ms / 1e9, fl / (ms * 1e-3) / (sms * clk_mhz * 1e6), clk_mhz);       \
  }

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount; int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double clk_mhz = clk_khz / 1000.0;
  printf("%s SMs=%d clk=%.0f MHz L2=%d MB smem/blk optin=%zu KB regs/SM=%d\n", p.name, sms, clk_mhz,
         p.l2CacheSize >> 20, p.sharedMemPerBlockOptin >> 10, p.regsPerMultiprocessor);
  float w[64]; for (int i = 0; i < 64; ++i) w[i] = 0.05f + i * 1e-4f;
  cudaMemcpyToSymbol(c_w, w, sizeof(w));
  float* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 8, thr = 256, iters = 4096;
  double nthr = (double)blocks * thr;
  TIME("ffma 2reg+imm chains16", nthr * iters * 16, (ffma_reg<16><<<blocks, thr>>>(out, 1.0001f, 0.5f, iters)));
  TIME("ffma 3reg chains8", nthr * iters * 16, (ffma_3reg<8><<<blocks, thr>>>(out, 1.0001f, 0.9999f, iters)));
  TIME("ffma const-bank conv19", nthr * (iters/8) * 8 * 19, (ffma_const<19><<<blocks, thr>>>(out, 1.0f, iters/8)));
  TIME("ffma2 conv19 (x2 lanes)", nthr * (iters/8) * 8 * 19 * 2, (ffma2_conv<19><<<blocks, thr>>>(out, 1.0f, iters/8)));
  TIME("ffma2 reg chains16 (x2)", nthr * iters * 16 * 2, (ffma2_reg<16><<<blocks, thr>>>(out, 1.0001f, 0.5f, iters)));
  size_t n = (size_t)1 << 28;  // 1 GiB per buffer
  float4 *a, *b; cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4);
  cudaMemset(a, 0, n * 4);
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0); copy4<<<sms * 16, 512>>>(a, b, n / 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy4 1GiB: %.3f ms  %.1f GB/s (r+w)\n", ms, 2.0 * n * 4 / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
