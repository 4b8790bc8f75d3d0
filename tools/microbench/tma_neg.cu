// Probe: does a 3-D fp32 TMA tile load accept negative and non-16-byte-aligned
// box starts (OOB elements zero-filled)?  Prints per-case OK/FAULT/MISMATCH.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap m, float* out, int cx, int cy) {
  extern __shared__ __align__(128) float s[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(40 * 12 * 4));
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(sa(s)), "l"(&m), "r"(cx), "r"(cy), "r"(0), "r"(sa(&bar)) : "memory");
  }
  __syncthreads();
  asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(sa(&bar)));
  for (int i = threadIdx.x; i < 480; i += blockDim.x) out[i] = s[i];
}
int main() {
  const int nx = 64, ny = 32, nz = 2;
  float* d; cudaMalloc(&d, nx * ny * nz * 4);
  float h[nx * ny * nz]; for (int i = 0; i < nx * ny * nz; ++i) h[i] = (float)(i + 1);
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  float* o; cudaMalloc(&o, 480 * 4);
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m;
  cuuint64_t dims[3] = {nx, ny, nz}, st[2] = {nx * 4, nx * ny * 4};
  cuuint32_t box[3] = {40, 12, 1}, es[3] = {1, 1, 1};
  int rc = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n", rc);
  int cases[][2] = {{0, 0}, {4, 2}, {-4, 0}, {-4, -2}, {-12, -9}, {60, 25}, {-8, 30}};
  for (auto& c : cases) {
    k<<<1, 128, 480 * 4>>>(m, o, c[0], c[1]);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("start (%d,%d): FAULT %s\n", c[0], c[1], cudaGetErrorString(e)); return 0; }
    float r[480]; cudaMemcpy(r, o, sizeof r, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int j = 0; j < 12; ++j) for (int i = 0; i < 40; ++i) {
      int gx = c[0] + i, gy = c[1] + j;
      float want = (gx >= 0 && gx < nx && gy >= 0 && gy < ny) ? h[gy * nx + gx] : 0.0f;
      bad += r[j * 40 + i] != want;
    }
    printf("start (%d,%d): %s (%d mismatches)\n", c[0], c[1], bad ? "MISMATCH" : "OK", bad);
  }
}
