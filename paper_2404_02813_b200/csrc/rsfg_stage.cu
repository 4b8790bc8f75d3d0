// rsfg_stage.cu -- host<->device copies of caller-owned PAGEABLE memory (the
// reference's callers hand over std::vector data, tiling.cpp:251).  A plain
// cudaMemcpy from pageable memory runs at ~10 GB/s (the driver bounces it
// through its own small pinned buffer on one thread); here the bytes go
// through a process-wide ring of pinned chunks, filled and drained by several
// host threads while the DMA engine moves the previous chunk, so PCIe runs at
// close to its pinned rate.  Pinned or registered host memory goes straight
// to cudaMemcpyAsync.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "rsfg_internal.h"

namespace rsfg {
namespace {

constexpr size_t kChunk = 16u << 20;  // bytes per pinned chunk
constexpr int kRing = 4;              // chunks in flight
constexpr int kMaxThreads = 16;       // host threads per chunk memcpy (cap)

int copy_threads() {
  static const int n = [] {
    const unsigned hw = std::thread::hardware_concurrency();
    return (int)std::min<unsigned>(kMaxThreads, std::max(1u, hw / 2));
  }();
  return n;
}

struct Pool {
  std::mutex mu;
  void* buf[kRing] = {};
  cudaEvent_t ev[kRing] = {};
  int dev = -1;
  bool ok = false;
};
Pool& pool() {
  static Pool p;
  return p;
}

// Pinned ring on the current device's context (events are per device).
bool pool_ready(Pool& p) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (p.ok && p.dev == dev) return true;
  for (int i = 0; i < kRing; ++i) {
    if (p.ev[i]) cudaEventDestroy(p.ev[i]), p.ev[i] = nullptr;
    if (!p.buf[i] && cudaMallocHost(&p.buf[i], kChunk) != cudaSuccess) return p.ok = false;
    if (cudaEventCreateWithFlags(&p.ev[i], cudaEventDisableTiming) != cudaSuccess) return p.ok = false;
  }
  p.dev = dev;
  return p.ok = true;
}

void par_memcpy(void* dst, const void* src, size_t n) {
  const int nt = copy_threads();
  const size_t per = (n + nt - 1) / nt;
  if (n < (1u << 20) || nt == 1) {
    std::memcpy(dst, src, n);
    return;
  }
  std::thread th[kMaxThreads - 1];
  for (int t = 1; t < nt; ++t) {
    const size_t a = std::min(n, t * per), b = std::min(n, a + per);
    th[t - 1] = std::thread([=] { std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a); });
  }
  std::memcpy(dst, src, std::min(n, per));
  for (int t = 1; t < nt; ++t) th[t - 1].join();
}

}  // namespace

bool host_is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

cudaError_t copy_h2d(void* dst, const void* src, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  if (host_is_pinned(src)) return cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st);
  Pool& p = pool();
  std::lock_guard<std::mutex> lk(p.mu);
  if (!pool_ready(p)) return cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st);
  bool used[kRing] = {};
  for (size_t off = 0, c = 0; off < n; off += kChunk, ++c) {
    const int b = (int)(c % kRing);
    const size_t len = std::min(kChunk, n - off);
    if (used[b]) {
      cudaError_t e = cudaEventSynchronize(p.ev[b]);  // the DMA that read this chunk is done
      if (e != cudaSuccess) return e;
    }
    par_memcpy(p.buf[b], static_cast<const char*>(src) + off, len);
    cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + off, p.buf[b], len, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaEventRecord(p.ev[b], st);
    if (e != cudaSuccess) return e;
    used[b] = true;
  }
  // the ring is reused by the next call: wait for the last DMAs out of it
  for (int b = 0; b < kRing; ++b)
    if (used[b]) {
      cudaError_t e = cudaEventSynchronize(p.ev[b]);
      if (e != cudaSuccess) return e;
    }
  return cudaSuccess;
}

cudaError_t copy_d2h(void* dst, const void* src, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  if (host_is_pinned(dst)) {
    cudaError_t e = cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st);
    return e == cudaSuccess ? cudaStreamSynchronize(st) : e;
  }
  Pool& p = pool();
  std::lock_guard<std::mutex> lk(p.mu);
  if (!pool_ready(p)) {
    cudaError_t e = cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st);
    return e == cudaSuccess ? cudaStreamSynchronize(st) : e;
  }
  const size_t nchunks = (n + kChunk - 1) / kChunk;
  // keep kRing DMAs queued; drain chunk c (host memcpy) while c+1.. transfer
  auto issue = [&](size_t c) {
    const size_t off = c * kChunk, len = std::min(kChunk, n - off);
    const int b = (int)(c % kRing);
    cudaError_t e = cudaMemcpyAsync(p.buf[b], static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, st);
    return e == cudaSuccess ? cudaEventRecord(p.ev[b], st) : e;
  };
  for (size_t c = 0; c < std::min<size_t>(kRing, nchunks); ++c)
    if (cudaError_t e = issue(c)) return e;
  for (size_t c = 0; c < nchunks; ++c) {
    const int b = (int)(c % kRing);
    if (cudaError_t e = cudaEventSynchronize(p.ev[b])) return e;
    const size_t off = c * kChunk, len = std::min(kChunk, n - off);
    par_memcpy(static_cast<char*>(dst) + off, p.buf[b], len);
    if (c + kRing < nchunks)
      if (cudaError_t e = issue(c + kRing)) return e;
  }
  return cudaSuccess;
}

}  // namespace rsfg
