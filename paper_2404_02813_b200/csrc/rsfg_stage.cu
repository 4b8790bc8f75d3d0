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
#include <condition_variable>
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

// Persistent memcpy workers (thread creation per chunk cost ~0.1 ms per 16 MB
// chunk): the caller posts one job, every worker copies its slice, the
// caller copies slice 0 and waits for the rest.
class CopyPool {
 public:
  explicit CopyPool(int n) : n_(n) {
    for (int t = 1; t < n_; ++t) th_.emplace_back([this, t] { run(t); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      quit_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void copy(void* dst, const void* src, size_t n) {
    if (n_ == 1 || n < (1u << 20)) {
      std::memcpy(dst, src, n);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      n_bytes_ = n;
      pending_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    slice(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return pending_ == 0; });
  }

 private:
  void slice(int t) {
    const size_t per = (n_bytes_ + n_ - 1) / n_;
    const size_t a = std::min(n_bytes_, t * per), b = std::min(n_bytes_, a + per);
    if (b > a) std::memcpy(dst_ + a, src_ + a, b - a);
  }
  void run(int t) {
    unsigned long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (quit_) return;
      }
      slice(t);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_one();
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  unsigned long long gen_ = 0;
  bool quit_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t n_bytes_ = 0;
  int pending_ = 0;
};

void par_memcpy(void* dst, const void* src, size_t n) {
  static CopyPool pool(copy_threads());  // used under Pool::mu (one copy at a time)
  pool.copy(dst, src, n);
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
