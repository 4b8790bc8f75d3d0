// rsfg_api.cu -- the C-ABI (include/rsfg.h): contexts, buffers, the step
// schedule, error mapping.  Host code; kernels live in rsfg_kernels.cu.
//
// One engine type serves both the monolithic state (rsf::init_evolution /
// evolve_step, rsf.cpp:293-357) and z-slabs: a state is the
// slab [0, nz) with no halo.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rsfg.h"
#include "rsfg_internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      const int code_ = (e_ == cudaErrorMemoryAllocation) ? RSFG_ERR_OOM : RSFG_ERR_CUDA;   \
      return fail(code_, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #expr); \
    }                                                                                       \
  } while (0)

// rsf::RsfParams::validate (rsf.cpp:10-20), same messages.
int validate(const rsfg_params* p) {
  if (!p) return fail(RSFG_ERR_PARAM, "RsfParams: null");
  if (p->sigma1 < 0.0) return fail(RSFG_ERR_PARAM, "RsfParams: sigma1 must be >= 0");
  if (p->sigma2 < 0.0) return fail(RSFG_ERR_PARAM, "RsfParams: sigma2 must be >= 0");
  if (!(p->epsilon > 0.0)) return fail(RSFG_ERR_PARAM, "RsfParams: epsilon must be > 0");
  if (!(p->dt > 0.0)) return fail(RSFG_ERR_PARAM, "RsfParams: dt must be > 0");
  if (p->max_iters < 1) return fail(RSFG_ERR_PARAM, "RsfParams: max_iters must be >= 1");
  if (p->convergence_fraction < 0.0 || p->convergence_fraction >= 1.0)
    return fail(RSFG_ERR_PARAM, "RsfParams: convergence_fraction must be in [0,1)");
  if (!(p->denom_floor > 0.0)) return fail(RSFG_ERR_PARAM, "RsfParams: denom_floor must be > 0");
  if (!(p->grad_floor > 0.0)) return fail(RSFG_ERR_PARAM, "RsfParams: grad_floor must be > 0");
  return RSFG_OK;
}

// gaussian_kernel (ops.cpp:9-29): f64 weights exp(-i^2/(2 sigma^2)) / sum.
int gaussian(double sigma, std::vector<double>& w) {
  if (sigma < 0.0 || !std::isfinite(sigma)) {
    char buf[96];
    snprintf(buf, sizeof buf, "gaussian_kernel: sigma must be >= 0, got %f", sigma);
    return fail(RSFG_ERR_PARAM, buf);
  }
  if (sigma == 0.0) {
    w.assign(1, 1.0);
    return RSFG_OK;
  }
  const int r = (int)std::ceil(3.0 * sigma);
  w.assign(2 * r + 1, 0.0);
  double sum = 0.0;
  for (int i = -r; i <= r; ++i) {
    const double v = std::exp(-((double)i * i) / (2.0 * sigma * sigma));
    w[i + r] = v;
    sum += v;
  }
  for (double& v : w) v /= sum;
  return RSFG_OK;
}

int make_taps(double sigma, rsfg::Taps& t) {
  std::vector<double> w;
  if (int rc = gaussian(sigma, w)) return rc;
  if ((int)w.size() > rsfg::kMaxTaps - 1)
    return fail(RSFG_ERR_PARAM, "sigma too large for this build (radius > 31)");
  std::memset(&t, 0, sizeof t);
  t.r = (int)(w.size() / 2);
  for (size_t i = 0; i < w.size(); ++i) t.w[i] = (float)w[i];
  return RSFG_OK;
}

constexpr int kSlots = 64;  // per-iteration counter ring

// Rows of the reference's 14-stage profile (rsf.cpp:46-61, names at
// rsf.cpp:228-233) that carry a fused kernel's time: the Heaviside pass
// when it runs as its own kernel; kernel 1 (Heaviside + y/x passes of the
// (H, H I) pairs); kernel 2 (z pass, region means, forces, delta, gradient,
// normalisation, curvature, Laplacian, combine, update).
constexpr int kStageH = 0;        // "H-I"
constexpr int kStageConv = 2;     // "K*H-I"
constexpr int kStageCombine = 11; // "R-combine"

}  // namespace

namespace rsfg {
void set_error(const std::string& msg) { g_err = msg; }
int gaussian_taps(double sigma, Taps& t) { return make_taps(sigma, t); }
}  // namespace rsfg

// ------------------------------------------------------------------ engine
struct rsfg_slab {
  int dev = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int nx = 0, ny = 0, nz = 0, z0 = 0, z1 = 0, zb = 0, ze = 0, h = 0;
  rsfg_params p{};
  int fields = 2, check_every = 25;
  rsfg::Taps t1{}, t2{}, tid{};
  rsfg::StepConsts c{};
  bool fast = true;
  float* phi[2] = {nullptr, nullptr};
  int cur = 0;
  float* image = nullptr;
  float* k1i = nullptr;
  float* ki = nullptr;  // == image when sigma2 == 0
  float2* P[2] = {nullptr, nullptr};
  float2* scratch = nullptr;
  unsigned long long* counters = nullptr;   // device [kSlots][2]
  unsigned long long* h_counters = nullptr; // host mirror (ordinary memory: 1 KB, read after a sync)
  unsigned int* mm = nullptr;               // device min/max scratch
  rsfg::XYMaps xymaps[2] = {};              // TMA maps for kernel 1, per phi buffer
  rsfg::ZMaps zmaps[2] = {};                // TMA maps for kernel 2 (zst4), per phi buffer
  rsfg::XYMaps xy2maps[2] = {};             // TMA maps for kernel 1 (xy2), per phi buffer
  int xy2_ty = 32;                          // xy2 tile height
  // Stored-Heaviside mode (fields=2, sigma2=0, zst4 + xy2): kernel 2 writes
  // (H-, H- I) of phi' and kernel 1 reads it.  hh_valid: the owned planes'
  // pairs match the current phi (halo planes are always recomputed).
  float2* hh = nullptr;
  bool hh_mode = false;
  bool hh_valid = false;
  std::string env_key;  // kernel-variant environment at setup (workspace reuse must match it)
  // Stage profiling (rsf::KernelProfile, rsf.hpp:64-69): while prof_on, every
  // kernel launch of a step is bracketed by a CUDA-event pair tagged with the
  // reference stage row that carries its time (kStage* below).
  bool prof_on = false;
  // rsfg_evolve workspaces come from the library's stream-ordered pool (freed
  // memory stays cached for the next call up to a threshold; slabs, whose
  // buffers may be exported over CUDA IPC, use plain cudaMalloc)
  bool pooled = false;
  std::vector<cudaEvent_t> prof_ev;  // 2 per launch group
  std::vector<int> prof_stage;
  int prof_used = 0;
  // Peer halo links (rsfg_slab_link): flags[side] = the last step whose halo
  // planes on `side` have arrived (written by the neighbour after its copy).
  unsigned int* flags = nullptr;
  struct Link {
    bool on = false;
    bool ipc = false;        // pointers opened with cudaIpcOpenMemHandle (closed on release)
    int peer_dev = 0;
    float* phi[2] = {nullptr, nullptr};  // the neighbour's phi buffers (peer/IPC mapped)
    unsigned int* flag = nullptr;        // the neighbour's flag word for this face
    size_t src_off = 0, dst_off = 0, bytes = 0;
    void* ipc_base[3] = {nullptr, nullptr, nullptr};
  } link[2];
  cudaStream_t push_stream = nullptr;
  cudaEvent_t k2_done = nullptr, push_done = nullptr;
  bool push_pending = false;
  int slot = 0;
  int iteration = 0;
  long long launches = 0;
  bool valid = true;
  bool initialized = false;

  rsfg::Geom geom() const {
    rsfg::Geom g;
    g.nx = nx;
    g.ny = ny;
    g.nz = nz;
    g.zb = zb;
    g.ze = ze;
    g.plane = (long long)nx * ny;
    return g;
  }
  size_t held() const { return (size_t)(ze - zb) * (size_t)nx * ny; }
  size_t owned() const { return (size_t)(z1 - z0) * (size_t)nx * ny; }
  size_t off(int z) const { return (size_t)(z - zb) * (size_t)nx * ny; }
};

struct rsfg_state {
  rsfg_slab e;
};

namespace {
void destroy_state(rsfg_state* st);
// rsfg_evolve workspace of this thread (opt-in, rsfg_options.reuse_workspace):
// freed by rsfg_release_workspace() or when the thread exits.
struct WorkspaceCache {
  rsfg_state* st = nullptr;
  ~WorkspaceCache() {
    if (st) destroy_state(st);
  }
};
thread_local WorkspaceCache t_cache;

// Environment switches that select kernel variants at setup (tests and
// probes flip them); a reused workspace must have been set up under the same.
std::string variant_env_key() {
  std::string k;
  for (const char* v : {"RSFG_HH", "RSFG_XY2", "RSFG_XY2_TY", "RSFG_TMA", "RSFG_ZST4", "RSFG_FUSED"}) {
    const char* e = std::getenv(v);
    k += v;
    k += '=';
    k += e ? e : "";
    k += ';';
  }
  return k;
}
}

namespace {

// Per-device stream-ordered memory pool for rsfg_evolve's workspace.  A
// workspace returned to it stays mapped (up to 1/8 of the device memory) so a
// repeated call skips cudaMalloc/cudaFree of several GB -- which measured
// 4 ms to 0.6 s per call on B200 (profiles/r02_e2e_probe.jsonl).
// rsfg_release_workspace() trims it.
std::mutex g_pool_mu;
cudaMemPool_t g_pools[64] = {};

cudaMemPool_t lib_pool(int dev) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!g_pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    if (cudaMemPoolCreate(&g_pools[dev], &props) != cudaSuccess) {
      cudaGetLastError();
      g_pools[dev] = nullptr;
      return nullptr;
    }
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    uint64_t keep = total_b / 8;
    cudaMemPoolSetAttribute(g_pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
  }
  return g_pools[dev];
}

cudaError_t dev_alloc(rsfg_slab* s, void** p, size_t bytes) {
  if (s->pooled) {
    if (cudaMemPool_t pool = lib_pool(s->dev)) return cudaMallocFromPoolAsync(p, bytes, pool, s->stream);
  }
  return cudaMalloc(p, bytes);
}

void dev_free(rsfg_slab* s, void* p) {
  if (!p) return;
  if (s->pooled)
    cudaFreeAsync(p, s->stream);
  else
    cudaFree(p);
}

void release(rsfg_slab* s) {
  if (!s) return;
  cudaSetDevice(s->dev);
  dev_free(s, s->phi[0]);
  dev_free(s, s->phi[1]);
  dev_free(s, s->image);
  dev_free(s, s->k1i);
  if (s->ki != s->image) dev_free(s, s->ki);
  dev_free(s, s->P[0]);
  dev_free(s, s->P[1]);
  dev_free(s, s->scratch);
  dev_free(s, s->hh);
  dev_free(s, s->counters);
  dev_free(s, s->mm);
  delete[] s->h_counters;
  s->h_counters = nullptr;
  for (cudaEvent_t e : s->prof_ev) cudaEventDestroy(e);
  s->prof_ev.clear();
  if (s->push_stream) cudaStreamSynchronize(s->push_stream), cudaStreamDestroy(s->push_stream);
  if (s->k2_done) cudaEventDestroy(s->k2_done);
  if (s->push_done) cudaEventDestroy(s->push_done);
  for (auto& L : s->link)
    for (void* b : L.ipc_base)
      if (b) cudaIpcCloseMemHandle(b);
  dev_free(s, s->flags);
  if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
}

int prof_begin(rsfg_slab* s) {
  const int i = s->prof_used;
  while ((int)s->prof_ev.size() < 2 * (i + 1)) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    s->prof_ev.push_back(e);
  }
  if ((int)s->prof_stage.size() < i + 1) s->prof_stage.resize(i + 1);
  if (cudaEventRecord(s->prof_ev[2 * i], s->stream) != cudaSuccess) return -1;
  s->prof_used = i + 1;
  return i;
}

// Brackets the launches of one scope with an event pair (no-op unless prof_on).
struct ProfScope {
  rsfg_slab* s;
  int stage, idx = -1;
  ProfScope(rsfg_slab* s_, int st) : s(s_), stage(st) {
    if (s->prof_on) idx = prof_begin(s);
  }
  ~ProfScope() {
    if (idx < 0) return;
    s->prof_stage[idx] = stage;
    cudaEventRecord(s->prof_ev[2 * idx + 1], s->stream);
  }
};

// Adds the recorded launch-group times to seconds[14] (syncs the stream).
void prof_collect(rsfg_slab* s, double* seconds) {
  if (s->prof_used == 0) return;
  cudaStreamSynchronize(s->stream);
  for (int i = 0; i < s->prof_used; ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, s->prof_ev[2 * i], s->prof_ev[2 * i + 1]) == cudaSuccess && seconds)
      seconds[s->prof_stage[i]] += 1e-3 * ms;
  }
  s->prof_used = 0;
}

void destroy_state(rsfg_state* st) {
  if (!st) return;
  release(&st->e);
  delete st;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  if (!enc) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  return enc;
}

// 3-D fp32 tensor map over the held planes of a slab buffer with `cols`
// floats per row (nx, or 2*nx for float2 pairs) and the given box.
bool encode_map(CUtensorMap* m, const void* ptr, int cols, int rows, int planes, int bx, int by, int bz) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)planes};
  const cuuint64_t strides[2] = {(cuuint64_t)cols * 4, (cuuint64_t)cols * rows * 4};
  const cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA descriptors for kernel 1's tiles (3-D fp32 maps of the held planes).
// Needs 16-byte row pitch (nx % 4 == 0); otherwise kernel 1 uses LDG.
void make_xy_maps(rsfg_slab* s) {
  s->xymaps[0].valid = s->xymaps[1].valid = false;
  int bx = 0, by = 0;
  // Opt-in: measured on B200 the single-shot TMA tile is not faster than the
  // batched-LDG prologue at 512^3 (profiles/r01_tma_vs_ldg.txt).
  const char* on = std::getenv("RSFG_TMA");
  if (!(on && on[0] == '1') || !s->fast || (s->nx % 4) != 0 || !rsfg::xy_tma_box(s->t1.r, &bx, &by)) return;
  const int planes = s->ze - s->zb;
  CUtensorMap img;
  if (!encode_map(&img, s->image, s->nx, s->ny, planes, bx, by, 1)) return;
  for (int b = 0; b < 2; ++b) {
    if (!encode_map(&s->xymaps[b].phi, s->phi[b], s->nx, s->ny, planes, bx, by, 1)) return;
    s->xymaps[b].img = img;
  }
  s->xymaps[0].valid = s->xymaps[1].valid = true;
}

// TMA descriptors for kernel 1's multi-plane variant (xy2).  Needs nx % 4 ==
// 0.  RSFG_XY2=0 selects the single-plane kernel 1; RSFG_XY2_TY=64 the
// 64 x 64 tile.
void make_xy2_maps(rsfg_slab* s) {
  s->xy2maps[0].valid = s->xy2maps[1].valid = false;
  const char* off = std::getenv("RSFG_XY2");
  if ((off && off[0] == '0') || !s->fast || (s->nx % 4) != 0) return;
  // Tile height: 64 x 64 (1 CTA/SM, 16 warps) amortises the Heaviside halo
  // better at large radii (fields=2; the fields=4 64 x 64 tile does not fit
  // shared memory); 64 x 32 (2 CTAs/SM) wins up to R = 12
  // (profiles/r01_xy2_tile_height.txt).  RSFG_XY2_TY=32|64 overrides.
  const char* ty = std::getenv("RSFG_XY2_TY");
  // (R >= 19: the 64 x 64 tile's haloed pairs exceed shared memory; 64 x 32.
  // The stored-Heaviside kernel 1 is a 64 x 32 tile at every radius.)
  const char* hh_env0 = std::getenv("RSFG_HH");
  const bool hh_possible = (hh_env0 ? hh_env0[0] == '1' : true) && s->t1.r <= rsfg::kHHMaxR && s->fields == 2 &&
                           s->t2.r == 0;
  s->xy2_ty = ty ? (std::atoi(ty) == 64 ? 64 : 32)
                 : (!hh_possible && s->t1.r >= 15 && s->t1.r <= 18 && s->fields == 2 ? 64 : 32);
  int bx = 0, by = 0;
  if (!rsfg::xy2_box(s->t1.r, s->xy2_ty, &bx, &by)) return;
  const int planes = s->ze - s->zb;
  CUtensorMap img;
  if (!encode_map(&img, s->image, s->nx, s->ny, planes, bx, by, 1)) return;
  for (int b = 0; b < 2; ++b) {
    if (!encode_map(&s->xy2maps[b].phi, s->phi[b], s->nx, s->ny, planes, bx, by, 1)) return;
    s->xy2maps[b].img = img;
  }
  s->xy2maps[0].valid = s->xy2maps[1].valid = true;
  // Stored-Heaviside mode (fields = 2, sigma2 = 0, every specialised radius):
  // kernel 2 evaluates H once per voxel instead of kernel 1 on every haloed
  // tile (rsfg_internal.h kHHMaxR).  RSFG_HH=0 turns it off.  Needs zst4 (it
  // writes the pairs).
  const char* hh_env = std::getenv("RSFG_HH");
  // (the stored-Heaviside kernels exist up to kHHMaxR: RSFG_HH=1 cannot force it past that)
  const bool hh_want = (hh_env ? hh_env[0] == '1' : true) && s->t1.r <= rsfg::kHHMaxR;
  if (hh_want && s->xy2_ty == 32 && s->fields == 2 && s->t2.r == 0 && s->zmaps[0].valid && s->hh) {
    CUtensorMap m;
    if (encode_map(&m, s->hh, 2 * s->nx, s->ny, planes, 2 * bx, by, 1)) {
      for (int b = 0; b < 2; ++b) s->xy2maps[b].hh = m, s->xy2maps[b].use_hh = true;
      s->hh_mode = true;
    }
  }
}

// TMA descriptors for kernel 2 (zst4).  Needs nx % 4 == 0 (16-byte phi rows).
// RSFG_ZST4=0 selects the LDG-staged kernel 2 instead.
void make_z_maps(rsfg_slab* s) {
  s->zmaps[0].valid = s->zmaps[1].valid = false;
  const char* off = std::getenv("RSFG_ZST4");
  if ((off && off[0] == '0') || !s->fast || (s->nx % 4) != 0) return;
  int bz = 0, ty = 8;
  if (!rsfg::zst4_box(s->t1.r, s->fields, &bz, &ty)) return;
  const int planes = s->ze - s->zb;
  // A P window deeper than the held planes is never loaded by TMA (the
  // kernel's in-range test fails for every group); encode a valid map anyway.
  rsfg::ZMaps m;
  for (int f = 0; f < 2; ++f) {
    const float2* P = s->P[f] ? s->P[f] : s->P[0];
    if (!encode_map(&m.p[f], P, 2 * s->nx, s->ny, planes, 64, ty, std::min(bz, planes))) return;
  }
  if (!encode_map(&m.ki, s->ki, s->nx, s->ny, planes, 32, ty, 1)) return;
  if (!encode_map(&m.k1i, s->k1i ? s->k1i : s->ki, s->nx, s->ny, planes, 32, ty, 1)) return;
  for (int b = 0; b < 2; ++b) {
    s->zmaps[b] = m;
    if (!encode_map(&s->zmaps[b].phi, s->phi[b], s->nx, s->ny, planes, 40, ty + 4, 1)) return;
  }
  s->zmaps[0].valid = s->zmaps[1].valid = true;
}

int setup(rsfg_slab* s, int nx, int ny, int nz, int z0, int z1, const rsfg_params* p,
          const rsfg_options* o) {
  if (int rc = validate(p)) return rc;
  rsfg_options opt;
  rsfg_options_default(&opt);
  if (o) opt = *o;
  if (opt.fields != 2 && opt.fields != 4) return fail(RSFG_ERR_PARAM, "options.fields must be 2 or 4");
  if (nx <= 0 || ny <= 0 || nz <= 0)
    return fail(RSFG_ERR_SHAPE, "volume dims must be positive");
  if (z0 < 0 || z1 > nz || z0 >= z1) return fail(RSFG_ERR_SHAPE, "slab range must satisfy 0 <= z0 < z1 <= nz");
  s->p = *p;
  s->fields = opt.fields;
  s->check_every = std::min(std::max(opt.check_every, 1), kSlots);
  s->dev = opt.device;
  if (int rc = make_taps(p->sigma1, s->t1)) return rc;
  if (int rc = make_taps(p->sigma2, s->t2)) return rc;
  std::memset(&s->tid, 0, sizeof s->tid);
  s->tid.w[0] = 1.0f;
  s->tid.r = 0;
  // fast path: specialised kernels for this radius that fit shared memory
  // (kernel 1: xy2 when rows are 16-byte aligned, else the LDG-staged xy)
  {
    const int r = s->t1.r;
    const int ty = (r >= 15 && r <= 18 && s->fields == 2) ? 64 : 32;
    s->fast = rsfg::has_fast_radius(r) &&
              (((nx % 4) == 0 && (rsfg::xy2_fits(r, s->fields, ty) || rsfg::xy2_fits(r, s->fields, 32))) ||
               rsfg::xy_fits(r, s->fields));
  }
  s->env_key = variant_env_key();
  s->nx = nx;
  s->ny = ny;
  s->nz = nz;
  s->z0 = z0;
  s->z1 = z1;
  s->h = std::max(std::max(s->t1.r, s->t2.r), 2);
  s->zb = std::max(z0 - s->h, 0);
  s->ze = std::min(z1 + s->h, nz);
  // Halo planes come from the adjacent slab only: a slab with an interior
  // face must be at least h planes thick (then every face exchanges h).
  if ((z0 > 0 || z1 < nz) && z1 - z0 < s->h)
    return fail(RSFG_ERR_SHAPE, "slab thinner than its halo (" + std::to_string(z1 - z0) + " < " +
                                    std::to_string(s->h) + " planes)");
  // Step scalars (rsf.cpp:86,105,118,142,161,334).
  const double eps = p->epsilon;
  s->c.inv_eps = (float)(1.0 / eps);
  s->c.c_delta = (float)((1.0 / M_PI) * eps);
  s->c.eps2 = (float)(eps * eps);
  s->c.alpha = (float)p->alpha;
  s->c.beta = (float)p->beta;
  s->c.denom_floor = (float)p->denom_floor;
  s->c.grad_floor = (float)p->grad_floor;
  s->c.dt = p->dt;
  s->c.dt_f = (float)p->dt;
  s->c.inv_grad_floor = (float)(1.0 / p->grad_floor);

  CUDA_TRY(cudaSetDevice(s->dev));
  CUDA_TRY(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  s->own_stream = true;
  const size_t held = s->held();
  CUDA_TRY(dev_alloc(s, (void**)&s->phi[0], held * sizeof(float)));
  CUDA_TRY(dev_alloc(s, (void**)&s->phi[1], held * sizeof(float)));
  CUDA_TRY(dev_alloc(s, (void**)&s->image, held * sizeof(float)));
  if (s->fields == 2) CUDA_TRY(dev_alloc(s, (void**)&s->k1i, held * sizeof(float)));
  if (s->t2.r > 0)
    CUDA_TRY(dev_alloc(s, (void**)&s->ki, held * sizeof(float)));
  else
    s->ki = s->image;
  CUDA_TRY(dev_alloc(s, (void**)&s->P[0], held * sizeof(float2)));
  if (s->fields == 4) CUDA_TRY(dev_alloc(s, (void**)&s->P[1], held * sizeof(float2)));
  if (!s->fast) CUDA_TRY(dev_alloc(s, (void**)&s->scratch, held * sizeof(float2) * (s->fields == 4 ? 4 : 2)));
  CUDA_TRY(dev_alloc(s, (void**)&s->counters, kSlots * 2 * sizeof(unsigned long long)));
  // the whole ring is read back at each check (only the stepped slots matter)
  CUDA_TRY(cudaMemsetAsync(s->counters, 0, kSlots * 2 * sizeof(unsigned long long), s->stream));
  CUDA_TRY(dev_alloc(s, (void**)&s->mm, 2 * sizeof(unsigned int)));
  // (not cudaMallocHost: page-locking per call stalls when much memory is pinned)
  s->h_counters = new unsigned long long[kSlots * 2]();
  CUDA_TRY(dev_alloc(s, (void**)&s->flags, 2 * sizeof(unsigned int)));
  CUDA_TRY(cudaMemsetAsync(s->flags, 0, 2 * sizeof(unsigned int), s->stream));
  if (s->fast && s->fields == 2 && s->t2.r == 0 && (s->nx % 4) == 0)
    CUDA_TRY(dev_alloc(s, (void**)&s->hh, held * sizeof(float2)));
  make_xy_maps(s);
  make_z_maps(s);
  make_xy2_maps(s);
  // Never-read halo planes must still be finite memory: zero everything once.
  CUDA_TRY(cudaMemsetAsync(s->phi[0], 0, held * sizeof(float), s->stream));
  CUDA_TRY(cudaMemsetAsync(s->phi[1], 0, held * sizeof(float), s->stream));
  return RSFG_OK;
}

// New parameters on an existing workspace of the same shape and radii.
int reconfigure(rsfg_slab* s, const rsfg_params* p, const rsfg_options* o) {
  if (int rc = validate(p)) return rc;
  s->p = *p;
  s->check_every = std::min(std::max(o->check_every, 1), kSlots);
  const double eps = p->epsilon;
  s->c.inv_eps = (float)(1.0 / eps);
  s->c.c_delta = (float)((1.0 / M_PI) * eps);
  s->c.eps2 = (float)(eps * eps);
  s->c.alpha = (float)p->alpha;
  s->c.beta = (float)p->beta;
  s->c.denom_floor = (float)p->denom_floor;
  s->c.grad_floor = (float)p->grad_floor;
  s->c.inv_grad_floor = (float)(1.0 / p->grad_floor);
  s->c.dt = p->dt;
  s->c.dt_f = (float)p->dt;
  s->cur = 0;
  s->slot = 0;
  s->iteration = 0;
  s->valid = true;
  s->initialized = false;
  s->hh_valid = false;
  s->prof_on = false;
  s->prof_used = 0;
  return RSFG_OK;
}

int upload(rsfg_slab* s, const float* phi, const float* image, cudaMemcpyKind kind) {
  CUDA_TRY(cudaSetDevice(s->dev));
  s->hh_valid = false;
  const size_t bytes = s->held() * sizeof(float);
  if (kind == cudaMemcpyHostToDevice) {  // caller memory, pageable or pinned
    CUDA_TRY(rsfg::copy_h2d(s->phi[s->cur], phi, bytes, s->stream));
    CUDA_TRY(rsfg::copy_h2d(s->image, image, bytes, s->stream));
    return RSFG_OK;
  }
  CUDA_TRY(cudaMemcpyAsync(s->phi[s->cur], phi, bytes, kind, s->stream));
  CUDA_TRY(cudaMemcpyAsync(s->image, image, bytes, kind, s->stream));
  return RSFG_OK;
}

int local_range(rsfg_slab* s, float* lo, float* hi) {
  CUDA_TRY(cudaSetDevice(s->dev));
  const unsigned int init[2] = {0xffffffffu, 0u};
  CUDA_TRY(cudaMemcpyAsync(s->mm, init, sizeof init, cudaMemcpyHostToDevice, s->stream));
  s->launches += rsfg::launch_minmax(s->geom(), s->image, s->z0, s->z1, s->mm, s->stream);
  unsigned int out[2];
  CUDA_TRY(cudaMemcpyAsync(out, s->mm, sizeof out, cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  *lo = rsfg::decode_ordered(out[0]);
  *hi = rsfg::decode_ordered(out[1]);
  return RSFG_OK;
}

// init_evolution's static part (rsf.cpp:299-311): K1*I (fields=2) and
// K2*I (sigma2 > 0) on the owned planes.  K2*I^2 is never formed: only
// F- - F+ enters E and it cancels.
int init_static(rsfg_slab* s, float i_min, float i_max) {
  CUDA_TRY(cudaSetDevice(s->dev));
  s->c.i_min = i_min;
  s->c.i_max = i_max;
  const rsfg::Geom g = s->geom();
  float* tmp0 = reinterpret_cast<float*>(s->P[0]);
  float* tmp1 = tmp0 + s->held();
  if (s->fields == 2) {
    if (s->t1.r > 0)
      s->launches += rsfg::launch_convolve(g, s->t1, s->image, s->k1i, tmp0, tmp1, s->z0, s->z1, s->stream);
    else
      CUDA_TRY(cudaMemcpyAsync(s->k1i + s->off(s->z0), s->image + s->off(s->z0), s->owned() * sizeof(float),
                               cudaMemcpyDeviceToDevice, s->stream));
  }
  if (s->t2.r > 0)
    s->launches += rsfg::launch_convolve(g, s->t2, s->image, s->ki, tmp0, tmp1, s->z0, s->z1, s->stream);
  CUDA_TRY(cudaGetLastError());
  s->initialized = true;
  return RSFG_OK;
}

int check_shape(const rsfg_slab* s) {
  if (s->nx < 2 || s->ny < 2 || s->nz < 2) {
    char buf[128];
    snprintf(buf, sizeof buf, "gradient: every axis needs extent >= 2, got %dx%dx%d", s->nx, s->ny, s->nz);
    return fail(RSFG_ERR_SHAPE, buf);
  }
  return RSFG_OK;
}

rsfg::StepBuffers buffers(rsfg_slab* s, float* out) {
  rsfg::StepBuffers b;
  b.phi = s->phi[s->cur];
  b.image = s->image;
  b.k1i = s->k1i;
  b.ki = s->ki;
  b.P[0] = s->P[0];
  b.P[1] = s->P[1];
  b.out = out;
  b.counters = s->counters + 2 * s->slot;
  b.hh = nullptr;
  return b;
}

// xy work for planes [a, b) of the current phi.
int xy_planes(rsfg_slab* s, int a, int b) {
  if (b <= a) return RSFG_OK;
  const rsfg::Geom g = s->geom();
  int n;
  if (s->fast) {
    if (s->hh_mode && !(s->hh_valid && a >= s->z0 && b <= s->z1)) {
      // pairs of planes kernel 2 did not write for the current phi
      ProfScope ps(s, kStageH);
      s->launches += rsfg::launch_hh(g, s->c.inv_eps, s->phi[s->cur], s->image, s->hh, a, b, s->stream);
    }
    ProfScope ps(s, kStageConv);
    n = rsfg::launch_xy2(g, s->fields, s->xy2_ty, s->t1, s->c.inv_eps, s->P[0], s->P[1], a, b, s->xy2maps[s->cur],
                         s->stream);
    if (n < 0)
      n = rsfg::launch_xy(g, s->fields, s->t1, s->c.inv_eps, s->phi[s->cur], s->image, s->P[0], s->P[1], a, b,
                          &s->xymaps[s->cur], s->stream);
  } else {
    ProfScope ps(s, kStageConv);
    n = rsfg::launch_generic_conv(g, s->fields, s->t1, s->c.inv_eps, s->phi[s->cur], s->image, s->P,
                                  s->scratch, a, b, 0, 0, s->stream);
  }
  if (n < 0) return fail(RSFG_ERR_CUDA, "xy launch failed");
  s->launches += n;
  CUDA_TRY(cudaGetLastError());
  return RSFG_OK;
}

int step_interior(rsfg_slab* s) {
  if (!s->valid) return fail(RSFG_ERR_STATE, "state invalidated by an earlier blowup or error");
  if (!s->initialized) return fail(RSFG_ERR_STATE, "slab not initialised");
  if (int rc = check_shape(s)) return rc;
  CUDA_TRY(cudaSetDevice(s->dev));
  return xy_planes(s, s->z0, s->z1);
}

// Halo xy work, then kernel 2 over the owned planes; mode kUpdate swaps.
int step_finish(rsfg_slab* s, rsfg::StepMode mode, float* out) {
  CUDA_TRY(cudaSetDevice(s->dev));
  const int r = s->t1.r;
  if (int rc = xy_planes(s, std::max(s->z0 - r, s->zb), s->z0)) return rc;
  if (int rc = xy_planes(s, s->z1, std::min(s->z1 + r, s->ze))) return rc;
  const rsfg::Geom g = s->geom();
  if (mode == rsfg::kUpdate) {
    // slot: [0] sign changes = 0, [1] first bad = ~0
    CUDA_TRY(cudaMemsetAsync(s->counters + 2 * s->slot, 0, sizeof(unsigned long long), s->stream));
    CUDA_TRY(cudaMemsetAsync(s->counters + 2 * s->slot + 1, 0xff, sizeof(unsigned long long), s->stream));
  }
  rsfg::StepBuffers b = buffers(s, out);
  int n;
  if (s->fast) {
    ProfScope ps(s, kStageCombine);
    n = -1;
    if (mode == rsfg::kUpdate) {
      b.hh = s->hh_mode ? s->hh : nullptr;
      n = rsfg::launch_zst4(g, s->fields, s->t1, s->c, b, s->z0, s->z1, s->zmaps[s->cur], s->stream);
      // the pairs now describe phi' (owned planes) iff zst4 ran and wrote them
      if (s->hh_mode) s->hh_valid = n >= 0;
    }
    if (n < 0) n = rsfg::launch_zst(g, s->fields, s->t1, s->c, b, s->z0, s->z1, mode, s->stream);
  } else {
    int m;
    {
      ProfScope ps(s, kStageConv);
      m = rsfg::launch_generic_conv(g, s->fields, s->t1, s->c.inv_eps, s->phi[s->cur], s->image, s->P,
                                    s->scratch, 0, 0, s->z0, s->z1, s->stream);
    }
    if (m < 0) return fail(RSFG_ERR_CUDA, "generic convolution launch failed");
    s->launches += m;
    ProfScope ps(s, kStageCombine);
    n = rsfg::launch_zst(g, s->fields, s->tid, s->c, b, s->z0, s->z1, mode, s->stream);
  }
  if (n < 0) return fail(RSFG_ERR_CUDA, "step launch failed");
  s->launches += n;
  CUDA_TRY(cudaGetLastError());
  if (mode == rsfg::kUpdate) {
    s->cur ^= 1;
    s->iteration += 1;
    s->slot = (s->slot + 1) % kSlots;
  }
  return RSFG_OK;
}

// Reads counters of the last `k` steps (oldest first).  Returns RSFG_OK or
// RSFG_ERR_BLOWUP with g_err set (rsf.cpp:346-352 message).
int check_counters(rsfg_slab* s, int k, long long* last_sign_changes, int* first_bad_iter) {
  CUDA_TRY(cudaMemcpyAsync(s->h_counters, s->counters, kSlots * 2 * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  if (first_bad_iter) *first_bad_iter = 0;
  for (int i = k; i >= 1; --i) {
    const int sl = ((s->slot - i) % kSlots + kSlots) % kSlots;
    const unsigned long long bad = s->h_counters[2 * sl + 1];
    if (last_sign_changes && i == 1) *last_sign_changes = (long long)s->h_counters[2 * sl];
    if (bad != ~0ull) {
      const int it = s->iteration - i + 1;  // 1-based iteration of that step
      const long long plane = (long long)s->nx * s->ny;
      const int x = (int)(bad % s->nx), y = (int)((bad / s->nx) % s->ny), z = (int)(bad / plane);
      if (first_bad_iter) *first_bad_iter = it;
      char buf[160];
      snprintf(buf, sizeof buf, "evolution produced a non-finite value at voxel (%d,%d,%d), iteration %d", x, y,
               z, it);
      g_err = buf;
      return RSFG_ERR_BLOWUP;
    }
  }
  return RSFG_OK;
}

int create_common(rsfg_state** out, const float* phi0, const float* image, int nx, int ny, int nz,
                  const rsfg_params* p, const rsfg_options* o, cudaMemcpyKind kind) {
  if (!out) return fail(RSFG_ERR_STATE, "null output handle");
  *out = nullptr;
  auto* st = new rsfg_state;
  rsfg_slab* s = &st->e;
  int rc = setup(s, nx, ny, nz, 0, nz, p, o);
  if (!rc) rc = upload(s, phi0, image, kind);
  float lo = 0, hi = 0;
  if (!rc) rc = local_range(s, &lo, &hi);
  if (!rc) rc = init_static(s, lo, hi);
  if (rc) {
    std::string keep = g_err;
    release(s);
    delete st;
    g_err = keep;
    return rc;
  }
  *out = st;
  return RSFG_OK;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

__attribute__((visibility("default"))) const char* rsfg_last_error(void) { return g_err.c_str(); }
__attribute__((visibility("default"))) const char* rsfg_version(void) { return "rsfg 0.1 (sm_100a)"; }

__attribute__((visibility("default"))) void rsfg_params_default(rsfg_params* p) {
  if (!p) return;
  p->sigma1 = 5.0;  // rsf.hpp:14-22
  p->sigma2 = 0.0;
  p->alpha = 58.5225;
  p->beta = 0.1;
  p->epsilon = 1.0;
  p->dt = 0.06;
  p->max_iters = 100;
  p->convergence_fraction = 0.0;
  p->denom_floor = 1e-8;
  p->grad_floor = 1e-8;
}

__attribute__((visibility("default"))) void rsfg_options_default(rsfg_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->device = 0;
  o->fields = RSFG_FIELDS_2;
  o->check_every = 25;
  o->use_graphs = 1;
  o->reuse_workspace = 0;
}

__attribute__((visibility("default"))) int rsfg_params_validate(const rsfg_params* p) { return validate(p); }

__attribute__((visibility("default"))) int rsfg_gaussian_kernel(double sigma, double* weights, int32_t cap, int32_t* radius) {
  std::vector<double> w;
  if (int rc = gaussian(sigma, w)) return rc;
  if ((int)w.size() > cap) return fail(RSFG_ERR_PARAM, "weights buffer too small");
  std::memcpy(weights, w.data(), w.size() * sizeof(double));
  if (radius) *radius = (int32_t)(w.size() / 2);
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_state_create(rsfg_state** out, const float* phi0, const float* image, int32_t nx, int32_t ny,
                      int32_t nz, const rsfg_params* p, const rsfg_options* o) {
  if (!phi0 || !image) return fail(RSFG_ERR_STATE, "null input buffer");
  return create_common(out, phi0, image, nx, ny, nz, p, o, cudaMemcpyHostToDevice);
}

__attribute__((visibility("default"))) int rsfg_state_create_device(rsfg_state** out, const float* d_phi0, const float* d_image, int32_t nx,
                             int32_t ny, int32_t nz, const rsfg_params* p, const rsfg_options* o) {
  if (!d_phi0 || !d_image) return fail(RSFG_ERR_STATE, "null input buffer");
  return create_common(out, d_phi0, d_image, nx, ny, nz, p, o, cudaMemcpyDeviceToDevice);
}

__attribute__((visibility("default"))) int rsfg_state_step(rsfg_state* st, double* frac) {
  if (!st) return fail(RSFG_ERR_STATE, "null state");
  rsfg_slab* s = &st->e;
  if (int rc = step_interior(s)) return rc;
  if (int rc = step_finish(s, rsfg::kUpdate, s->phi[s->cur ^ 1])) return rc;
  long long sc = 0;
  int bad_it = 0;
  int rc = check_counters(s, 1, &sc, &bad_it);
  if (rc == RSFG_ERR_BLOWUP) {
    // rsf.cpp:346-353 throws before the swap: phi and iteration unchanged.
    s->cur ^= 1;
    s->hh_valid = false;
    s->iteration -= 1;
    s->slot = (s->slot + kSlots - 1) % kSlots;
    return rc;
  }
  if (rc) return rc;
  if (frac) *frac = (double)sc / ((double)s->nx * s->ny * s->nz);
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_state_run(rsfg_state* st, int32_t n, rsfg_report* rep) {
  if (!st) return fail(RSFG_ERR_STATE, "null state");
  rsfg_slab* s = &st->e;
  int done = 0, pending = 0;
  const long long l0 = s->launches;
  while (done < n) {
    if (int rc = step_interior(s)) return rc;
    if (int rc = step_finish(s, rsfg::kUpdate, s->phi[s->cur ^ 1])) return rc;
    ++done;
    ++pending;
    if (pending == s->check_every || done == n) {
      long long sc = 0;
      int bad_it = 0;
      int rc = check_counters(s, pending, &sc, &bad_it);
      pending = 0;
      if (rep) {
        rep->iterations = done;
        rep->last_sign_change_fraction = (double)sc / ((double)s->nx * s->ny * s->nz);
      }
      if (rc == RSFG_ERR_BLOWUP) {
        s->valid = false;
        if (rep) rep->blowup_iteration = bad_it;
        return rc;
      }
      if (rc) return rc;
    }
  }
  if (rep) rep->gpu_launches = s->launches - l0;
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_state_profile(rsfg_state* st, int32_t steps, double* ms) {
  if (!st || !ms || steps < 1) return fail(RSFG_ERR_STATE, "bad argument");
  rsfg_slab* s = &st->e;
  CUDA_TRY(cudaSetDevice(s->dev));
  std::vector<cudaEvent_t> ev(3 * (size_t)steps);
  for (auto& e : ev) CUDA_TRY(cudaEventCreate(&e));
  int rc = RSFG_OK;
  for (int i = 0; i < steps && !rc; ++i) {
    cudaEventRecord(ev[3 * i], s->stream);
    rc = step_interior(s);
    cudaEventRecord(ev[3 * i + 1], s->stream);
    if (!rc) rc = step_finish(s, rsfg::kUpdate, s->phi[s->cur ^ 1]);
    cudaEventRecord(ev[3 * i + 2], s->stream);
  }
  cudaStreamSynchronize(s->stream);
  ms[0] = ms[1] = 0.0;
  for (int i = 0; i < steps && !rc; ++i) {
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 1]);
    cudaEventElapsedTime(&b, ev[3 * i + 1], ev[3 * i + 2]);
    ms[0] += a / steps;
    ms[1] += b / steps;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  if (rc) return rc;
  long long sc = 0;
  int bad = 0;
  return check_counters(s, std::min(steps, kSlots), &sc, &bad);
}

__attribute__((visibility("default"))) const char* rsfg_profile_name(int32_t i) {
  static const char* names[] = {"xy: H-/H+ fields, K*x, K*y (rsf.cpp:75-94, ops.cpp:74-160)",
                                "zst: K*z, r+-, F- - F+, delta, grad/|grad|, div, lap, combine, update "
                                "(rsf.cpp:96-168, 324-352)"};
  return (i >= 0 && i < 2) ? names[i] : "";
}

// The reference's 14 stage rows (rsf.cpp:228-233) and which row carries each
// stage's time here (the kernels fuse them; kStage* above).
namespace {
const char* const kStageNames[RSFG_STAGE_COUNT] = {"H-I",  "H+I",      "K*H-I",     "K*H+I",       "K*H-",
                                                   "K*H+", "delta",    "grad",      "grad-mag",    "laplacian",
                                                   "grad/|grad|", "R-combine", "E+", "E-"};
const int kStageCarrier[RSFG_STAGE_COUNT] = {kStageH,    kStageH,       kStageConv,    kStageConv,   kStageConv,
                                             kStageConv, kStageCombine, kStageCombine, kStageCombine, kStageCombine,
                                             kStageCombine, kStageCombine, kStageCombine, kStageCombine};
}  // namespace

__attribute__((visibility("default"))) const char* rsfg_stage_name(int32_t i) {
  return (i >= 0 && i < RSFG_STAGE_COUNT) ? kStageNames[i] : "";
}

__attribute__((visibility("default"))) int32_t rsfg_stage_carrier(int32_t i) {
  return (i >= 0 && i < RSFG_STAGE_COUNT) ? kStageCarrier[i] : -1;
}

__attribute__((visibility("default"))) int rsfg_state_step_profiled(rsfg_state* st, double* frac, double* seconds) {
  if (!st || !seconds) return fail(RSFG_ERR_STATE, "null argument");
  rsfg_slab* s = &st->e;
  s->prof_used = 0;
  s->prof_on = true;
  int rc = rsfg_state_step(st, frac);
  s->prof_on = false;
  prof_collect(s, rc == RSFG_OK ? seconds : nullptr);
  return rc;
}

// evolve_step(state, I, p, ...) takes p every call (rsf.cpp:324-357): the
// scalar knobs (epsilon, alpha, beta, dt, floors) may change between steps;
// the kernels (sigma1, sigma2) are the state's own (st.k1/st.k2, rsf.cpp:299-300).
__attribute__((visibility("default"))) int rsfg_state_set_params(rsfg_state* st, const rsfg_params* p) {
  if (!st) return fail(RSFG_ERR_STATE, "null state");
  if (int rc = validate(p)) return rc;
  rsfg_slab* s = &st->e;
  const bool eps_changed = p->epsilon != s->p.epsilon;
  const double sig1 = s->p.sigma1, sig2 = s->p.sigma2;
  s->p = *p;
  s->p.sigma1 = sig1;
  s->p.sigma2 = sig2;
  const double eps = p->epsilon;
  s->c.inv_eps = (float)(1.0 / eps);
  s->c.c_delta = (float)((1.0 / M_PI) * eps);
  s->c.eps2 = (float)(eps * eps);
  s->c.alpha = (float)p->alpha;
  s->c.beta = (float)p->beta;
  s->c.denom_floor = (float)p->denom_floor;
  s->c.grad_floor = (float)p->grad_floor;
  s->c.inv_grad_floor = (float)(1.0 / p->grad_floor);
  s->c.dt = p->dt;
  s->c.dt_f = (float)p->dt;
  if (eps_changed) s->hh_valid = false;  // stored (H-, H- I) pairs used the old epsilon
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_state_energy(rsfg_state* st, float* E) {
  if (!st || !E) return fail(RSFG_ERR_STATE, "null argument");
  rsfg_slab* s = &st->e;
  if (int rc = step_interior(s)) return rc;
  if (int rc = step_finish(s, rsfg::kEnergy, s->phi[s->cur ^ 1])) return rc;
  CUDA_TRY(cudaMemcpyAsync(E, s->phi[s->cur ^ 1], s->held() * sizeof(float), cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_state_read_phi(rsfg_state* st, float* phi) {
  if (!st || !phi) return fail(RSFG_ERR_STATE, "null argument");
  rsfg_slab* s = &st->e;
  CUDA_TRY(cudaSetDevice(s->dev));
  CUDA_TRY(rsfg::copy_d2h(phi, s->phi[s->cur], s->held() * sizeof(float), s->stream));
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_state_write_phi(rsfg_state* st, const float* phi) {
  if (!st || !phi) return fail(RSFG_ERR_STATE, "null argument");
  rsfg_slab* s = &st->e;
  CUDA_TRY(cudaSetDevice(s->dev));
  CUDA_TRY(rsfg::copy_h2d(s->phi[s->cur], phi, s->held() * sizeof(float), s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  s->valid = true;
  s->hh_valid = false;
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_state_mask(rsfg_state* st, float* mask) {
  if (!st || !mask) return fail(RSFG_ERR_STATE, "null argument");
  rsfg_slab* s = &st->e;
  CUDA_TRY(cudaSetDevice(s->dev));
  float* tmp = reinterpret_cast<float*>(s->P[0]);
  s->launches += rsfg::launch_mask(s->phi[s->cur], tmp, (long long)s->held(), s->stream);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(mask, tmp, s->held() * sizeof(float), cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_state_iteration(const rsfg_state* st, int32_t* it) {
  if (!st || !it) return fail(RSFG_ERR_STATE, "null argument");
  *it = st->e.iteration;
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_state_device_phi(rsfg_state* st, float** d) {
  if (!st || !d) return fail(RSFG_ERR_STATE, "null argument");
  *d = st->e.phi[st->e.cur];
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_state_stream(rsfg_state* st, void** stream) {
  if (!st || !stream) return fail(RSFG_ERR_STATE, "null argument");
  *stream = (void*)st->e.stream;
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_state_sync(rsfg_state* st) {
  if (!st) return fail(RSFG_ERR_STATE, "null state");
  CUDA_TRY(cudaStreamSynchronize(st->e.stream));
  return RSFG_OK;
}

__attribute__((visibility("default"))) int64_t rsfg_state_launches(const rsfg_state* st) { return st ? st->e.launches : 0; }

__attribute__((visibility("default"))) int rsfg_state_variant(const rsfg_state* st, int32_t* flags, int32_t* xyb,
                                                               int32_t* zstb) {
  if (!st) return fail(RSFG_ERR_STATE, "null state");
  const rsfg_slab* s = &st->e;
  const int f = (s->fast && s->xy2maps[0].valid ? 1 : 0) | (s->fast && s->zmaps[0].valid ? 2 : 0) |
                (s->hh_mode ? 4 : 0);
  if (flags) *flags = f;
  // kernel 1: reads phi + I (or the stored pairs, 8 B either way), writes P
  // (8 B per field pair); kernel 2: reads P, phi, K2*I (+ K1*I for fields=2),
  // writes phi' (+ the 8-byte pairs in the stored-Heaviside mode).
  const int np = s->fields == 4 ? 2 : 1;
  if (xyb) *xyb = 8 + 8 * np;
  if (zstb) *zstb = 8 * np + 4 + 4 + (s->fields == 2 ? 4 : 0) + 4 + (s->hh_mode ? 8 : 0);
  return RSFG_OK;
}

__attribute__((visibility("default"))) void rsfg_state_destroy(rsfg_state* st) { destroy_state(st); }

// ------------------------------------------------------------------ evolve
namespace {
int evolve_impl(const float* image, float* phi, int nx, int ny, int nz, const rsfg_params* p,
                const rsfg_options* o, rsfg_stop_fn stop, void* user, int stop_every, rsfg_report* rep) {
  rsfg_report local{};
  if (!rep) rep = &local;
  std::memset(rep, 0, sizeof *rep);
  if (int rc = validate(p)) return rc;
  if (!image || !phi) return fail(RSFG_ERR_STATE, "null input buffer");
  rsfg_options opt;
  rsfg_options_default(&opt);
  if (o) opt = *o;
  cudaSetDevice(opt.device);
  cudaEvent_t ev[5];
  for (auto& e : ev) cudaEventCreate(&e);
  struct EvGuard {
    cudaEvent_t* ev;
    ~EvGuard() {
      for (int i = 0; i < 5; ++i) cudaEventDestroy(ev[i]);
    }
  } guard{ev};

  // Workspace reuse: the last evolve's device buffers stay with the calling
  // thread and serve the next call of the same shape/radii (no cudaMalloc,
  // stream or pinned-buffer setup on the hot e2e path).
  rsfg_state* st = nullptr;
  if (t_cache.st && !opt.reuse_workspace) {  // opt-out frees a kept workspace
    rsfg_state_destroy(t_cache.st);
    t_cache.st = nullptr;
  }
  if (opt.reuse_workspace && t_cache.st) {
    rsfg_slab* c = &t_cache.st->e;
    if (c->dev == opt.device && c->nx == nx && c->ny == ny && c->nz == nz && c->fields == opt.fields &&
        c->p.sigma1 == p->sigma1 && c->p.sigma2 == p->sigma2 && c->env_key == variant_env_key()) {
      st = t_cache.st;
      t_cache.st = nullptr;
      if (int rc = reconfigure(c, p, &opt)) {
        rsfg_state_destroy(st);
        return rc;
      }
    } else {
      rsfg_state_destroy(t_cache.st);
      t_cache.st = nullptr;
    }
  }
  const auto t_setup = std::chrono::steady_clock::now();
  if (!st) {
    st = new rsfg_state;
    st->e.pooled = true;
    if (int rc = setup(&st->e, nx, ny, nz, 0, nz, p, &opt)) {
      release(&st->e);
      delete st;
      return rc;
    }
  }
  rep->ms_setup = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_setup).count();
  rsfg_slab* s = &st->e;
  struct StGuard {
    rsfg_state* st;
    bool keep;
    ~StGuard() {
      if (keep && st->e.valid) {
        if (t_cache.st) rsfg_state_destroy(t_cache.st);
        t_cache.st = st;
      } else {
        rsfg_state_destroy(st);
      }
    }
  } sguard{st, opt.reuse_workspace != 0};
  // The image goes up first; phi0's upload then runs on a side stream under
  // the image range + static convolutions (which do not read phi), and the
  // loop waits for it.  ms_h2d is the image upload, ms_init the overlapped
  // init + phi0 upload.
  cudaStream_t side = nullptr;
  cudaEvent_t phi_up = nullptr;
  struct SideGuard {
    cudaStream_t* st;
    cudaEvent_t* e;
    ~SideGuard() {  // on every return path the copy from the caller's buffer is finished
      if (*st) cudaStreamSynchronize(*st), cudaStreamDestroy(*st);
      if (*e) cudaEventDestroy(*e);
    }
  } side_guard{&side, &phi_up};
  CUDA_TRY(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&phi_up, cudaEventDisableTiming));
  const size_t held_bytes = s->held() * sizeof(float);
  s->hh_valid = false;
  cudaEventRecord(ev[0], s->stream);
  CUDA_TRY(rsfg::copy_h2d(s->image, image, held_bytes, s->stream));
  cudaEventRecord(ev[1], s->stream);
  float lo, hi;
  if (int rc = local_range(s, &lo, &hi)) return rc;
  if (int rc = init_static(s, lo, hi)) return rc;
  CUDA_TRY(cudaStreamWaitEvent(side, ev[0], 0));  // after setup's memsets of phi[]
  CUDA_TRY(rsfg::copy_h2d(s->phi[s->cur], phi, held_bytes, side));
  CUDA_TRY(cudaEventRecord(phi_up, side));
  CUDA_TRY(cudaStreamWaitEvent(s->stream, phi_up, 0));
  cudaEventRecord(ev[2], s->stream);

  const bool per_step = p->convergence_fraction > 0.0;
  s->prof_used = 0;
  s->prof_on = opt.profile_stages != 0;  // KernelProfile* passed to evolve (rsf.cpp:359-384)
  struct ProfOff {
    rsfg_slab* s;
    ~ProfOff() { s->prof_on = false; }
  } prof_off{s};
  std::vector<float> host_phi;
  int pending = 0;
  const long long l0 = s->launches;
  for (int it = 0; it < p->max_iters; ++it) {
    if (int rc = step_interior(s)) return rc;
    if (int rc = step_finish(s, rsfg::kUpdate, s->phi[s->cur ^ 1])) return rc;
    ++pending;
    const bool want_stop = stop && stop_every > 0 && s->iteration % stop_every == 0;
    if (per_step || want_stop || pending == s->check_every || it + 1 == p->max_iters) {
      long long sc = 0;
      int bad_it = 0;
      int rc = check_counters(s, pending, &sc, &bad_it);
      prof_collect(s, rep->stage_seconds);
      pending = 0;
      rep->iterations = s->iteration;
      rep->last_sign_change_fraction = (double)sc / ((double)nx * ny * nz);
      if (rc == RSFG_ERR_BLOWUP) {
        rep->blowup_iteration = bad_it;
        std::sscanf(g_err.c_str(), "evolution produced a non-finite value at voxel (%d,%d,%d)", &rep->blowup_x,
                    &rep->blowup_y, &rep->blowup_z);
        return rc;
      }
      if (rc) return rc;
      // rsf.cpp:378: early stop on the sign-change fraction.
      if (per_step && rep->last_sign_change_fraction < p->convergence_fraction) break;
      // rsf.cpp:379-381: user stop callback with the current phi.
      if (want_stop) {
        host_phi.resize(s->held());
        if (int rc2 = rsfg_state_read_phi(st, host_phi.data())) return rc2;
        if (stop(host_phi.data(), nx, ny, nz, s->iteration, user)) break;
      }
    }
  }
  cudaEventRecord(ev[3], s->stream);
  CUDA_TRY(rsfg::copy_d2h(phi, s->phi[s->cur], s->held() * sizeof(float), s->stream));
  cudaEventRecord(ev[4], s->stream);
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  float ms;
  cudaEventElapsedTime(&ms, ev[0], ev[1]);
  rep->ms_h2d = ms;
  cudaEventElapsedTime(&ms, ev[1], ev[2]);
  rep->ms_init = ms;
  cudaEventElapsedTime(&ms, ev[2], ev[3]);
  rep->ms_loop = ms;
  cudaEventElapsedTime(&ms, ev[3], ev[4]);
  rep->ms_d2h = ms;
  rep->iterations = s->iteration;
  rep->gpu_launches = s->launches - l0;
  return RSFG_OK;
}

struct SliceStop {
  rsfg_stop_fn stop;
  void* user;
  std::vector<float> slice;
};

int slice_stop(const float* phi, int32_t nx, int32_t ny, int32_t, int32_t it, void* u) {
  auto* ss = static_cast<SliceStop*>(u);
  ss->slice.assign(phi, phi + (size_t)nx * ny);  // take_slice_z(phi, 0), rsf.cpp:368-369
  return ss->stop(ss->slice.data(), nx, ny, 1, it, ss->user);
}
}  // namespace

__attribute__((visibility("default"))) int rsfg_evolve(const float* image, float* phi, int32_t nx, int32_t ny, int32_t nz, const rsfg_params* p,
                const rsfg_options* o, rsfg_stop_fn stop, void* user, int32_t stop_every, rsfg_report* rep) {
  if (int rc = validate(p)) return rc;
  if (nz == 1) {
    // rsf.cpp:363-372: evolve a duplicated slice pair, return slice 0.
    if (!image || !phi) return fail(RSFG_ERR_STATE, "null input buffer");
    const size_t n = (size_t)nx * ny;
    std::vector<float> I2(2 * n), P2(2 * n);
    std::copy(image, image + n, I2.begin());
    std::copy(image, image + n, I2.begin() + n);
    std::copy(phi, phi + n, P2.begin());
    std::copy(phi, phi + n, P2.begin() + n);
    SliceStop ss{stop, user, {}};
    int rc = evolve_impl(I2.data(), P2.data(), nx, ny, 2, p, o, stop ? slice_stop : nullptr, &ss, stop_every, rep);
    if (rc) return rc;
    std::copy(P2.begin(), P2.begin() + n, phi);
    return RSFG_OK;
  }
  return evolve_impl(image, phi, nx, ny, nz, p, o, stop, user, stop_every, rep);
}

__attribute__((visibility("default"))) void rsfg_release_workspace(void) {
  rsfg_state_destroy(t_cache.st);
  t_cache.st = nullptr;
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (cudaMemPool_t p : g_pools)
    if (p) cudaMemPoolTrimTo(p, 0);  // cached workspace memory back to the device
}

__attribute__((visibility("default"))) int rsfg_extract_mask(const float* phi, float* mask, int64_t n, int32_t device) {
  if (n <= 0) return RSFG_OK;
  if (!phi || !mask) return fail(RSFG_ERR_STATE, "null argument");
  CUDA_TRY(cudaSetDevice(device));
  float *dp = nullptr, *dm = nullptr;
  cudaStream_t st;
  CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaError_t e = cudaMalloc(&dp, n * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&dm, n * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpyAsync(dp, phi, n * sizeof(float), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    rsfg::launch_mask(dp, dm, n, st);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(mask, dm, n * sizeof(float), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(dp);
  cudaFree(dm);
  cudaStreamDestroy(st);
  if (e != cudaSuccess) return fail(e == cudaErrorMemoryAllocation ? RSFG_ERR_OOM : RSFG_ERR_CUDA, cudaGetErrorString(e));
  return RSFG_OK;
}

// ------------------------------------------------------------------- slabs
__attribute__((visibility("default"))) int rsfg_slab_create(rsfg_slab** out, int32_t nx, int32_t ny, int32_t nz, int32_t z0, int32_t z1,
                     const rsfg_params* p, const rsfg_options* o) {
  if (!out) return fail(RSFG_ERR_STATE, "null output handle");
  *out = nullptr;
  auto* s = new rsfg_slab;
  if (int rc = setup(s, nx, ny, nz, z0, z1, p, o)) {
    std::string keep = g_err;
    release(s);
    delete s;
    g_err = keep;
    return rc;
  }
  *out = s;
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_slab_geometry(const rsfg_slab* s, int32_t* zb, int32_t* ze, int32_t* halo) {
  if (!s) return fail(RSFG_ERR_STATE, "null slab");
  if (zb) *zb = s->zb;
  if (ze) *ze = s->ze;
  if (halo) *halo = s->h;
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_slab_upload(rsfg_slab* s, const float* phi, const float* image) {
  if (!s || !phi || !image) return fail(RSFG_ERR_STATE, "null argument");
  if (int rc = upload(s, phi, image, cudaMemcpyHostToDevice)) return rc;
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_slab_upload_device(rsfg_slab* s, const float* phi, const float* image) {
  if (!s || !phi || !image) return fail(RSFG_ERR_STATE, "null argument");
  if (int rc = upload(s, phi, image, cudaMemcpyDeviceToDevice)) return rc;
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_slab_local_range(rsfg_slab* s, float* lo, float* hi) {
  if (!s || !lo || !hi) return fail(RSFG_ERR_STATE, "null argument");
  return local_range(s, lo, hi);
}

__attribute__((visibility("default"))) int rsfg_slab_init(rsfg_slab* s, float lo, float hi) {
  if (!s) return fail(RSFG_ERR_STATE, "null slab");
  return init_static(s, lo, hi);
}

__attribute__((visibility("default"))) int rsfg_slab_halo(rsfg_slab* s, int32_t side, void** send, void** recv, int64_t* bytes) {
  if (!s || !send || !recv || !bytes) return fail(RSFG_ERR_STATE, "null argument");
  const size_t plane = (size_t)s->nx * s->ny;
  float* cur = s->phi[s->cur];
  if (side == 0) {
    const int k = s->z0 - s->zb;  // halo planes below (0 on the global face)
    *recv = cur;
    *send = cur + s->off(s->z0);
    *bytes = (int64_t)k * plane * sizeof(float);
  } else {
    const int k = s->ze - s->z1;
    *recv = cur + s->off(s->z1);
    *send = cur + s->off(s->z1 - k);
    *bytes = (int64_t)k * plane * sizeof(float);
  }
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_slab_set_stream(rsfg_slab* s, void* stream) {
  if (!s) return fail(RSFG_ERR_STATE, "null slab");
  if (s->own_stream && s->stream) {
    CUDA_TRY(cudaStreamSynchronize(s->stream));
    cudaStreamDestroy(s->stream);
  }
  s->stream = (cudaStream_t)stream;
  s->own_stream = false;
  return RSFG_OK;
}

namespace {
int enable_peer(int from, int to);
}

__attribute__((visibility("default"))) int rsfg_slab_exchange(rsfg_slab* lo, rsfg_slab* hi) {
  if (!lo || !hi) return fail(RSFG_ERR_STATE, "null slab");
  if (lo->z1 != hi->z0 || lo->nx != hi->nx || lo->ny != hi->ny || lo->nz != hi->nz)
    return fail(RSFG_ERR_SHAPE, "slabs are not z-adjacent pieces of one volume");
  void *lo_send, *lo_recv, *hi_send, *hi_recv;
  int64_t lo_bytes, hi_bytes;
  rsfg_slab_halo(lo, 1, &lo_send, &lo_recv, &lo_bytes);
  rsfg_slab_halo(hi, 0, &hi_send, &hi_recv, &hi_bytes);
  if (lo_bytes != hi_bytes) return fail(RSFG_ERR_SHAPE, "halo sizes differ across the face");
  if (lo->dev != hi->dev) {  // direct NVLink copies instead of staging through the host
    if (int rc = enable_peer(lo->dev, hi->dev)) return rc;
    if (int rc = enable_peer(hi->dev, lo->dev)) return rc;
  }
  cudaEvent_t e_hi, e_lo;
  CUDA_TRY(cudaSetDevice(hi->dev));
  CUDA_TRY(cudaEventCreateWithFlags(&e_hi, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(e_hi, hi->stream));
  CUDA_TRY(cudaSetDevice(lo->dev));
  CUDA_TRY(cudaEventCreateWithFlags(&e_lo, cudaEventDisableTiming));
  CUDA_TRY(cudaStreamWaitEvent(lo->stream, e_hi, 0));
  CUDA_TRY(cudaMemcpyPeerAsync(hi_recv, hi->dev, lo_send, lo->dev, (size_t)lo_bytes, lo->stream));
  CUDA_TRY(cudaMemcpyPeerAsync(lo_recv, lo->dev, hi_send, hi->dev, (size_t)hi_bytes, lo->stream));
  CUDA_TRY(cudaEventRecord(e_lo, lo->stream));
  CUDA_TRY(cudaSetDevice(hi->dev));
  CUDA_TRY(cudaStreamWaitEvent(hi->stream, e_lo, 0));
  cudaEventDestroy(e_hi);
  cudaEventDestroy(e_lo);
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_slab_step_interior(rsfg_slab* s) {
  if (!s) return fail(RSFG_ERR_STATE, "null slab");
  return step_interior(s);
}

__attribute__((visibility("default"))) int rsfg_slab_step_finish(rsfg_slab* s) {
  if (!s) return fail(RSFG_ERR_STATE, "null slab");
  return step_finish(s, rsfg::kUpdate, s->phi[s->cur ^ 1]);
}

__attribute__((visibility("default"))) int rsfg_slab_counters(rsfg_slab* s, int64_t* sign_changes, int64_t* first_bad) {
  if (!s) return fail(RSFG_ERR_STATE, "null slab");
  const int sl = (s->slot + kSlots - 1) % kSlots;
  unsigned long long h[2];
  CUDA_TRY(cudaMemcpyAsync(h, s->counters + 2 * sl, sizeof h, cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  if (sign_changes) *sign_changes = (int64_t)h[0];
  if (first_bad) *first_bad = h[1] == ~0ull ? -1 : (int64_t)h[1];
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_slab_download(rsfg_slab* s, float* phi_owned) {
  if (!s || !phi_owned) return fail(RSFG_ERR_STATE, "null argument");
  CUDA_TRY(cudaSetDevice(s->dev));
  CUDA_TRY(rsfg::copy_d2h(phi_owned, s->phi[s->cur] + s->off(s->z0), s->owned() * sizeof(float), s->stream));
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_slab_device_phi(rsfg_slab* s, float** d) {
  if (!s || !d) return fail(RSFG_ERR_STATE, "null argument");
  *d = s->phi[s->cur];
  return RSFG_OK;
}

__attribute__((visibility("default"))) int64_t rsfg_slab_launches(const rsfg_slab* s) { return s ? s->launches : 0; }

__attribute__((visibility("default"))) void rsfg_slab_destroy(rsfg_slab* s) {
  if (!s) return;
  release(s);
  delete s;
}


// ------------------------------------------------------- peer halo links
namespace {
// What a neighbour needs to push into this slab: geometry, the two phi
// buffers and the flag words -- raw pointers (same process) or CUDA IPC
// handles (another process on this node).
struct PeerDesc {
  uint32_t magic, version;
  int32_t dev, nx, ny, nz, z0, z1, zb, ze, ipc, pad;
  uint64_t phi[2], flags;
  cudaIpcMemHandle_t h_phi[2], h_flags;
};
static_assert(sizeof(PeerDesc) <= RSFG_PEER_DESC_BYTES, "descriptor too large");
constexpr uint32_t kDescMagic = 0x52534647u;  // "RSFG"

using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValueFn wait_value_fn() {
  static WaitValueFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (WaitValueFn) nullptr;
    return reinterpret_cast<WaitValueFn>(f);
  }();
  return fn;
}

// The slab's stream waits until flags[side] >= v (halo of step v arrived).
int wait_flag(rsfg_slab* s, int side, unsigned int v) {
  static const bool no_memops = std::getenv("RSFG_NO_STREAM_MEMOPS") != nullptr;
  WaitValueFn fn = no_memops ? nullptr : wait_value_fn();
  if (fn && fn((CUstream)s->stream, (CUdeviceptr)(s->flags + side), v, CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS)
    return RSFG_OK;
  s->launches += rsfg::launch_flag_wait(s->flags + side, v, s->stream);
  CUDA_TRY(cudaGetLastError());
  return RSFG_OK;
}

int enable_peer(int from, int to) {
  if (from == to) return RSFG_OK;
  int can = 0;
  CUDA_TRY(cudaDeviceCanAccessPeer(&can, from, to));
  if (!can) return fail(RSFG_ERR_COMM, "no peer access from device " + std::to_string(from) + " to " + std::to_string(to));
  CUDA_TRY(cudaSetDevice(from));
  cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
  else if (e != cudaSuccess) return fail(RSFG_ERR_COMM, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
  return RSFG_OK;
}

// One step with linked faces: interior xy work, wait for the halos of this
// step, finish (kernel 2 -> phi'), then push the new boundary planes into the
// neighbours' halos and bump their flags on a side stream that overlaps the
// next step's interior work.
int step_linked(rsfg_slab* s) {
  if (int rc = step_interior(s)) return rc;
  const unsigned int it = (unsigned int)s->iteration;
  for (int side = 0; side < 2; ++side)
    if (s->link[side].on)
      if (int rc = wait_flag(s, side, it)) return rc;
  // the previous push read the buffer this step's successor will overwrite
  if (s->push_pending) CUDA_TRY(cudaStreamWaitEvent(s->stream, s->push_done, 0));
  if (int rc = step_finish(s, rsfg::kUpdate, s->phi[s->cur ^ 1])) return rc;
  if (!s->link[0].on && !s->link[1].on) return RSFG_OK;
  CUDA_TRY(cudaEventRecord(s->k2_done, s->stream));
  CUDA_TRY(cudaStreamWaitEvent(s->push_stream, s->k2_done, 0));
  for (int side = 0; side < 2; ++side) {
    const rsfg_slab::Link& L = s->link[side];
    if (!L.on) continue;
    CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<char*>(L.phi[s->cur]) + L.dst_off,
                             reinterpret_cast<const char*>(s->phi[s->cur]) + L.src_off, L.bytes, cudaMemcpyDefault,
                             s->push_stream));
    s->launches += rsfg::launch_flag_store(L.flag, (unsigned int)s->iteration, s->push_stream);
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventRecord(s->push_done, s->push_stream));
  s->push_pending = true;
  return RSFG_OK;
}

// Counters of the last k steps without formatting: sign changes of the last
// step, the earliest (1-based) iteration with a non-finite value and its
// smallest global index (0 / -1 if none).
int read_counters(rsfg_slab* s, int k, long long* last_sc, int* bad_it, long long* bad_idx) {
  CUDA_TRY(cudaSetDevice(s->dev));
  CUDA_TRY(cudaMemcpyAsync(s->h_counters, s->counters, kSlots * 2 * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, s->stream));
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  *bad_it = 0;
  *bad_idx = -1;
  for (int i = k; i >= 1; --i) {
    const int sl = ((s->slot - i) % kSlots + kSlots) % kSlots;
    if (i == 1) *last_sc = (long long)s->h_counters[2 * sl];
    const unsigned long long bad = s->h_counters[2 * sl + 1];
    if (bad != ~0ull && *bad_it == 0) {
      *bad_it = s->iteration - i + 1;
      *bad_idx = (long long)bad;
    }
  }
  return RSFG_OK;
}
}  // namespace

__attribute__((visibility("default"))) int rsfg_slab_peer_desc(rsfg_slab* s, void* desc, int32_t ipc) {
  if (!s || !desc) return fail(RSFG_ERR_STATE, "null argument");
  PeerDesc d{};
  d.magic = kDescMagic;
  d.version = 1;
  d.dev = s->dev;
  d.nx = s->nx, d.ny = s->ny, d.nz = s->nz, d.z0 = s->z0, d.z1 = s->z1, d.zb = s->zb, d.ze = s->ze;
  d.ipc = ipc ? 1 : 0;
  d.phi[0] = (uint64_t)(uintptr_t)s->phi[0];
  d.phi[1] = (uint64_t)(uintptr_t)s->phi[1];
  d.flags = (uint64_t)(uintptr_t)s->flags;
  if (ipc) {
    CUDA_TRY(cudaSetDevice(s->dev));
    CUDA_TRY(cudaIpcGetMemHandle(&d.h_phi[0], s->phi[0]));
    CUDA_TRY(cudaIpcGetMemHandle(&d.h_phi[1], s->phi[1]));
    CUDA_TRY(cudaIpcGetMemHandle(&d.h_flags, s->flags));
  }
  std::memset(desc, 0, RSFG_PEER_DESC_BYTES);
  std::memcpy(desc, &d, sizeof d);
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_slab_link(rsfg_slab* s, int32_t side, const void* desc) {
  if (!s || !desc || (side != 0 && side != 1)) return fail(RSFG_ERR_STATE, "bad argument");
  PeerDesc d;
  std::memcpy(&d, desc, sizeof d);
  if (d.magic != kDescMagic || d.version != 1) return fail(RSFG_ERR_STATE, "not a peer descriptor");
  if (d.nx != s->nx || d.ny != s->ny || d.nz != s->nz || (side == 0 ? d.z1 != s->z0 : d.z0 != s->z1))
    return fail(RSFG_ERR_SHAPE, "peer slab is not the z-neighbour on that face");
  rsfg_slab::Link& L = s->link[side];
  if (L.on) return fail(RSFG_ERR_STATE, "face already linked");
  CUDA_TRY(cudaSetDevice(s->dev));
  if (d.ipc) {
    void* p[3];
    const cudaIpcMemHandle_t* h[3] = {&d.h_phi[0], &d.h_phi[1], &d.h_flags};
    for (int i = 0; i < 3; ++i) {
      cudaError_t e = cudaIpcOpenMemHandle(&p[i], *h[i], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        for (int j = 0; j < i; ++j) cudaIpcCloseMemHandle(p[j]);
        return fail(RSFG_ERR_COMM, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
      }
      L.ipc_base[i] = p[i];
    }
    L.phi[0] = static_cast<float*>(p[0]);
    L.phi[1] = static_cast<float*>(p[1]);
    L.flag = static_cast<unsigned int*>(p[2]);
    L.ipc = true;
  } else {
    if (int rc = enable_peer(s->dev, d.dev)) return rc;
    CUDA_TRY(cudaSetDevice(s->dev));
    L.phi[0] = reinterpret_cast<float*>((uintptr_t)d.phi[0]);
    L.phi[1] = reinterpret_cast<float*>((uintptr_t)d.phi[1]);
    L.flag = reinterpret_cast<unsigned int*>((uintptr_t)d.flags);
  }
  const size_t plane = (size_t)s->nx * s->ny * sizeof(float);
  if (side == 1) {  // neighbour above: its halo planes [d.zb, d.z0) are our owned planes
    L.flag += 0;    // it receives on its side 0
    L.src_off = s->off(d.zb) * sizeof(float);
    L.dst_off = 0;
    L.bytes = (size_t)(d.z0 - d.zb) * plane;
  } else {          // neighbour below: its halo planes [d.z1, d.ze)
    L.flag += 1;
    L.src_off = s->off(s->z0) * sizeof(float);
    L.dst_off = (size_t)(d.z1 - d.zb) * plane;
    L.bytes = (size_t)(d.ze - d.z1) * plane;
  }
  if (d.zb < s->zb && side == 1) return fail(RSFG_ERR_SHAPE, "neighbour halo exceeds this slab");
  L.peer_dev = d.dev;
  L.on = true;
  if (!s->push_stream) {
    CUDA_TRY(cudaStreamCreateWithFlags(&s->push_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&s->k2_done, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&s->push_done, cudaEventDisableTiming));
  }
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_slab_step_linked(rsfg_slab* s) {
  if (!s) return fail(RSFG_ERR_STATE, "null slab");
  return step_linked(s);
}

// rsf::evolve over several GPUs of this process: z-slabs on
// devices[0..n), halos pushed over peer memory (NVLink) every step; bitwise
// equal to rsfg_evolve on one device.
__attribute__((visibility("default"))) int rsfg_evolve_multi(const float* image, float* phi, int32_t nx, int32_t ny,
                                                             int32_t nz, const rsfg_params* p, const rsfg_options* o,
                                                             const int32_t* devices, int32_t n_devices,
                                                             rsfg_stop_fn stop, void* user, int32_t stop_every,
                                                             rsfg_report* rep) {
  rsfg_report local{};
  if (!rep) rep = &local;
  std::memset(rep, 0, sizeof *rep);
  if (int rc = validate(p)) return rc;
  if (!image || !phi || !devices || n_devices < 1) return fail(RSFG_ERR_STATE, "null argument");
  rsfg_options opt;
  rsfg_options_default(&opt);
  if (o) opt = *o;
  if (n_devices == 1 || nz == 1) {
    opt.device = devices[0];
    return rsfg_evolve(image, phi, nx, ny, nz, p, &opt, stop, user, stop_every, rep);
  }
  rsfg::Taps t1, t2;
  if (int rc = make_taps(p->sigma1, t1)) return rc;
  if (int rc = make_taps(p->sigma2, t2)) return rc;
  const int h = std::max(std::max(t1.r, t2.r), 2);
  const int n = n_devices;
  if (nz / n < h)
    return fail(RSFG_ERR_SHAPE, "nz=" + std::to_string(nz) + " over " + std::to_string(n) +
                                    " slabs leaves a slab thinner than the halo (" + std::to_string(h) + ")");
  std::vector<rsfg_slab*> sl(n, nullptr);
  struct Guard {
    std::vector<rsfg_slab*>& v;
    ~Guard() {
      for (rsfg_slab* s : v)
        if (s) release(s), delete s;
    }
  } guard{sl};
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const size_t plane = (size_t)nx * ny;
  int z = 0;
  for (int i = 0; i < n; ++i) {  // balanced ranges (spmd.plan_slabs)
    const int cnt = nz / n + (i < nz % n ? 1 : 0);
    rsfg_options oi = opt;
    oi.device = devices[i];
    sl[i] = new rsfg_slab;
    if (int rc = setup(sl[i], nx, ny, nz, z, z + cnt, p, &oi)) return rc;
    if (int rc = upload(sl[i], phi + (size_t)sl[i]->zb * plane, image + (size_t)sl[i]->zb * plane,
                        cudaMemcpyHostToDevice))
      return rc;
    z += cnt;
  }
  float lo = 0.f, hi = 0.f;
  for (int i = 0; i < n; ++i) {
    float a, b;
    if (int rc = local_range(sl[i], &a, &b)) return rc;
    lo = i ? std::min(lo, a) : a;
    hi = i ? std::max(hi, b) : b;
  }
  const auto t1c = clk::now();
  for (int i = 0; i < n; ++i)
    if (int rc = init_static(sl[i], lo, hi)) return rc;
  char desc[RSFG_PEER_DESC_BYTES];
  for (int i = 0; i < n; ++i) {
    if (i > 0) {
      if (int rc = rsfg_slab_peer_desc(sl[i - 1], desc, 0)) return rc;
      if (int rc = rsfg_slab_link(sl[i], 0, desc)) return rc;
    }
    if (i + 1 < n) {
      if (int rc = rsfg_slab_peer_desc(sl[i + 1], desc, 0)) return rc;
      if (int rc = rsfg_slab_link(sl[i], 1, desc)) return rc;
    }
  }
  for (int i = 0; i < n; ++i) CUDA_TRY(cudaStreamSynchronize(sl[i]->stream));
  const auto t2c = clk::now();
  const bool per_step = p->convergence_fraction > 0.0;
  const int check_every = sl[0]->check_every;
  long long l0 = 0;
  for (rsfg_slab* s : sl) l0 += s->launches;
  int pending = 0;
  std::vector<float> host_phi;
  for (int it = 0; it < p->max_iters; ++it) {
    for (rsfg_slab* s : sl)
      if (int rc = step_linked(s)) return rc;
    ++pending;
    const bool want_stop = stop && stop_every > 0 && (it + 1) % stop_every == 0;
    if (per_step || want_stop || pending == check_every || it + 1 == p->max_iters) {
      long long sc_all = 0, best_idx = -1;
      int best_it = 0;
      for (rsfg_slab* s : sl) {
        long long sc = 0, bidx = -1;
        int bit = 0;
        if (int rc = read_counters(s, pending, &sc, &bit, &bidx)) return rc;
        sc_all += sc;
        if (bit && (!best_it || bit < best_it || (bit == best_it && bidx < best_idx))) best_it = bit, best_idx = bidx;
      }
      pending = 0;
      rep->iterations = it + 1;
      rep->last_sign_change_fraction = (double)sc_all / ((double)nx * ny * nz);
      if (best_it) {
        const int x = (int)(best_idx % nx), y = (int)((best_idx / nx) % ny), zz = (int)(best_idx / (long long)plane);
        char buf[160];
        snprintf(buf, sizeof buf, "evolution produced a non-finite value at voxel (%d,%d,%d), iteration %d", x, y, zz,
                 best_it);
        rep->blowup_iteration = best_it;
        rep->blowup_x = x, rep->blowup_y = y, rep->blowup_z = zz;
        return fail(RSFG_ERR_BLOWUP, buf);
      }
      if (per_step && rep->last_sign_change_fraction < p->convergence_fraction) break;  // rsf.cpp:378
      if (want_stop) {  // rsf.cpp:379-381: StopCheck with the whole volume's current phi
        host_phi.resize((size_t)nx * ny * nz);
        for (rsfg_slab* s : sl) {
          CUDA_TRY(cudaSetDevice(s->dev));
          CUDA_TRY(rsfg::copy_d2h(host_phi.data() + (size_t)s->z0 * plane, s->phi[s->cur] + s->off(s->z0),
                                  s->owned() * sizeof(float), s->stream));
        }
        if (stop(host_phi.data(), nx, ny, nz, it + 1, user)) break;
      }
    }
  }
  for (rsfg_slab* s : sl) CUDA_TRY(cudaStreamSynchronize(s->stream));
  const auto t3c = clk::now();
  for (rsfg_slab* s : sl) {
    CUDA_TRY(cudaSetDevice(s->dev));
    CUDA_TRY(rsfg::copy_d2h(phi + (size_t)s->z0 * plane, s->phi[s->cur] + s->off(s->z0), s->owned() * sizeof(float),
                            s->stream));
  }
  const auto t4c = clk::now();
  auto ms = [](clk::duration d) { return std::chrono::duration<double, std::milli>(d).count(); };
  rep->ms_h2d = ms(t1c - t0);
  rep->ms_init = ms(t2c - t1c);
  rep->ms_loop = ms(t3c - t2c);
  rep->ms_d2h = ms(t4c - t3c);
  long long l1 = 0;
  for (rsfg_slab* s : sl) l1 += s->launches;
  rep->gpu_launches = l1 - l0;
  return RSFG_OK;
}

__attribute__((visibility("default"))) void rsfg_blob_params_default(rsfg_blob_params* b) {
  if (!b) return;
  b->sigma_b = 3.0;  // seeding.hpp:13-16
  b->response_threshold = 0.1;
  b->nms_radius = 0.0;
  b->dark = 0;
}

__attribute__((visibility("default"))) int rsfg_init_phi_device(const float* d_image, int32_t nx, int32_t ny,
                                                                int32_t nz, const rsfg_blob_params* bp,
                                                                double seed_radius, float* d_phi0, int32_t device,
                                                                int32_t* n_seeds, int32_t* seeds_xyz,
                                                                float* seeds_resp, int32_t cap,
                                                                int32_t* iterations) {
  rsfg_blob_params b;
  rsfg_blob_params_default(&b);
  if (bp) b = *bp;
  if (!d_image || !d_phi0) return fail(RSFG_ERR_STATE, "init_phi: null buffer");
  // BlobParams::validate (seeding.cpp:13-19), init_phi (seeding.cpp:223)
  if (!(b.sigma_b > 0.0)) return fail(RSFG_ERR_PARAM, "BlobParams: sigma_b must be > 0");
  if (b.response_threshold < 0.0) return fail(RSFG_ERR_PARAM, "BlobParams: response_threshold must be >= 0");
  const double nms = b.nms_radius > 0.0 ? b.nms_radius : 2.0 * b.sigma_b;
  if (nms < 1.0) return fail(RSFG_ERR_PARAM, "BlobParams: nms_radius must be >= 1");
  if (seed_radius < 0.0) return fail(RSFG_ERR_PARAM, "init_phi: seed_radius must be >= 0");
  if (nx <= 0 || ny <= 0 || nz <= 0) return fail(RSFG_ERR_SHAPE, "volume dims must be positive");
  if (nx < 5 || ny < 5) return fail(RSFG_ERR_SHAPE, "hessian_det_slice: slice must be at least 5x5");
  CUDA_TRY(cudaSetDevice(device));
  cudaStream_t st;
  CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  std::vector<rsfg::SeedHost> seeds;
  long long nl = 0;
  int rc = rsfg::seed_detect(d_image, nx, ny, nz, b.sigma_b, b.response_threshold, nms, b.dark != 0, seeds, st, &nl);
  int it = 0;
  if (!rc && !seeds.empty()) rc = rsfg::seed_distance(nx, ny, nz, seeds, (float)seed_radius, d_phi0, st, &it, &nl);
  cudaStreamDestroy(st);
  if (rc == -2) return fail(RSFG_ERR_OOM, "init_phi: out of device memory");
  if (rc == -3) return fail(RSFG_ERR_PARAM, "init_phi: too many seed candidates");
  if (rc) return fail(RSFG_ERR_CUDA, std::string("init_phi: CUDA error: ") + cudaGetErrorString(cudaGetLastError()));
  if (n_seeds) *n_seeds = (int32_t)seeds.size();
  for (size_t k = 0; k < seeds.size() && (int32_t)k < cap; ++k) {
    if (seeds_xyz) {
      seeds_xyz[3 * k] = seeds[k].x;
      seeds_xyz[3 * k + 1] = seeds[k].y;
      seeds_xyz[3 * k + 2] = seeds[k].z;
    }
    if (seeds_resp) seeds_resp[k] = seeds[k].response;
  }
  if (iterations) *iterations = it;
  if (seeds.empty())
    return fail(RSFG_ERR_PARAM,
                "init_phi: no seeds detected; lower response_threshold (or adjust sigma_b) and retry");
  return RSFG_OK;
}

// rsf::init_phi with HOST buffers (seeding.cpp:221-235): the image goes up,
// seeding and the distance run on the device, phi0 comes back.
__attribute__((visibility("default"))) int rsfg_init_phi(const float* image, int32_t nx, int32_t ny, int32_t nz,
                                                         const rsfg_blob_params* bp, double seed_radius,
                                                         float* phi0, int32_t device, int32_t* n_seeds,
                                                         int32_t* seeds_xyz, float* seeds_resp, int32_t cap,
                                                         int32_t* iterations) {
  if (!image || !phi0) return fail(RSFG_ERR_STATE, "init_phi: null buffer");
  if (nx <= 0 || ny <= 0 || nz <= 0) return fail(RSFG_ERR_SHAPE, "volume dims must be positive");
  CUDA_TRY(cudaSetDevice(device));
  const size_t bytes = (size_t)nx * ny * nz * sizeof(float);
  float* d_img = nullptr;
  float* d_phi = nullptr;
  if (cudaMalloc(&d_img, bytes) != cudaSuccess || cudaMalloc(&d_phi, bytes) != cudaSuccess) {
    cudaFree(d_img);
    cudaFree(d_phi);
    return fail(RSFG_ERR_OOM, "init_phi: out of device memory");
  }
  int rc = RSFG_OK;
  if (cudaMemcpy(d_img, image, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
    rc = fail(RSFG_ERR_CUDA, "init_phi: upload failed");
  if (!rc)
    rc = rsfg_init_phi_device(d_img, nx, ny, nz, bp, seed_radius, d_phi, device, n_seeds, seeds_xyz, seeds_resp,
                              cap, iterations);
  if (!rc && cudaMemcpy(phi0, d_phi, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = fail(RSFG_ERR_CUDA, "init_phi: download failed");
  cudaFree(d_img);
  cudaFree(d_phi);
  return rc;
}

}  // extern "C"
