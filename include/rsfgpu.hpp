// rsfgpu.hpp -- header-only C++ wrapper over the C-ABI (rsfg.h) with the
// reference's exact C++ surface: the same function names, argument meaning,
// defaults and exception types as /root/reference/proj/include/rsf/rsf.hpp
// (RsfParams, evolve, init_evolution, evolve_step, energy, extract_mask) and
// of seeding.hpp / tiling.hpp (BlobParams, init_phi, plan_tiles,
// run_pipeline) in namespace rsfgpu.  A caller of rsf::evolve switches by changing the
// namespace (and linking librsfg.so); see INTEGRATION.md.
#pragma once

#include <algorithm>
#include <array>
#include <cstddef>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "rsfg.h"

namespace rsfgpu {

// Exception types mirroring rsf::param_error / shape_error / blowup_error
// (reference core.hpp:11-32).
class param_error : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class shape_error : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class blowup_error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class cuda_error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class io_error : public std::runtime_error {  // rsf::io_error (core.hpp:23-26)
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == RSFG_OK) return;
  const std::string msg = rsfg_last_error();
  switch (rc) {
    case RSFG_ERR_PARAM: throw param_error(msg);
    case RSFG_ERR_SHAPE: throw shape_error(msg);
    case RSFG_ERR_BLOWUP: throw blowup_error(msg);
    case RSFG_ERR_IO: throw io_error(msg);
    default: throw cuda_error(msg);
  }
}

struct Dims {
  int nx = 0, ny = 0, nz = 0;
  std::size_t voxels() const { return (std::size_t)nx * ny * nz; }
  bool operator==(const Dims& o) const { return nx == o.nx && ny == o.ny && nz == o.nz; }
};

// rsf::Volume subset: dims + x-fastest fp32 data (volume.hpp:23-54).
struct Volume {
  Dims dims;
  std::vector<float> data;
  Volume() = default;
  Volume(int nx, int ny, int nz, float fill = 0.0f) : dims{nx, ny, nz}, data(dims.voxels(), fill) {}
  std::size_t voxels() const { return dims.voxels(); }
};

// rsf::RsfParams (rsf.hpp:13-26), same defaults.
struct RsfParams {
  double sigma1 = 5.0;
  double sigma2 = 0.0;
  double alpha = 58.5225;
  double beta = 0.1;
  double epsilon = 1.0;
  double dt = 0.06;
  int max_iters = 100;
  double convergence_fraction = 0.0;
  double denom_floor = 1e-8;
  double grad_floor = 1e-8;

  rsfg_params c() const {
    return rsfg_params{sigma1, sigma2, alpha, beta, epsilon, dt, max_iters, convergence_fraction,
                       denom_floor, grad_floor};
  }
  void validate() const {
    const rsfg_params p = c();
    check(rsfg_params_validate(&p));
  }
};

using StopCheck = std::function<bool(const Volume& phi, int iteration)>;

inline void check_same_dims(const Volume& a, const Volume& b, const char* what) {
  if (!(a.dims == b.dims))
    throw shape_error(std::string(what) + ": dims mismatch " + std::to_string(a.dims.nx) + "x" +
                      std::to_string(a.dims.ny) + "x" + std::to_string(a.dims.nz) + " vs " +
                      std::to_string(b.dims.nx) + "x" + std::to_string(b.dims.ny) + "x" +
                      std::to_string(b.dims.nz));
}

inline std::string to_string(const Dims& d) {  // core.hpp:46-48
  return std::to_string(d.nx) + "x" + std::to_string(d.ny) + "x" + std::to_string(d.nz);
}

// rsf::replicate_z / take_slice_z (volume.hpp:78-79, volume.cpp:47-67).
inline Volume replicate_z(const Volume& v) {
  if (v.dims.nz != 1) throw shape_error("replicate_z: expects nz == 1");
  Volume out(v.dims.nx, v.dims.ny, 2);
  std::copy(v.data.begin(), v.data.end(), out.data.begin());
  std::copy(v.data.begin(), v.data.end(), out.data.begin() + (std::ptrdiff_t)v.voxels());
  return out;
}
inline Volume take_slice_z(const Volume& v, int z) {
  if (z < 0 || z >= v.dims.nz) throw shape_error("take_slice_z: z out of range");
  Volume out(v.dims.nx, v.dims.ny, 1);
  const std::size_t n = out.voxels();
  std::copy(v.data.begin() + (std::ptrdiff_t)(n * z), v.data.begin() + (std::ptrdiff_t)(n * (z + 1)),
            out.data.begin());
  return out;
}

// Worker count (core.hpp:50-60).  The reference's OpenMP width has no GPU
// meaning: every call runs on one device stream, results never depend on it.
inline void set_worker_count(int) {}
inline int worker_count() { return 1; }
namespace detail {
inline int effective_workers() { return 1; }
}  // namespace detail

// rsf::KernelProfile (rsf.hpp:64-69): the reference's 14 stage rows
// (rsf.cpp:228-233).  Filled from per-kernel CUDA events; the kernels fuse
// stages, so each kernel's time lands on one row and the rows fused into it
// stay 0 (rsfg.h, RSFG_STAGE_COUNT; carrier(i) names the row).
struct KernelProfile {
  static constexpr int kCount = RSFG_STAGE_COUNT;
  static const std::array<const char*, kCount>& names() {
    static const std::array<const char*, kCount> n = [] {
      std::array<const char*, kCount> a{};
      for (int i = 0; i < kCount; ++i) a[i] = rsfg_stage_name(i);
      return a;
    }();
    return n;
  }
  static int carrier(int i) { return rsfg_stage_carrier(i); }
  std::array<double, kCount> seconds{};
  long iterations = 0;
};

// rsf::EvolveWorkspace (rsf.hpp:72-77): the scratch fields live on the device
// inside the EvolutionState; kept so evolve_step has the reference signature.
struct EvolveWorkspace {};

// rsf::evolve (rsf.hpp:97-98), same signature; `options` (appended) selects
// the device and the convolution form (RSFG_FIELDS_2 default, RSFG_FIELDS_4
// the reference form).
inline Volume evolve(Volume phi0, const Volume& I, const RsfParams& p, StopCheck stop = nullptr,
                     int stop_every = 25, KernelProfile* profile = nullptr, const rsfg_options* options = nullptr) {
  p.validate();
  check_same_dims(phi0, I, "evolve");
  const rsfg_params cp = p.c();
  rsfg_options o;
  rsfg_options_default(&o);
  if (options) o = *options;
  o.profile_stages = profile ? 1 : 0;
  struct Ctx {
    StopCheck* stop;
  } ctx{&stop};
  auto tramp = [](const float* phi, int32_t nx, int32_t ny, int32_t nz, int32_t it, void* u) -> int {
    auto* c = static_cast<Ctx*>(u);
    Volume v(nx, ny, nz);
    std::memcpy(v.data.data(), phi, v.voxels() * sizeof(float));
    return (*c->stop)(v, it) ? 1 : 0;
  };
  rsfg_report rep{};
  check(rsfg_evolve(I.data.data(), phi0.data.data(), I.dims.nx, I.dims.ny, I.dims.nz, &cp, &o,
                    stop ? +tramp : nullptr, &ctx, stop_every, &rep));
  if (profile) {
    for (int k = 0; k < KernelProfile::kCount; ++k) profile->seconds[k] += rep.stage_seconds[k];
    profile->iterations += rep.iterations;
  }
  return phi0;
}

// rsf::evolve over several GPUs of this process (rsfg_evolve_multi): z-slabs
// on `devices` with their halos pushed over NVLink peer memory every step;
// bitwise equal to evolve() on one GPU; same StopCheck semantics.
inline Volume evolve_multi(Volume phi0, const Volume& I, const RsfParams& p, const std::vector<int>& devices,
                           StopCheck stop = nullptr, int stop_every = 25, const rsfg_options* options = nullptr) {
  p.validate();
  check_same_dims(phi0, I, "evolve");
  if (devices.empty()) throw param_error("evolve_multi: no devices");
  const rsfg_params cp = p.c();
  std::vector<int32_t> dv(devices.begin(), devices.end());
  struct Ctx {
    StopCheck* stop;
  } ctx{&stop};
  auto tramp = [](const float* phi, int32_t nx, int32_t ny, int32_t nz, int32_t it, void* u) -> int {
    auto* c = static_cast<Ctx*>(u);
    Volume v(nx, ny, nz);
    std::memcpy(v.data.data(), phi, v.voxels() * sizeof(float));
    return (*c->stop)(v, it) ? 1 : 0;
  };
  check(rsfg_evolve_multi(I.data.data(), phi0.data.data(), I.dims.nx, I.dims.ny, I.dims.nz, &cp, options, dv.data(),
                          (int32_t)dv.size(), stop ? +tramp : nullptr, &ctx, stop_every, nullptr));
  return phi0;
}

// rsf::extract_mask (rsf.hpp:101).
inline Volume extract_mask(const Volume& phi, int device = 0) {
  Volume m(phi.dims.nx, phi.dims.ny, phi.dims.nz);
  check(rsfg_extract_mask(phi.data.data(), m.data.data(), (int64_t)phi.voxels(), device));
  return m;
}

// rsf::EvolutionState + init_evolution / evolve_step / energy (rsf.hpp:54-88),
// with the state resident on the GPU (phi, K1*I / K2*I, the kernels, the
// image range).  phi() downloads the current level set.
class EvolutionState {
 public:
  EvolutionState(const Volume& phi0, const Volume& I, const RsfParams& p,
                 const rsfg_options* options = nullptr)
      : dims_(phi0.dims), p_(p) {
    check_same_dims(phi0, I, "init_evolution");
    const rsfg_params cp = p.c();
    check(rsfg_state_create(&s_, phi0.data.data(), I.data.data(), dims_.nx, dims_.ny, dims_.nz, &cp, options));
  }
  EvolutionState(const EvolutionState&) = delete;
  EvolutionState& operator=(const EvolutionState&) = delete;
  EvolutionState(EvolutionState&& o) noexcept : s_(o.s_), dims_(o.dims_), p_(o.p_) { o.s_ = nullptr; }
  ~EvolutionState() { rsfg_state_destroy(s_); }

  int iteration() const {
    int32_t it = 0;
    check(rsfg_state_iteration(s_, &it));
    return it;
  }
  Volume phi() const {
    Volume v(dims_.nx, dims_.ny, dims_.nz);
    check(rsfg_state_read_phi(s_, v.data.data()));
    return v;
  }
  const Dims& dims() const { return dims_; }
  rsfg_state* handle() const { return s_; }

 private:
  // evolve_step takes p on every call (rsf.cpp:324-357): push changed scalars.
  void sync_params(const RsfParams& p) {
    if (p.epsilon == p_.epsilon && p.alpha == p_.alpha && p.beta == p_.beta && p.dt == p_.dt &&
        p.denom_floor == p_.denom_floor && p.grad_floor == p_.grad_floor)
      return;
    const rsfg_params cp = p.c();
    check(rsfg_state_set_params(s_, &cp));
    const double s1 = p_.sigma1, s2 = p_.sigma2;
    p_ = p;
    p_.sigma1 = s1;
    p_.sigma2 = s2;
  }
  friend double evolve_step(EvolutionState&, const Volume&, const RsfParams&, EvolveWorkspace&, KernelProfile*);
  friend Volume energy(const EvolutionState&, const Volume&, const RsfParams&);
  rsfg_state* s_ = nullptr;
  Dims dims_;
  RsfParams p_;
};

// rsf::init_evolution (rsf.hpp:79): phi0 by value, like the reference.
inline EvolutionState init_evolution(Volume phi0, const Volume& I, const RsfParams& p,
                                     const rsfg_options* options = nullptr) {
  p.validate();
  return EvolutionState(phi0, I, p, options);
}

// rsf::evolve_step (rsf.hpp:87-88), same signature.  I must be the image the
// state was initialised with (its device copy is used); p's scalars apply to
// this step, sigma stays the state's (st.k1/st.k2, rsf.cpp:299-300).
inline double evolve_step(EvolutionState& st, const Volume& I, const RsfParams& p, EvolveWorkspace& ws,
                          KernelProfile* profile = nullptr) {
  (void)ws;
  if (!(I.dims == st.dims_)) throw shape_error("evolve_step: image dims differ from the state's");
  st.sync_params(p);
  double frac = 0.0;
  if (profile) {
    double secs[RSFG_STAGE_COUNT] = {};
    check(rsfg_state_step_profiled(st.s_, &frac, secs));
    for (int k = 0; k < KernelProfile::kCount; ++k) profile->seconds[k] += secs[k];
    profile->iterations += 1;  // rsf.cpp:355
  } else {
    check(rsfg_state_step(st.s_, &frac));
  }
  return frac;
}

// rsf::energy (rsf.hpp:82): the update field E of the current state.
inline Volume energy(const EvolutionState& st, const Volume& I, const RsfParams& p) {
  p.validate();
  if (!(I.dims == st.dims_)) throw shape_error("energy: image dims differ from the state's");
  EvolutionState& m = const_cast<EvolutionState&>(st);  // logically const: phi is not advanced
  m.sync_params(p);
  Volume E(st.dims_.nx, st.dims_.ny, st.dims_.nz);
  check(rsfg_state_energy(st.s_, E.data.data()));
  return E;
}

// Short forms (the state already holds I and p).
inline double evolve_step(EvolutionState& st) {
  double frac = 0.0;
  check(rsfg_state_step(st.handle(), &frac));
  return frac;
}
inline Volume energy(EvolutionState& st) {
  Volume E(st.dims().nx, st.dims().ny, st.dims().nz);
  check(rsfg_state_energy(st.handle(), E.data.data()));
  return E;
}

// rsf::region_intensities (rsf.hpp:39-41) on the GPU.
inline std::pair<Volume, Volume> region_intensities(const Volume& I, const Volume& phi, double sigma1,
                                                    double epsilon, double denom_floor = 1e-8, int device = 0) {
  check_same_dims(I, phi, "region_intensities");
  Volume rp(I.dims.nx, I.dims.ny, I.dims.nz), rm(I.dims.nx, I.dims.ny, I.dims.nz);
  check(rsfg_region_intensities(I.data.data(), phi.data.data(), I.dims.nx, I.dims.ny, I.dims.nz, sigma1, epsilon,
                                denom_floor, rp.data.data(), rm.data.data(), device));
  return {std::move(rp), std::move(rm)};
}

// rsf::directional_forces (rsf.hpp:47-50) on the GPU.
inline std::pair<Volume, Volume> directional_forces(const Volume& I, const Volume& r_plus, const Volume& r_minus,
                                                    const Volume& KI, const Volume& KI2, int device = 0) {
  check_same_dims(I, r_plus, "directional_forces");
  check_same_dims(I, r_minus, "directional_forces");
  check_same_dims(I, KI, "directional_forces");
  check_same_dims(I, KI2, "directional_forces");
  Volume Fp(I.dims.nx, I.dims.ny, I.dims.nz), Fm(I.dims.nx, I.dims.ny, I.dims.nz);
  check(rsfg_directional_forces(r_plus.data.data(), r_minus.data.data(), KI.data.data(), KI2.data.data(),
                                (int64_t)I.voxels(), Fp.data.data(), Fm.data.data(), device));
  return {std::move(Fp), std::move(Fm)};
}

// ---- seeding and curtain tiling around the hot path ------

enum class Polarity { bright_on_dark, dark_on_bright };  // seeding.hpp:10

// rsf::BlobParams (seeding.hpp:12-20), same defaults.
struct BlobParams {
  double sigma_b = 3.0;
  double response_threshold = 0.1;
  double nms_radius = 0.0;
  Polarity polarity = Polarity::bright_on_dark;
  double resolved_nms_radius() const { return nms_radius > 0.0 ? nms_radius : 2.0 * sigma_b; }
  rsfg_blob_params c() const {
    return rsfg_blob_params{sigma_b, response_threshold, nms_radius, polarity == Polarity::dark_on_bright ? 1 : 0};
  }
};

struct Seed {  // seeding.hpp:22-25
  int x = 0, y = 0, z = 0;
  float response = 0.0f;
};
struct SeedSet {  // seeding.hpp:27-31
  std::vector<Seed> points;
  double detection_scale = 0.0;
  double response_threshold = 0.0;
};

// rsf::init_phi (seeding.hpp:60-61, seeding.cpp:221-235): seeds and the
// distance field computed on the GPU; same seeds, same order.
inline std::pair<Volume, SeedSet> init_phi(const Volume& vol, const BlobParams& bp, double seed_radius = 2.0,
                                           int device = 0) {
  const rsfg_blob_params cb = bp.c();
  Volume phi(vol.dims.nx, vol.dims.ny, vol.dims.nz);
  int32_t cap = (int32_t)std::min<std::size_t>(vol.voxels(), 1u << 16), n = 0, it = 0;
  std::vector<int32_t> xyz;
  std::vector<float> resp;
  for (;;) {
    xyz.assign(3 * (std::size_t)cap, 0);
    resp.assign(cap, 0.0f);
    check(rsfg_init_phi(vol.data.data(), vol.dims.nx, vol.dims.ny, vol.dims.nz, &cb, seed_radius, phi.data.data(),
                        device, &n, xyz.data(), resp.data(), cap, &it));
    if (n <= cap) break;
    cap = n;  // more seeds than the first buffer held: rerun with room for all
  }
  SeedSet s;
  s.detection_scale = bp.sigma_b;
  s.response_threshold = bp.response_threshold;
  s.points.resize(n);
  for (int32_t k = 0; k < n; ++k) s.points[k] = Seed{xyz[3 * k], xyz[3 * k + 1], xyz[3 * k + 2], resp[k]};
  return {std::move(phi), std::move(s)};
}

struct TileBox {  // tiling.hpp:13-17
  int ix = 0, iy = 0, iz = 0;
  Dims core_origin, core_extent;
  Dims pad_origin, pad_extent;
};
struct TileLayout {  // tiling.hpp:19-24
  Dims vol_dims;
  Dims tile_size;
  int curtain = 0;
  std::vector<TileBox> tiles;
};
enum class MergeMode { linear, minimum, maximum, average };  // tiling.hpp:26

// rsf::plan_tiles (tiling.hpp:28-30, tiling.cpp:14-59).
inline TileLayout plan_tiles(Dims dims, Dims tile_size, double sigma1, double sigma2) {
  TileLayout L;
  L.vol_dims = dims;
  L.tile_size = tile_size;
  int32_t n = 0, curtain = 0;
  check(rsfg_plan_tiles(dims.nx, dims.ny, dims.nz, tile_size.nx, tile_size.ny, tile_size.nz, sigma1, sigma2, nullptr,
                        0, &n, &curtain));
  std::vector<rsfg_tile> t(n);
  check(rsfg_plan_tiles(dims.nx, dims.ny, dims.nz, tile_size.nx, tile_size.ny, tile_size.nz, sigma1, sigma2, t.data(),
                        n, &n, &curtain));
  L.curtain = curtain;
  for (const rsfg_tile& c : t)
    L.tiles.push_back(TileBox{c.ix, c.iy, c.iz, Dims{c.core_origin[0], c.core_origin[1], c.core_origin[2]},
                              Dims{c.core_extent[0], c.core_extent[1], c.core_extent[2]},
                              Dims{c.pad_origin[0], c.pad_origin[1], c.pad_origin[2]},
                              Dims{c.pad_extent[0], c.pad_extent[1], c.pad_extent[2]}});
  return L;
}

inline rsfg_tile c_tile(const TileBox& t) {
  return rsfg_tile{t.ix, t.iy, t.iz, {t.core_origin.nx, t.core_origin.ny, t.core_origin.nz},
                   {t.core_extent.nx, t.core_extent.ny, t.core_extent.nz},
                   {t.pad_origin.nx, t.pad_origin.ny, t.pad_origin.nz},
                   {t.pad_extent.nx, t.pad_extent.ny, t.pad_extent.nz}};
}
inline std::vector<rsfg_tile> c_tiles(const TileLayout& L) {
  std::vector<rsfg_tile> v;
  for (const TileBox& t : L.tiles) v.push_back(c_tile(t));
  return v;
}

// rsf::tile_file_name (tiling.cpp:195-199).
inline std::string tile_file_name(const TileBox& t) {
  char buf[64];
  const rsfg_tile c = c_tile(t);
  check(rsfg_tile_file_name(&c, buf, sizeof buf));
  return buf;
}

// rsf::save_manifest / load_manifest (tiling.cpp:277-321); paths as strings.
inline void save_manifest(const std::string& path, const TileLayout& L) {
  const std::vector<rsfg_tile> v = c_tiles(L);
  check(rsfg_save_manifest(path.c_str(), L.vol_dims.nx, L.vol_dims.ny, L.vol_dims.nz, L.tile_size.nx,
                           L.tile_size.ny, L.tile_size.nz, L.curtain, v.data(), (int32_t)v.size()));
}
inline TileLayout load_manifest(const std::string& path) {
  int32_t d[3], ts[3], c = 0, n = 0;
  check(rsfg_load_manifest(path.c_str(), d, ts, &c, nullptr, 0, &n));
  std::vector<rsfg_tile> v(n);
  check(rsfg_load_manifest(path.c_str(), d, ts, &c, v.data(), n, &n));
  TileLayout L;
  L.vol_dims = Dims{d[0], d[1], d[2]};
  L.tile_size = Dims{ts[0], ts[1], ts[2]};
  L.curtain = c;
  for (const rsfg_tile& t : v)
    L.tiles.push_back(TileBox{t.ix, t.iy, t.iz, Dims{t.core_origin[0], t.core_origin[1], t.core_origin[2]},
                              Dims{t.core_extent[0], t.core_extent[1], t.core_extent[2]},
                              Dims{t.pad_origin[0], t.pad_origin[1], t.pad_origin[2]},
                              Dims{t.pad_extent[0], t.pad_extent[1], t.pad_extent[2]}});
  return L;
}

// rsf::merge_from_dir (tiling.cpp:323-332): tiles read and merged on the GPU.
inline Volume merge_from_dir(const std::string& dir, const TileLayout& L, MergeMode mode = MergeMode::linear,
                             int device = 0) {
  const std::vector<rsfg_tile> v = c_tiles(L);
  Volume out(L.vol_dims.nx, L.vol_dims.ny, L.vol_dims.nz);
  check(rsfg_merge_from_dir_host(dir.c_str(), L.vol_dims.nx, L.vol_dims.ny, L.vol_dims.nz, L.tile_size.nx,
                                 L.tile_size.ny, L.tile_size.nz, L.curtain, v.data(), (int32_t)v.size(),
                                 (int32_t)mode, out.data.data(), device));
  return out;
}

struct PipelineOptions {  // tiling.hpp:41-47
  bool global_seeding = false;
  MergeMode merge = MergeMode::linear;
  BlobParams blob;
  double seed_radius = 2.0;
  std::string spill_dir;  // when set, per-tile phi is written here + manifest
  int device = 0;
  int fields = RSFG_FIELDS_2;
};
struct PipelineResult {  // tiling.hpp:49-53
  Volume phi;
  Volume mask;
  std::vector<std::string> warnings;
};

// rsf::run_pipeline (tiling.hpp:58-60, tiling.cpp:201-275): every tile is
// seeded, initialised and evolved on one GPU, then merged on the device.
// `workers` is accepted for signature parity; tiles run back to back on the
// device (the output never depended on the worker count).
inline PipelineResult run_pipeline(const Volume& vol, const RsfParams& rsf_params, const BlobParams& blob_params,
                                   const TileLayout& layout, int workers, const PipelineOptions& opts = {}) {
  (void)workers;
  rsf_params.validate();
  if (!(layout.vol_dims == vol.dims)) throw shape_error("run_pipeline: layout does not match the volume");
  const rsfg_params cp = rsf_params.c();
  const rsfg_blob_params cb = blob_params.c();
  rsfg_pipeline_options o;
  rsfg_pipeline_options_default(&o);
  o.global_seeding = opts.global_seeding ? 1 : 0;
  o.merge = (int32_t)opts.merge;
  o.seed_radius = opts.seed_radius;
  o.device = opts.device;
  o.fields = opts.fields;
  o.spill_dir = opts.spill_dir.empty() ? nullptr : opts.spill_dir.c_str();
  PipelineResult r;
  r.phi = Volume(vol.dims.nx, vol.dims.ny, vol.dims.nz);
  r.mask = Volume(vol.dims.nx, vol.dims.ny, vol.dims.nz);
  std::vector<char> w(1 << 16, 0);
  int32_t nw = 0;
  check(rsfg_run_pipeline(vol.data.data(), vol.dims.nx, vol.dims.ny, vol.dims.nz, &cp, &cb, layout.tile_size.nx,
                          layout.tile_size.ny, layout.tile_size.nz, &o, r.phi.data.data(), r.mask.data.data(),
                          w.data(), (int32_t)w.size(), &nw));
  std::string all(w.data());
  for (std::size_t a = 0; a < all.size();) {
    std::size_t b = all.find('\n', a);
    if (b == std::string::npos) b = all.size();
    if (b > a) r.warnings.push_back(all.substr(a, b - a));
    a = b + 1;
  }
  return r;
}

}  // namespace rsfgpu
