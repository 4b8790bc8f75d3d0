// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference library (compiled by
// oracle/Makefile straight from /root/reference/proj/src into
// oracle/_ref/librsfref*.so).  It lets tests/ and bench.py's reference arm
// call the reference's own public C++ API (include/rsf/*.hpp) from ctypes:
// rsf::evolve / init_evolution / evolve_step / energy / extract_mask, the
// phantom generator, perturb, init_phi, merge_phi and run_pipeline.  No reference source is copied
// here; every call goes to the reference's compiled code.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "rsf/phantom.hpp"
#include "rsf/rsf.hpp"
#include "rsf/seeding.hpp"
#include "rsf/tiling.hpp"
#include "rsf/validation.hpp"
#include "rsf/volume_io.hpp"

namespace {
thread_local std::string g_err;

struct RefParams {  // field-for-field rsf::RsfParams (rsf.hpp:13-26)
  double sigma1, sigma2, alpha, beta, epsilon, dt;
  int32_t max_iters;
  double convergence_fraction, denom_floor, grad_floor;
};

rsf::RsfParams to_ref(const RefParams* p) {
  rsf::RsfParams r;
  r.sigma1 = p->sigma1;
  r.sigma2 = p->sigma2;
  r.alpha = p->alpha;
  r.beta = p->beta;
  r.epsilon = p->epsilon;
  r.dt = p->dt;
  r.max_iters = p->max_iters;
  r.convergence_fraction = p->convergence_fraction;
  r.denom_floor = p->denom_floor;
  r.grad_floor = p->grad_floor;
  return r;
}

rsf::Volume make_vol(const float* d, int nx, int ny, int nz) {
  rsf::Volume v(nx, ny, nz);
  std::memcpy(v.data.data(), d, v.voxels() * sizeof(float));
  return v;
}

// 0 ok, 1 param, 2 shape, 3 blowup, 8 io, 7 other
int code_of(const std::exception& e) {
  if (dynamic_cast<const rsf::io_error*>(&e)) return 8;
  if (dynamic_cast<const rsf::param_error*>(&e)) return 1;
  if (dynamic_cast<const rsf::shape_error*>(&e)) return 2;
  if (dynamic_cast<const rsf::blowup_error*>(&e)) return 3;
  return 7;
}

struct RefState {
  rsf::EvolutionState st;
  rsf::EvolveWorkspace ws;
  rsf::Volume I;
  rsf::RsfParams p;
};
}  // namespace

#define GUARD(...)                  \
  try {                             \
    __VA_ARGS__;                    \
    return 0;                       \
  } catch (const std::exception& e) { \
    g_err = e.what();               \
    return code_of(e);              \
  }

extern "C" {

const char* rsfref_last_error() { return g_err.c_str(); }
void rsfref_set_workers(int n) { rsf::set_worker_count(n); }
int rsfref_workers() { return rsf::detail::effective_workers(); }

int rsfref_evolve(const float* I, float* phi, int nx, int ny, int nz, const RefParams* p) {
  GUARD({
    rsf::Volume out = rsf::evolve(make_vol(phi, nx, ny, nz), make_vol(I, nx, ny, nz), to_ref(p));
    std::memcpy(phi, out.data.data(), out.voxels() * sizeof(float));
  })
}

int rsfref_state_create(void** out, const float* phi0, const float* I, int nx, int ny, int nz,
                        const RefParams* p) {
  GUARD({
    auto* s = new RefState;
    try {
      s->p = to_ref(p);
      s->I = make_vol(I, nx, ny, nz);
      s->st = rsf::init_evolution(make_vol(phi0, nx, ny, nz), s->I, s->p);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  })
}

int rsfref_state_step(void* h, double* frac) {
  auto* s = static_cast<RefState*>(h);
  GUARD({ *frac = rsf::evolve_step(s->st, s->I, s->p, s->ws); })
}

int rsfref_state_phi(void* h, float* out) {
  auto* s = static_cast<RefState*>(h);
  std::memcpy(out, s->st.phi.data.data(), s->st.phi.voxels() * sizeof(float));
  return 0;
}

int rsfref_state_set_phi(void* h, const float* in) {
  auto* s = static_cast<RefState*>(h);
  std::memcpy(s->st.phi.data.data(), in, s->st.phi.voxels() * sizeof(float));
  return 0;
}

int rsfref_state_energy(void* h, float* out) {
  auto* s = static_cast<RefState*>(h);
  GUARD({
    rsf::Volume E = rsf::energy(s->st, s->I, s->p);
    std::memcpy(out, E.data.data(), E.voxels() * sizeof(float));
  })
}

int rsfref_state_static(void* h, float* KI, float* KI2, float* imin, float* imax) {
  auto* s = static_cast<RefState*>(h);
  std::memcpy(KI, s->st.KI.data.data(), s->st.KI.voxels() * sizeof(float));
  std::memcpy(KI2, s->st.KI2.data.data(), s->st.KI2.voxels() * sizeof(float));
  *imin = s->st.i_min;
  *imax = s->st.i_max;
  return 0;
}

void rsfref_state_destroy(void* h) { delete static_cast<RefState*>(h); }

int rsfref_convolve(const float* v, int nx, int ny, int nz, double sigma, float* out) {
  GUARD({
    rsf::Volume o = rsf::convolve_separable(make_vol(v, nx, ny, nz), rsf::gaussian_kernel(sigma));
    std::memcpy(out, o.data.data(), o.voxels() * sizeof(float));
  })
}

int rsfref_gaussian_kernel(double sigma, double* w, int cap, int* radius) {
  GUARD({
    rsf::Kernel1D k = rsf::gaussian_kernel(sigma);
    if (static_cast<int>(k.weights.size()) > cap) throw rsf::param_error("cap");
    std::memcpy(w, k.weights.data(), k.weights.size() * sizeof(double));
    *radius = k.radius;
  })
}

int rsfref_extract_mask(const float* phi, int nx, int ny, int nz, float* mask) {
  GUARD({
    rsf::Volume m = rsf::extract_mask(make_vol(phi, nx, ny, nz));
    std::memcpy(mask, m.data.data(), m.voxels() * sizeof(float));
  })
}

// generate_network (phantom.cpp:55-184) + perturb (phantom.cpp:186-214).
int rsfref_phantom(int nx, int ny, int nz, int n_branches, double rmin, double rmax, double tortuosity,
                   float fg, float bg, uint64_t seed, int tree_connected, double axial_blur,
                   double noise_sigma, int contrast_axis, double lo, double hi, uint64_t noise_seed,
                   float* image, float* gt) {
  GUARD({
    rsf::PhantomSpec s;
    s.dims = {nx, ny, nz};
    s.n_branches = n_branches;
    s.radius_min = rmin;
    s.radius_max = rmax;
    s.tortuosity = tortuosity;
    s.foreground = fg;
    s.background = bg;
    s.rng_seed = seed;
    s.tree_connected = tree_connected != 0;
    s.axial_blur_sigma = axial_blur;
    rsf::PhantomResult r = rsf::generate_network(s);
    rsf::PerturbSpec ps;
    ps.gaussian_sigma = noise_sigma;
    ps.contrast_axis = static_cast<rsf::Axis>(contrast_axis);
    ps.contrast_lo = lo;
    ps.contrast_hi = hi;
    rsf::Volume img = rsf::perturb(r.image, ps, noise_seed);
    std::memcpy(image, img.data.data(), img.voxels() * sizeof(float));
    std::memcpy(gt, r.gt_mask.data.data(), r.gt_mask.voxels() * sizeof(float));
  })
}

// detect_seeds (seeding.cpp:83-145): up to cap seeds as x, y, z triples and
// responses, in the reference's order; *n gets the full count.
int rsfref_detect_seeds(const float* vol, int nx, int ny, int nz, double sigma_b, double threshold, double nms,
                        int dark, int* xyz, float* resp, int cap, int* n) {
  GUARD({
    rsf::BlobParams bp;
    bp.sigma_b = sigma_b;
    bp.response_threshold = threshold;
    bp.nms_radius = nms;
    bp.polarity = dark ? rsf::Polarity::dark_on_bright : rsf::Polarity::bright_on_dark;
    const rsf::SeedSet s = rsf::detect_seeds(make_vol(vol, nx, ny, nz), bp);
    *n = static_cast<int>(s.points.size());
    for (int k = 0; k < *n && k < cap; ++k) {
      xyz[3 * k] = s.points[k].x;
      xyz[3 * k + 1] = s.points[k].y;
      xyz[3 * k + 2] = s.points[k].z;
      resp[k] = s.points[k].response;
    }
  })
}

// init_phi (seeding.cpp:221-235); returns the seed count through *n_seeds.
int rsfref_init_phi(const float* vol, int nx, int ny, int nz, double sigma_b, double threshold, double nms,
                    int dark, double seed_radius, float* phi, int* n_seeds) {
  GUARD({
    rsf::BlobParams bp;
    bp.sigma_b = sigma_b;
    bp.response_threshold = threshold;
    bp.nms_radius = nms;
    bp.polarity = dark ? rsf::Polarity::dark_on_bright : rsf::Polarity::bright_on_dark;
    auto [p, seeds] = rsf::init_phi(make_vol(vol, nx, ny, nz), bp, seed_radius);
    std::memcpy(phi, p.data.data(), p.voxels() * sizeof(float));
    *n_seeds = static_cast<int>(seeds.points.size());
  })
}

double rsfref_dice(const float* a, const float* b, int nx, int ny, int nz) {
  return rsf::dice(make_vol(a, nx, ny, nz), make_vol(b, nx, ny, nz));
}

// merge_phi (tiling.cpp:99-193) of caller-provided tile fields over
// plan_tiles((nx, ny, nz), (tx, ty, tz), sigma1, sigma2).
int rsfref_merge_phi(const float* const* tiles, int n_tiles, int nx, int ny, int nz, int tx, int ty, int tz,
                     double sigma1, double sigma2, int mode, float* out) {
  GUARD({
    const rsf::TileLayout L = rsf::plan_tiles({nx, ny, nz}, {tx, ty, tz}, sigma1, sigma2);
    if ((int)L.tiles.size() != n_tiles) throw rsf::shape_error("rsfref_merge_phi: tile count");
    std::vector<rsf::Volume> v;
    for (int i = 0; i < n_tiles; ++i) {
      const rsf::Dims& e = L.tiles[i].pad_extent;
      v.push_back(make_vol(tiles[i], e.nx, e.ny, e.nz));
    }
    rsf::Volume m = rsf::merge_phi(v, L, static_cast<rsf::MergeMode>(mode));
    std::memcpy(out, m.data.data(), m.voxels() * sizeof(float));
  })
}

// run_pipeline (tiling.cpp:201-275) with default BlobParams(sigma_b, threshold).
int rsfref_run_pipeline(const float* image, int nx, int ny, int nz, const RefParams* p, double sigma_b,
                        double threshold, int tx, int ty, int tz, int global_seeding, int mode, double seed_radius,
                        float* phi, float* mask, int* n_warnings) {
  GUARD({
    rsf::BlobParams bp;
    bp.sigma_b = sigma_b;
    bp.response_threshold = threshold;
    const rsf::TileLayout L = rsf::plan_tiles({nx, ny, nz}, {tx, ty, tz}, p->sigma1, p->sigma2);
    rsf::PipelineOptions o;
    o.global_seeding = global_seeding != 0;
    o.merge = static_cast<rsf::MergeMode>(mode);
    o.seed_radius = seed_radius;
    const rsf::PipelineResult r = rsf::run_pipeline(make_vol(image, nx, ny, nz), to_ref(p), bp, L, 0, o);
    std::memcpy(phi, r.phi.data.data(), r.phi.voxels() * sizeof(float));
    std::memcpy(mask, r.mask.data.data(), r.mask.voxels() * sizeof(float));
    *n_warnings = static_cast<int>(r.warnings.size());
  })
}

// save_manifest (tiling.cpp:277-295) of plan_tiles(dims, tile, sigma1, sigma2).
int rsfref_save_manifest(const char* path, int nx, int ny, int nz, int tx, int ty, int tz, double sigma1,
                         double sigma2) {
  GUARD({ rsf::save_manifest(path, rsf::plan_tiles({nx, ny, nz}, {tx, ty, tz}, sigma1, sigma2)); })
}

// load_manifest + merge_from_dir (tiling.cpp:297-332) into out.
int rsfref_merge_from_dir(const char* dir, const char* manifest, int mode, float* out, long cap) {
  GUARD({
    const rsf::TileLayout L = rsf::load_manifest(manifest);
    rsf::Volume m = rsf::merge_from_dir(dir, L, static_cast<rsf::MergeMode>(mode));
    if ((long)m.voxels() > cap) throw rsf::shape_error("rsfref_merge_from_dir: capacity");
    std::memcpy(out, m.data.data(), m.voxels() * sizeof(float));
  })
}

// read_volume (volume_io.cpp:24-113) into out (capacity cap floats).
int rsfref_read_volume(const char* header, float* out, long cap, int* nx, int* ny, int* nz, float* range2) {
  GUARD({
    rsf::Volume v = rsf::read_volume(header);
    *nx = v.dims.nx, *ny = v.dims.ny, *nz = v.dims.nz;
    if ((long)v.voxels() > cap) throw rsf::shape_error("rsfref_read_volume: capacity");
    std::memcpy(out, v.data.data(), v.voxels() * sizeof(float));
    range2[0] = v.value_range->first, range2[1] = v.value_range->second;
  })
}

// rsf::region_intensities (rsf.hpp:39-41, rsf.cpp:235-266).
int rsfref_region_intensities(const float* I, const float* phi, int nx, int ny, int nz, double sigma1,
                              double epsilon, double denom_floor, float* r_plus, float* r_minus) {
  GUARD({
    auto rr = rsf::region_intensities(make_vol(I, nx, ny, nz), make_vol(phi, nx, ny, nz), sigma1, epsilon,
                                      denom_floor);
    std::memcpy(r_plus, rr.first.data.data(), rr.first.voxels() * sizeof(float));
    std::memcpy(r_minus, rr.second.data.data(), rr.second.voxels() * sizeof(float));
  })
}

// rsf::directional_forces (rsf.hpp:47-50, rsf.cpp:268-291).
int rsfref_directional_forces(const float* I, const float* rp, const float* rm, const float* KI, const float* KI2,
                              int nx, int ny, int nz, float* Fp, float* Fm) {
  GUARD({
    auto ff = rsf::directional_forces(make_vol(I, nx, ny, nz), make_vol(rp, nx, ny, nz), make_vol(rm, nx, ny, nz),
                                      make_vol(KI, nx, ny, nz), make_vol(KI2, nx, ny, nz));
    std::memcpy(Fp, ff.first.data.data(), ff.first.voxels() * sizeof(float));
    std::memcpy(Fm, ff.second.data.data(), ff.second.voxels() * sizeof(float));
  })
}

}  // extern "C"
