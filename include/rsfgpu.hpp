// rsfgpu.hpp -- header-only C++ wrapper over the C-ABI (rsfg.h) with the
// reference's exact C++ surface: the same function names, argument meaning,
// defaults and exception types as /root/reference/proj/include/rsf/rsf.hpp
// (RsfParams, evolve, init_evolution, evolve_step, energy, extract_mask) in
// namespace rsfgpu.  A caller of rsf::evolve switches by changing the
// namespace (and linking librsfg.so); see INTEGRATION.md.
#pragma once

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

inline void check(int rc) {
  if (rc == RSFG_OK) return;
  const std::string msg = rsfg_last_error();
  switch (rc) {
    case RSFG_ERR_PARAM: throw param_error(msg);
    case RSFG_ERR_SHAPE: throw shape_error(msg);
    case RSFG_ERR_BLOWUP: throw blowup_error(msg);
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

// rsf::evolve (rsf.hpp:97-98).  `options` selects the device and the
// convolution form (RSFG_FIELDS_2 default, RSFG_FIELDS_4 reference form).
inline Volume evolve(Volume phi0, const Volume& I, const RsfParams& p, StopCheck stop = nullptr,
                     int stop_every = 25, const rsfg_options* options = nullptr) {
  p.validate();
  check_same_dims(phi0, I, "evolve");
  const rsfg_params cp = p.c();
  struct Ctx {
    StopCheck* stop;
  } ctx{&stop};
  auto tramp = [](const float* phi, int32_t nx, int32_t ny, int32_t nz, int32_t it, void* u) -> int {
    auto* c = static_cast<Ctx*>(u);
    Volume v(nx, ny, nz);
    std::memcpy(v.data.data(), phi, v.voxels() * sizeof(float));
    return (*c->stop)(v, it) ? 1 : 0;
  };
  check(rsfg_evolve(I.data.data(), phi0.data.data(), I.dims.nx, I.dims.ny, I.dims.nz, &cp, options,
                    stop ? +tramp : nullptr, &ctx, stop_every, nullptr));
  return phi0;
}

// rsf::extract_mask (rsf.hpp:101).
inline Volume extract_mask(const Volume& phi, int device = 0) {
  Volume m(phi.dims.nx, phi.dims.ny, phi.dims.nz);
  check(rsfg_extract_mask(phi.data.data(), m.data.data(), (int64_t)phi.voxels(), device));
  return m;
}

// rsf::EvolutionState + init_evolution / evolve_step / energy (rsf.hpp:54-88),
// with the state resident on the GPU.
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
  rsfg_state* handle() { return s_; }

 private:
  friend double evolve_step(EvolutionState&);
  friend Volume energy(EvolutionState&);
  rsfg_state* s_ = nullptr;
  Dims dims_;
  RsfParams p_;
};

inline EvolutionState init_evolution(const Volume& phi0, const Volume& I, const RsfParams& p,
                                     const rsfg_options* options = nullptr) {
  p.validate();
  return EvolutionState(phi0, I, p, options);
}

inline double evolve_step(EvolutionState& st) {
  double frac = 0.0;
  check(rsfg_state_step(st.s_, &frac));
  return frac;
}

inline Volume energy(EvolutionState& st) {
  Volume E(st.dims_.nx, st.dims_.ny, st.dims_.nz);
  check(rsfg_state_energy(st.s_, E.data.data()));
  return E;
}

}  // namespace rsfgpu
