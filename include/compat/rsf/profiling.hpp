// compat/rsf/profiling.hpp -- lets the reference's OWN src/profiling.cpp
// (profile_evolution / profile_table, profiling.cpp:8-63) compile unmodified
// against the GPU library: compile it with
//
//     g++ -Drsf=rsfgpu -I<repo>/include/compat -I<repo>/include
//         /root/reference/proj/src/profiling.cpp ... -lrsfg
//
// The namespace swap (-Drsf=rsfgpu) is the only change; everything
// profiling.cpp uses -- Volume/Dims, replicate_z, check_same_dims,
// to_string(Dims), param_error, RsfParams, init_evolution, EvolveWorkspace,
// evolve_step(st, I, p, ws, &prof), KernelProfile (14 rows), detail::
// effective_workers -- comes from rsfgpu.hpp with the reference's signatures
// (rsf.hpp:13-101).  The declarations below are profiling.hpp's API
// (ProfileRow / ProfileReport / profile_evolution / profile_table).
#pragma once

#include <string>
#include <vector>

#include "rsfgpu.hpp"

namespace rsfgpu {

struct ProfileRow {
  std::string kernel;
  double ms_per_iter = 0.0;
  double percent = 0.0;
};

struct ProfileReport {
  std::vector<ProfileRow> rows;
  int iterations = 0;
  int warmup = 0;
  Dims dims;
  int workers = 0;
  double total_ms_per_iter = 0.0;
};

ProfileReport profile_evolution(const Volume& I, Volume phi0, const RsfParams& params, int iterations = 10,
                                int warmup = 2);

std::string profile_table(const ProfileReport& report);

}  // namespace rsfgpu
