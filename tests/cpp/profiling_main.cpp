// Driver for the reference's own src/profiling.cpp compiled against the GPU
// library (include/compat/rsf/profiling.hpp, -Drsf=rsfgpu): the reference's
// profile_evolution times our kernels through rsfgpu::evolve_step(st, I, p,
// ws, &KernelProfile) and its profile_table prints the 14-row report.
//   profiling_check table      -- formatting only (no GPU)
//   profiling_check run N      -- profile_evolution on an N^3 sphere case
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "rsf/profiling.hpp"

int main(int argc, char** argv) {
  using namespace rsfgpu;
  if (argc >= 2 && std::strcmp(argv[1], "table") == 0) {
    ProfileReport r;
    r.iterations = 3;
    r.warmup = 1;
    r.dims = Dims{8, 8, 8};
    r.workers = detail::effective_workers();
    for (int k = 0; k < KernelProfile::kCount; ++k)
      r.rows.push_back(ProfileRow{KernelProfile::names()[k], k == 2 ? 1.5 : 0.0, k == 2 ? 100.0 : 0.0});
    r.total_ms_per_iter = 1.5;
    std::fputs(profile_table(r).c_str(), stdout);
    return 0;
  }
  if (argc >= 3 && std::strcmp(argv[1], "run") == 0) {
    const int n = std::atoi(argv[2]);
    Volume I(n, n, n), phi0(n, n, n);
    for (int z = 0; z < n; ++z)
      for (int y = 0; y < n; ++y)
        for (int x = 0; x < n; ++x) {
          const double dx = x - 0.5 * n, dy = y - 0.4 * n, dz = z - 0.55 * n;
          const double r = std::sqrt(dx * dx + dy * dy + dz * dz);
          const std::size_t i = (std::size_t)x + (std::size_t)n * (y + (std::size_t)n * z);
          I.data[i] = (float)(r < 0.25 * n ? 200.0 : 50.0) + (float)((i * 2654435761u) % 17);
          phi0.data[i] = (float)(r - 0.3 * n);
        }
    RsfParams p;
    p.sigma1 = 3.0;
    try {
      ProfileReport r = profile_evolution(I, phi0, p, 5, 2);
      std::fputs(profile_table(r).c_str(), stdout);
    } catch (const std::exception& e) {
      std::fprintf(stderr, "error: %s\n", e.what());
      return 1;
    }
    return 0;
  }
  std::fprintf(stderr, "usage: %s table | run N\n", argv[0]);
  return 2;
}
