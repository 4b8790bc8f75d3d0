// Drives include/rsfgpu.hpp (the reference-shaped C++ surface) the way a
// reference caller would: rsf::evolve, init_phi, plan_tiles, run_pipeline
// (rsf.hpp:97-101, seeding.hpp:60-61, tiling.hpp:28-60) with the namespace
// switched to rsfgpu.  Used by tests/test_cpp_wrapper.py.
//   wrapper_check cpu                      exceptions + plan_tiles, no GPU
//   wrapper_check gpu nx ny nz image out   evolve / init_phi / run_pipeline
#include <cstdio>
#include <fstream>
#include <string>

#include "rsfgpu.hpp"

static void dump(const std::string& path, const rsfgpu::Volume& v) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data.data()), (std::streamsize)(v.voxels() * sizeof(float)));
}

template <class E, class F>
static bool throws(F&& f, const char* want) {
  try {
    f();
  } catch (const E& e) {
    return std::string(e.what()).find(want) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  if (mode == "cpu") {
    rsfgpu::RsfParams bad;
    bad.dt = 0.0;
    const bool e1 = throws<rsfgpu::param_error>([&] { bad.validate(); }, "dt must be > 0");
    const bool e2 = throws<rsfgpu::param_error>(
        [&] { rsfgpu::plan_tiles({64, 64, 64}, {8, 8, 8}, 3.0, 0.0); }, "");
    const rsfgpu::TileLayout L = rsfgpu::plan_tiles({100, 80, 60}, {48, 40, 30}, 2.0, 1.0);
    std::printf("{\"param_error\": %d, \"tile_error\": %d, \"curtain\": %d, \"tiles\": [", e1, e2, L.curtain);
    for (std::size_t i = 0; i < L.tiles.size(); ++i) {
      const rsfgpu::TileBox& t = L.tiles[i];
      std::printf("%s[%d,%d,%d,%d,%d,%d,%d,%d,%d,%d,%d,%d,%d,%d,%d]", i ? "," : "", t.ix, t.iy, t.iz,
                  t.core_origin.nx, t.core_origin.ny, t.core_origin.nz, t.core_extent.nx, t.core_extent.ny,
                  t.core_extent.nz, t.pad_origin.nx, t.pad_origin.ny, t.pad_origin.nz, t.pad_extent.nx,
                  t.pad_extent.ny, t.pad_extent.nz);
    }
    std::printf("]}\n");
    return 0;
  }
  if (argc < 7) return 2;
  const int nx = std::stoi(argv[2]), ny = std::stoi(argv[3]), nz = std::stoi(argv[4]);
  const std::string out = argv[6];
  rsfgpu::Volume img(nx, ny, nz);
  std::ifstream(argv[5], std::ios::binary)
      .read(reinterpret_cast<char*>(img.data.data()), (std::streamsize)(img.voxels() * sizeof(float)));

  rsfgpu::BlobParams bp;
  auto [phi0, seeds] = rsfgpu::init_phi(img, bp, 2.0);
  dump(out + "/init_phi.raw", phi0);

  rsfgpu::RsfParams p;
  p.sigma1 = 2.0;
  p.max_iters = 20;
  const rsfgpu::Volume phi = rsfgpu::evolve(phi0, img, p);
  dump(out + "/evolve_phi.raw", phi);
  dump(out + "/mask.raw", rsfgpu::extract_mask(phi));

  const rsfgpu::TileLayout L = rsfgpu::plan_tiles(img.dims, {nx / 2, ny / 2, nz / 2}, p.sigma1, p.sigma2);
  const rsfgpu::PipelineResult r = rsfgpu::run_pipeline(img, p, bp, L, 4);
  dump(out + "/pipe_phi.raw", r.phi);
  dump(out + "/pipe_mask.raw", r.mask);

  std::printf("{\"n_seeds\": %zu, \"seed0\": [%d, %d, %d, %.9g], \"n_tiles\": %zu, \"n_warnings\": %zu}\n",
              seeds.points.size(), seeds.points.empty() ? -1 : seeds.points[0].x,
              seeds.points.empty() ? -1 : seeds.points[0].y, seeds.points.empty() ? -1 : seeds.points[0].z,
              seeds.points.empty() ? 0.0 : (double)seeds.points[0].response, L.tiles.size(), r.warnings.size());
  return 0;
}
