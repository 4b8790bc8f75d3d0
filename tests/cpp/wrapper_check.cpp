// Drives include/rsfgpu.hpp (the reference-shaped C++ surface) the way a
// reference caller would: rsf::evolve, init_phi, plan_tiles, run_pipeline
// (rsf.hpp:97-101, seeding.hpp:60-61, tiling.hpp:28-71) with the namespace
// switched to rsfgpu.  Used by tests/test_cpp_wrapper.py.
//   wrapper_check cpu [dir]                exceptions, plan_tiles, manifest; no GPU
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
    const std::string mf = argc > 2 ? std::string(argv[2]) + "/layout.manifest" : "layout.manifest";
    rsfgpu::save_manifest(mf, L);
    const rsfgpu::TileLayout B = rsfgpu::load_manifest(mf);
    bool same = B.curtain == L.curtain && B.vol_dims == L.vol_dims && B.tile_size == L.tile_size &&
                B.tiles.size() == L.tiles.size();
    for (std::size_t i = 0; same && i < B.tiles.size(); ++i)
      same = B.tiles[i].pad_extent == L.tiles[i].pad_extent && B.tiles[i].core_origin == L.tiles[i].core_origin;
    const bool e3 = throws<rsfgpu::io_error>([&] { rsfgpu::load_manifest(mf + ".missing"); }, "cannot open manifest");
    std::printf("{\"manifest_roundtrip\": %d, \"io_error\": %d, \"last_name\": \"%s\", ", same, e3,
                rsfgpu::tile_file_name(L.tiles.back()).c_str());
    std::printf("\"param_error\": %d, \"tile_error\": %d, \"curtain\": %d, \"tiles\": [", e1, e2, L.curtain);
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
  // two z-slabs with peer-linked halos (one device here): the same bits
  dump(out + "/evolve_multi_phi.raw", rsfgpu::evolve_multi(phi0, img, p, {0, 0}));
  dump(out + "/mask.raw", rsfgpu::extract_mask(phi));

  const rsfgpu::TileLayout L = rsfgpu::plan_tiles(img.dims, {nx / 2, ny / 2, nz / 2}, p.sigma1, p.sigma2);
  rsfgpu::PipelineOptions po;
  po.spill_dir = out;  // tiles + layout.manifest next to the other outputs
  const rsfgpu::PipelineResult r = rsfgpu::run_pipeline(img, p, bp, L, 4, po);
  dump(out + "/pipe_phi.raw", r.phi);
  dump(out + "/pipe_mask.raw", r.mask);
  const rsfgpu::TileLayout back = rsfgpu::load_manifest(out + "/layout.manifest");
  dump(out + "/merged_from_dir.raw", rsfgpu::merge_from_dir(out, back));

  std::printf("{\"n_seeds\": %zu, \"seed0\": [%d, %d, %d, %.9g], \"n_tiles\": %zu, \"n_warnings\": %zu}\n",
              seeds.points.size(), seeds.points.empty() ? -1 : seeds.points[0].x,
              seeds.points.empty() ? -1 : seeds.points[0].y, seeds.points.empty() ? -1 : seeds.points[0].z,
              seeds.points.empty() ? 0.0 : (double)seeds.points[0].response, L.tiles.size(), r.warnings.size());
  return 0;
}
