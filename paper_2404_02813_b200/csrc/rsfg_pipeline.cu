// rsfg_pipeline.cu -- curtain tiling around the hot path (SURVEY.md 8(f)
// row f3; reference tiling.cpp:14-275): plan_tiles, merge_phi on the device,
// and run_pipeline driving the library's own device paths per tile (extract
// -> seeds -> distance -> evolve) before one device merge.
//
// merge_phi is exact: every output voxel gathers the tiles whose padded box
// contains it in increasing tile index -- the order in which the reference's
// tile loop accumulates (tiling.cpp:116-150) -- with the same f64 weights and
// accumulation, so identical tile fields merge to identical bits.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/rsfg.h"
#include "rsfg_internal.h"

namespace {

struct TileDev {  // per-axis geometry of the layout (tiles are a regular grid)
  int n[3];       // volume extent
  int t[3];       // tile size
  int nt[3];      // tiles per axis
  int curtain;    // max(layout curtain, 1) for the ramps
};

// axis_weight (tiling.cpp:84-97)
__device__ __forceinline__ double axis_weight(int x, int core0, int core1, int pad0, int pad1, int n, int curtain) {
  double w = 1.0;
  if (core0 > 0) {
    const double ramp = ((double)(x - pad0) + 0.5) / (2.0 * curtain);
    w = fmin(w, fmin(fmax(ramp, 0.0), 1.0));
  }
  if (core1 < n) {
    const double ramp = ((double)(pad1 - x) - 0.5) / (2.0 * curtain);
    w = fmin(w, fmin(fmax(ramp, 0.0), 1.0));
  }
  return w;
}

struct Axis {  // candidate tiles of one axis covering coordinate c (<= 3)
  int k, idx[3], core0[3], core1[3], pad0[3], pad1[3];
};

__device__ __forceinline__ Axis covering(int c, int n, int t, int nt, int curtain_raw) {
  Axis a;
  a.k = 0;
  const int ci = min(c / t, nt - 1);
  for (int i = max(ci - 1, 0); i <= min(ci + 1, nt - 1); ++i) {
    const int core0 = i * t, core1 = min(core0 + t, n);
    const int pad0 = max(core0 - curtain_raw, 0), pad1 = min(core1 + curtain_raw, n);
    if (c >= pad0 && c < pad1) {
      a.idx[a.k] = i;
      a.core0[a.k] = core0;
      a.core1[a.k] = core1;
      a.pad0[a.k] = pad0;
      a.pad1[a.k] = pad1;
      ++a.k;
    }
  }
  return a;
}

// merge_phi (tiling.cpp:99-193) for one output voxel per thread.
__global__ void merge_kernel(const float* const* __restrict__ tiles, TileDev L, int curtain_raw, int mode,
                             float* __restrict__ out, unsigned int* __restrict__ uncovered) {
  const size_t n = (size_t)L.n[0] * L.n[1] * L.n[2];
  for (size_t gi = blockIdx.x * (size_t)blockDim.x + threadIdx.x; gi < n; gi += (size_t)gridDim.x * blockDim.x) {
    const int x = (int)(gi % L.n[0]), y = (int)((gi / L.n[0]) % L.n[1]), z = (int)(gi / ((size_t)L.n[0] * L.n[1]));
    const Axis ax = covering(x, L.n[0], L.t[0], L.nt[0], curtain_raw);
    const Axis ay = covering(y, L.n[1], L.t[1], L.nt[1], curtain_raw);
    const Axis az = covering(z, L.n[2], L.t[2], L.nt[2], curtain_raw);
    double acc = 0.0, wsum = 0.0;
    int count = 0;
    float first = 0.0f;
    for (int a = 0; a < az.k; ++a) {  // increasing tile index: z, then y, then x
      const double wz = axis_weight(z, az.core0[a], az.core1[a], az.pad0[a], az.pad1[a], L.n[2], L.curtain);
      for (int b = 0; b < ay.k; ++b) {
        const double wy = axis_weight(y, ay.core0[b], ay.core1[b], ay.pad0[b], ay.pad1[b], L.n[1], L.curtain);
        for (int c = 0; c < ax.k; ++c) {
          const double wx = axis_weight(x, ax.core0[c], ax.core1[c], ax.pad0[c], ax.pad1[c], L.n[0], L.curtain);
          const double w = wx * wy * wz;
          const int ti = (az.idx[a] * L.nt[1] + ay.idx[b]) * L.nt[0] + ax.idx[c];
          const int ex = ax.pad1[c] - ax.pad0[c], ey = ay.pad1[b] - ay.pad0[b];
          const float vf = tiles[ti][(size_t)(x - ax.pad0[c]) +
                                     (size_t)ex * ((size_t)(y - ay.pad0[b]) + (size_t)ey * (z - az.pad0[a]))];
          const double v = vf;
          switch (mode) {
            case RSFG_MERGE_LINEAR:
              acc += w * v;
              wsum += w;
              break;
            case RSFG_MERGE_MINIMUM:
              acc = count ? fmin(acc, v) : v;
              break;
            case RSFG_MERGE_MAXIMUM:
              acc = count ? fmax(acc, v) : v;
              break;
            default:  // average
              acc += v;
              wsum += 1.0;
          }
          if (count == 0) first = vf;
          ++count;
        }
      }
    }
    if (count == 0) {
      atomicAdd(uncovered, 1u);
      out[gi] = 0.0f;
    } else if (count == 1) {
      out[gi] = first;  // exclusive region: the owner's value, bit for bit
    } else {
      out[gi] = (mode == RSFG_MERGE_LINEAR || mode == RSFG_MERGE_AVERAGE) ? (float)(acc / wsum) : (float)acc;
    }
  }
}

__global__ void extract_kernel(const float* __restrict__ vol, int nx, int ny, float* __restrict__ tile, int ox,
                               int oy, int oz, int ex, int ey, int ez) {
  const size_t n = (size_t)ex * ey * ez;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int x = (int)(i % ex), y = (int)((i / ex) % ey), z = (int)(i / ((size_t)ex * ey));
    tile[i] = vol[(size_t)(ox + x) + (size_t)nx * ((size_t)(oy + y) + (size_t)ny * (oz + z))];
  }
}

__global__ void fill_kernel(float* __restrict__ p, size_t n, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

int perr(int code, const std::string& m) {
  rsfg::set_error(m);
  return code;
}

std::string dims_str(int a, int b, int c) {
  return std::to_string(a) + "x" + std::to_string(b) + "x" + std::to_string(c);
}

int plan(int nx, int ny, int nz, int tx, int ty, int tz, double s1, double s2, std::vector<rsfg_tile>& out,
         int* curtain_out) {
  if (nx <= 0 || ny <= 0 || nz <= 0) return perr(RSFG_ERR_SHAPE, "plan_tiles: bad volume dims " + dims_str(nx, ny, nz));
  if (tx <= 0 || ty <= 0 || tz <= 0) return perr(RSFG_ERR_PARAM, "plan_tiles: tile_size must be positive");
  if (s1 < 0.0 || s2 < 0.0) return perr(RSFG_ERR_PARAM, "plan_tiles: sigma must be >= 0");
  const int curtain = (int)std::ceil(3.0 * std::max(s1, s2));  // tiling.cpp:21
  for (int t : {tx, ty, tz})
    if (t < 2 * curtain)
      return perr(RSFG_ERR_PARAM, "plan_tiles: tile_size " + dims_str(tx, ty, tz) + " too small for curtain " +
                                      std::to_string(curtain) + " (needs >= 2*curtain per axis)");
  const int ntx = (nx + tx - 1) / tx, nty = (ny + ty - 1) / ty, ntz = (nz + tz - 1) / tz;
  out.clear();
  for (int iz = 0; iz < ntz; ++iz)
    for (int iy = 0; iy < nty; ++iy)
      for (int ix = 0; ix < ntx; ++ix) {
        rsfg_tile t;
        t.ix = ix, t.iy = iy, t.iz = iz;
        const int o[3] = {ix * tx, iy * ty, iz * tz}, s[3] = {tx, ty, tz}, n[3] = {nx, ny, nz};
        for (int a = 0; a < 3; ++a) {
          t.core_origin[a] = o[a];
          t.core_extent[a] = std::min(s[a], n[a] - o[a]);
          t.pad_origin[a] = std::max(o[a] - curtain, 0);
          t.pad_extent[a] = std::min(o[a] + t.core_extent[a] + curtain, n[a]) - t.pad_origin[a];
        }
        out.push_back(t);
      }
  *curtain_out = curtain;
  return RSFG_OK;
}

int merge_device(const float* const* d_tiles_host, int n_tiles, int nx, int ny, int nz, int tx, int ty, int tz,
                 int curtain, int mode, float* d_out, cudaStream_t st) {
  TileDev L;
  L.n[0] = nx, L.n[1] = ny, L.n[2] = nz;
  L.t[0] = tx, L.t[1] = ty, L.t[2] = tz;
  L.nt[0] = (nx + tx - 1) / tx, L.nt[1] = (ny + ty - 1) / ty, L.nt[2] = (nz + tz - 1) / tz;
  L.curtain = std::max(curtain, 1);
  if (L.nt[0] * L.nt[1] * L.nt[2] != n_tiles) return perr(RSFG_ERR_SHAPE, "merge_phi: tile count does not match layout");
  const float** d_ptrs = nullptr;
  unsigned int* d_unc = nullptr;
  if (cudaMallocAsync(&d_ptrs, n_tiles * sizeof(float*), st) != cudaSuccess ||
      cudaMallocAsync(&d_unc, sizeof(unsigned int), st) != cudaSuccess)
    return perr(RSFG_ERR_OOM, "merge_phi: out of device memory");
  cudaMemcpyAsync(d_ptrs, d_tiles_host, n_tiles * sizeof(float*), cudaMemcpyHostToDevice, st);
  cudaMemsetAsync(d_unc, 0, sizeof(unsigned int), st);
  merge_kernel<<<148 * 8, 256, 0, st>>>(d_ptrs, L, curtain, mode, d_out, d_unc);
  unsigned int unc = 0;
  cudaMemcpyAsync(&unc, d_unc, sizeof unc, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_ptrs, st);
  cudaFreeAsync(d_unc, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return perr(RSFG_ERR_CUDA, "merge_phi: CUDA error");
  if (unc) return perr(RSFG_ERR_SHAPE, "merge_phi: layout leaves voxels uncovered");
  return RSFG_OK;
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) int rsfg_plan_tiles(int32_t nx, int32_t ny, int32_t nz, int32_t tx, int32_t ty,
                                                           int32_t tz, double sigma1, double sigma2, rsfg_tile* tiles,
                                                           int32_t cap, int32_t* n_tiles, int32_t* curtain) {
  std::vector<rsfg_tile> v;
  int c = 0;
  if (int rc = plan(nx, ny, nz, tx, ty, tz, sigma1, sigma2, v, &c)) return rc;
  if (n_tiles) *n_tiles = (int32_t)v.size();
  if (curtain) *curtain = c;
  for (size_t i = 0; tiles && i < v.size() && (int32_t)i < cap; ++i) tiles[i] = v[i];
  return RSFG_OK;
}

__attribute__((visibility("default"))) int rsfg_merge_phi_device(const float* const* d_tile_phis, int32_t n_tiles,
                                                                 int32_t nx, int32_t ny, int32_t nz, int32_t tx,
                                                                 int32_t ty, int32_t tz, int32_t curtain, int32_t mode,
                                                                 float* d_out, int32_t device) {
  if (!d_tile_phis || !d_out) return perr(RSFG_ERR_STATE, "merge_phi: null buffer");
  if (mode < 0 || mode > 3) return perr(RSFG_ERR_PARAM, "merge_phi: unknown mode");
  if (cudaSetDevice(device) != cudaSuccess) return perr(RSFG_ERR_CUDA, "merge_phi: bad device");
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return perr(RSFG_ERR_CUDA, "stream");
  const int rc = merge_device(d_tile_phis, n_tiles, nx, ny, nz, tx, ty, tz, curtain, mode, d_out, st);
  cudaStreamDestroy(st);
  return rc;
}

__attribute__((visibility("default"))) void rsfg_pipeline_options_default(rsfg_pipeline_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->global_seeding = 0;  // tiling.hpp:41-47
  o->merge = RSFG_MERGE_LINEAR;
  o->seed_radius = 2.0;
  o->device = 0;
  o->fields = RSFG_FIELDS_2;
  o->spill_dir = nullptr;
}

// run_pipeline (tiling.cpp:201-275) on one GPU: host image in, merged phi and
// mask out (host).  Tiles run one after another, each entirely on the device.
__attribute__((visibility("default"))) int rsfg_run_pipeline(const float* image, int32_t nx, int32_t ny, int32_t nz,
                                                             const rsfg_params* p, const rsfg_blob_params* bp,
                                                             int32_t tx, int32_t ty, int32_t tz,
                                                             const rsfg_pipeline_options* o, float* phi_out,
                                                             float* mask_out, char* warnings, int32_t warnings_cap,
                                                             int32_t* n_warnings) {
  if (!image || !phi_out || !p) return perr(RSFG_ERR_STATE, "run_pipeline: null buffer");
  rsfg_pipeline_options opt;
  rsfg_pipeline_options_default(&opt);
  if (o) opt = *o;
  rsfg_blob_params blob;
  rsfg_blob_params_default(&blob);
  if (bp) blob = *bp;
  if (int rc = rsfg_params_validate(p)) return rc;
  if (!(blob.sigma_b > 0.0)) return perr(RSFG_ERR_PARAM, "BlobParams: sigma_b must be > 0");
  if (blob.response_threshold < 0.0) return perr(RSFG_ERR_PARAM, "BlobParams: response_threshold must be >= 0");
  const double nms = blob.nms_radius > 0.0 ? blob.nms_radius : 2.0 * blob.sigma_b;
  if (nms < 1.0) return perr(RSFG_ERR_PARAM, "BlobParams: nms_radius must be >= 1");
  std::vector<rsfg_tile> tiles;
  int curtain = 0;
  if (int rc = plan(nx, ny, nz, tx, ty, tz, p->sigma1, p->sigma2, tiles, &curtain)) return rc;
  if (cudaSetDevice(opt.device) != cudaSuccess) return perr(RSFG_ERR_CUDA, "run_pipeline: bad device");
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return perr(RSFG_ERR_CUDA, "stream");
  const size_t n = (size_t)nx * ny * nz;
  const bool spill = opt.spill_dir && opt.spill_dir[0];
  const std::string spill_dir = spill ? opt.spill_dir : "";
  float* d_vol = nullptr;
  float* d_out = nullptr;
  std::vector<float*> tphi(tiles.size(), nullptr);
  std::vector<std::string> warn;
  int rc = RSFG_OK;
  auto cleanup = [&]() {
    for (float* q : tphi) cudaFree(q);
    cudaFree(d_vol);
    cudaFree(d_out);
    cudaStreamDestroy(st);
  };
  if (cudaMalloc(&d_vol, n * sizeof(float)) != cudaSuccess) {
    cleanup();
    return perr(RSFG_ERR_OOM, "run_pipeline: out of device memory");
  }
  cudaMemcpyAsync(d_vol, image, n * sizeof(float), cudaMemcpyHostToDevice, st);
  std::vector<rsfg::SeedHost> global;
  if (opt.global_seeding) {
    const int r = rsfg::seed_detect(d_vol, nx, ny, nz, blob.sigma_b, blob.response_threshold, nms, blob.dark != 0,
                                    global, st, nullptr);
    if (r) {
      cleanup();
      return perr(RSFG_ERR_CUDA, "run_pipeline: seed detection failed");
    }
  }
  for (size_t ti = 0; ti < tiles.size() && rc == RSFG_OK; ++ti) {
    const rsfg_tile& t = tiles[ti];
    const int ex = t.pad_extent[0], ey = t.pad_extent[1], ez = t.pad_extent[2];
    const size_t tn = (size_t)ex * ey * ez;
    float* d_tile = nullptr;
    if (cudaMalloc(&tphi[ti], tn * sizeof(float)) != cudaSuccess || cudaMalloc(&d_tile, tn * sizeof(float)) != cudaSuccess) {
      cudaFree(d_tile);
      rc = perr(RSFG_ERR_OOM, "run_pipeline: out of device memory");
      break;
    }
    extract_kernel<<<148 * 4, 256, 0, st>>>(d_vol, nx, ny, d_tile, t.pad_origin[0], t.pad_origin[1], t.pad_origin[2],
                                            ex, ey, ez);
    std::vector<rsfg::SeedHost> seeds;
    if (opt.global_seeding) {  // scatter (tiling.cpp:229-237)
      for (const auto& s : global)
        if (s.x >= t.pad_origin[0] && s.x < t.pad_origin[0] + ex && s.y >= t.pad_origin[1] &&
            s.y < t.pad_origin[1] + ey && s.z >= t.pad_origin[2] && s.z < t.pad_origin[2] + ez)
          seeds.push_back({s.x - t.pad_origin[0], s.y - t.pad_origin[1], s.z - t.pad_origin[2], s.response});
    } else if (ex >= 5 && ey >= 5) {
      if (rsfg::seed_detect(d_tile, ex, ey, ez, blob.sigma_b, blob.response_threshold, nms, blob.dark != 0, seeds, st,
                            nullptr))
        rc = perr(RSFG_ERR_CUDA, "run_pipeline: seed detection failed");
    } else {
      rc = perr(RSFG_ERR_SHAPE, "hessian_det_slice: slice must be at least 5x5");
    }
    if (rc) {
      cudaFree(d_tile);
      break;
    }
    char name[64];
    std::snprintf(name, sizeof name, "tile_z%02d_y%02d_x%02d.vmh", t.iz, t.iy, t.ix);
    if (seeds.empty()) {
      fill_kernel<<<148 * 4, 256, 0, st>>>(tphi[ti], tn, (float)std::max(curtain, 1));
      warn.push_back(std::string("tile ") + name + ": no seeds found; contributing an empty-interior field");
    } else if (rsfg::seed_distance(ex, ey, ez, seeds, (float)opt.seed_radius, tphi[ti], st, nullptr, nullptr)) {
      rc = perr(RSFG_ERR_CUDA, "run_pipeline: distance failed");
    } else {
      // evolve (rsf.cpp:359-384) on the device; nz == 1 tiles take the host
      // entry, which replicates the slice like the reference.
      cudaStreamSynchronize(st);
      rsfg_options eo;
      rsfg_options_default(&eo);
      eo.device = opt.device;
      eo.fields = opt.fields;
      eo.reuse_workspace = 0;
      if (ez == 1) {
        std::vector<float> hp(tn), hi(tn);
        cudaMemcpy(hp.data(), tphi[ti], tn * sizeof(float), cudaMemcpyDeviceToHost);
        cudaMemcpy(hi.data(), d_tile, tn * sizeof(float), cudaMemcpyDeviceToHost);
        const int e = rsfg_evolve(hi.data(), hp.data(), ex, ey, ez, p, &eo, nullptr, nullptr, 0, nullptr);
        if (e) rc = perr(e, rsfg_last_error());
        else cudaMemcpy(tphi[ti], hp.data(), tn * sizeof(float), cudaMemcpyHostToDevice);
      } else {
        rsfg_state* s = nullptr;
        int e = rsfg_state_create_device(&s, tphi[ti], d_tile, ex, ey, ez, p, &eo);
        for (int it = 0; !e && it < p->max_iters; ++it) {
          double frac = 0.0;
          if (p->convergence_fraction > 0.0) {
            e = rsfg_state_step(s, &frac);
            if (!e && frac < p->convergence_fraction) break;
          } else {
            rsfg_report rep;
            e = rsfg_state_run(s, p->max_iters, &rep);
            break;
          }
        }
        float* d_final = nullptr;
        if (!e) e = rsfg_state_device_phi(s, &d_final);
        if (!e) {
          cudaMemcpy(tphi[ti], d_final, tn * sizeof(float), cudaMemcpyDeviceToDevice);
        } else {
          rc = perr(e, rsfg_last_error());
        }
        if (s) rsfg_state_destroy(s);
      }
    }
    cudaFree(d_tile);
    // tiling.cpp:256-259: the tile's phi goes to spill_dir as it completes
    if (rc == RSFG_OK && spill) {
      if (cudaStreamSynchronize(st) != cudaSuccess) {
        rc = perr(RSFG_ERR_CUDA, "run_pipeline: CUDA error");
      } else {
        const int e = rsfg_write_volume_device((spill_dir + "/" + name).c_str(), tphi[ti], ex, ey, ez, nullptr,
                                               nullptr, opt.device);
        if (e) rc = perr(e, rsfg_last_error());
      }
    }
  }
  // tiling.cpp:262-263: the manifest once every tile is on disk
  if (rc == RSFG_OK && spill) {
    const int e = rsfg_save_manifest((spill_dir + "/layout.manifest").c_str(), nx, ny, nz, tx, ty, tz, curtain,
                                     tiles.data(), (int32_t)tiles.size());
    if (e) rc = e;
  }
  if (rc == RSFG_OK) {
    if (cudaMalloc(&d_out, n * sizeof(float)) != cudaSuccess) {
      rc = perr(RSFG_ERR_OOM, "run_pipeline: out of device memory");
    } else {
      rc = merge_device(tphi.data(), (int)tphi.size(), nx, ny, nz, tx, ty, tz, curtain, opt.merge, d_out, st);
    }
  }
  if (rc == RSFG_OK) {
    cudaMemcpyAsync(phi_out, d_out, n * sizeof(float), cudaMemcpyDeviceToHost, st);
    if (mask_out) {
      rsfg::launch_mask(d_out, d_vol, (long long)n, st);  // d_vol reused as the mask buffer
      cudaMemcpyAsync(mask_out, d_vol, n * sizeof(float), cudaMemcpyDeviceToHost, st);
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) rc = perr(RSFG_ERR_CUDA, "run_pipeline: CUDA error");
  }
  std::sort(warn.begin(), warn.end());
  if (n_warnings) *n_warnings = (int32_t)warn.size();
  if (warnings && warnings_cap > 0) {
    std::string all;
    for (const auto& w : warn) all += w + "\n";
    std::snprintf(warnings, warnings_cap, "%s", all.c_str());
  }
  cleanup();
  return rc;
}

__attribute__((visibility("default"))) int rsfg_tile_file_name(const rsfg_tile* t, char* buf, int32_t cap) {
  if (!t || !buf || cap <= 0) return perr(RSFG_ERR_STATE, "tile_file_name: null buffer");
  const int k = std::snprintf(buf, cap, "tile_z%02d_y%02d_x%02d.vmh", t->iz, t->iy, t->ix);
  return k < cap ? RSFG_OK : perr(RSFG_ERR_STATE, "tile_file_name: buffer too small");
}

// save_manifest (tiling.cpp:277-295): same keys, order and spacing.
__attribute__((visibility("default"))) int rsfg_save_manifest(const char* path, int32_t nx, int32_t ny, int32_t nz,
                                                              int32_t tx, int32_t ty, int32_t tz, int32_t curtain,
                                                              const rsfg_tile* tiles, int32_t n_tiles) {
  const std::string ps = path ? path : "";
  std::ofstream out(ps, std::ios::trunc);
  if (!out) return perr(RSFG_ERR_IO, "cannot write manifest: " + ps);
  out << "dims: " << nx << " " << ny << " " << nz << "\n";
  out << "tile_size: " << tx << " " << ty << " " << tz << "\n";
  out << "curtain: " << curtain << "\n";
  for (int32_t i = 0; i < n_tiles; ++i) {
    const rsfg_tile& t = tiles[i];
    out << "tile: " << t.ix << " " << t.iy << " " << t.iz;
    for (const int32_t* a : {t.core_origin, t.core_extent, t.pad_origin, t.pad_extent})
      out << " " << a[0] << " " << a[1] << " " << a[2];
    out << "\n";
  }
  if (!out) return perr(RSFG_ERR_IO, "short write to manifest: " + ps);
  return RSFG_OK;
}

namespace {
int load_manifest(const std::string& ps, int32_t* dims3, int32_t* tile3, int32_t* curtain,
                  std::vector<rsfg_tile>& tiles) {
  std::ifstream in(ps);
  if (!in) return perr(RSFG_ERR_IO, "cannot open manifest: " + ps);
  int d[3] = {0, 0, 0}, ts[3] = {0, 0, 0}, c = 0;
  std::string line;
  while (std::getline(in, line)) {  // tiling.cpp:297-321
    if (line.empty() || line[0] == '#') continue;
    std::istringstream ls(line);
    std::string key;
    ls >> key;
    if (key == "dims:") {
      ls >> d[0] >> d[1] >> d[2];
    } else if (key == "tile_size:") {
      ls >> ts[0] >> ts[1] >> ts[2];
    } else if (key == "curtain:") {
      ls >> c;
    } else if (key == "tile:") {
      rsfg_tile t;
      ls >> t.ix >> t.iy >> t.iz;
      for (int32_t* a : {t.core_origin, t.core_extent, t.pad_origin, t.pad_extent}) ls >> a[0] >> a[1] >> a[2];
      tiles.push_back(t);
    } else {
      return perr(RSFG_ERR_IO, "unknown manifest key '" + key + "' in " + ps);
    }
    if (!ls) return perr(RSFG_ERR_IO, "garbled manifest line in " + ps + ": " + line);
  }
  if (tiles.empty()) return perr(RSFG_ERR_IO, "manifest has no tiles: " + ps);
  for (int k = 0; k < 3; ++k) {
    if (dims3) dims3[k] = d[k];
    if (tile3) tile3[k] = ts[k];
  }
  if (curtain) *curtain = c;
  return RSFG_OK;
}
}  // namespace

__attribute__((visibility("default"))) int rsfg_load_manifest(const char* path, int32_t* dims3, int32_t* tile_size3,
                                                              int32_t* curtain, rsfg_tile* tiles, int32_t cap,
                                                              int32_t* n_tiles) {
  std::vector<rsfg_tile> v;
  if (int rc = load_manifest(path ? path : "", dims3, tile_size3, curtain, v)) return rc;
  if (n_tiles) *n_tiles = (int32_t)v.size();
  for (size_t i = 0; tiles && i < v.size() && (int32_t)i < cap; ++i) tiles[i] = v[i];
  return RSFG_OK;
}

// merge_from_dir (tiling.cpp:323-332): each tile file is read straight into a
// device buffer (rsfg_read_volume_device), then one device merge.
__attribute__((visibility("default"))) int rsfg_merge_from_dir(const char* dir, int32_t nx, int32_t ny, int32_t nz,
                                                               int32_t tx, int32_t ty, int32_t tz, int32_t curtain,
                                                               const rsfg_tile* layout_tiles, int32_t n_tiles,
                                                               int32_t mode, float* d_out, int32_t device) {
  if (!dir || !layout_tiles || !d_out) return perr(RSFG_ERR_STATE, "merge_from_dir: null argument");
  if (mode < 0 || mode > 3) return perr(RSFG_ERR_PARAM, "merge_phi: unknown mode");
  const int32_t d[3] = {nx, ny, nz}, ts[3] = {tx, ty, tz};
  const std::vector<rsfg_tile> tiles(layout_tiles, layout_tiles + std::max(n_tiles, 0));
  if (cudaSetDevice(device) != cudaSuccess) return perr(RSFG_ERR_CUDA, "merge_from_dir: bad device");
  std::vector<float*> tphi(tiles.size(), nullptr);
  int rc = RSFG_OK;
  for (size_t i = 0; i < tiles.size() && !rc; ++i) {
    const rsfg_tile& t = tiles[i];
    const int64_t tn = (int64_t)t.pad_extent[0] * t.pad_extent[1] * t.pad_extent[2];
    char name[64];
    rsfg_tile_file_name(&t, name, sizeof name);
    const std::string hp = std::string(dir) + "/" + name;
    int32_t fx = 0, fy = 0, fz = 0, eb = 0;
    double sp[3];
    if ((rc = rsfg_volume_info(hp.c_str(), &fx, &fy, &fz, sp, &eb))) break;
    if (fx != t.pad_extent[0] || fy != t.pad_extent[1] || fz != t.pad_extent[2]) {
      rc = perr(RSFG_ERR_SHAPE, "merge_phi: tile " + std::string(name) + " dims do not match its box");
      break;
    }
    if (cudaMalloc(&tphi[i], tn * sizeof(float)) != cudaSuccess) {
      rc = perr(RSFG_ERR_OOM, "merge_from_dir: out of device memory");
      break;
    }
    rc = rsfg_read_volume_device(hp.c_str(), tphi[i], tn, device, nullptr, nullptr);
  }
  if (!rc) {
    cudaStream_t st;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
      rc = perr(RSFG_ERR_CUDA, "stream");
    } else {
      rc = merge_device(tphi.data(), (int)tphi.size(), d[0], d[1], d[2], ts[0], ts[1], ts[2], curtain, mode, d_out,
                        st);
      cudaStreamDestroy(st);
    }
  }
  for (float* q : tphi) cudaFree(q);
  return rc;
}

// Same with a HOST output buffer (the reference's merge_from_dir returns a
// host Volume): merged on the device, one D2H.
__attribute__((visibility("default"))) int rsfg_merge_from_dir_host(const char* dir, int32_t nx, int32_t ny,
                                                                    int32_t nz, int32_t tx, int32_t ty, int32_t tz,
                                                                    int32_t curtain, const rsfg_tile* tiles,
                                                                    int32_t n_tiles, int32_t mode, float* out,
                                                                    int32_t device) {
  if (!out) return perr(RSFG_ERR_STATE, "merge_from_dir: null argument");
  if (nx <= 0 || ny <= 0 || nz <= 0) return perr(RSFG_ERR_SHAPE, "merge_from_dir: bad volume dims");
  if (cudaSetDevice(device) != cudaSuccess) return perr(RSFG_ERR_CUDA, "merge_from_dir: bad device");
  const size_t bytes = (size_t)nx * ny * nz * sizeof(float);
  float* d_out = nullptr;
  if (cudaMalloc(&d_out, bytes) != cudaSuccess) return perr(RSFG_ERR_OOM, "merge_from_dir: out of device memory");
  int rc = rsfg_merge_from_dir(dir, nx, ny, nz, tx, ty, tz, curtain, tiles, n_tiles, mode, d_out, device);
  if (!rc && cudaMemcpy(out, d_out, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = perr(RSFG_ERR_CUDA, "merge_from_dir: CUDA error");
  cudaFree(d_out);
  return rc;
}

}  // extern "C"
