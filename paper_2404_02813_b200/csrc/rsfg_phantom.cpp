// rsfg_phantom.cpp -- synthetic tube-network inputs.
//
// Host restatement of the reference generator so the benchmark and the
// GPU-box tests can make inputs without the reference: random-walk
// centerlines with bounded-curvature jitter, a swept-ball signed distance,
// 1-voxel anti-aliased edges, optional axial blur (phantom.cpp:55-184), then
// Gaussian noise and an intensity ramp (phantom.cpp:186-214).  Randomness is
// the reference's SplitMix64 + Box-Muller (rng.hpp:10-60), so a spec yields
// the same volume as rsf::generate_network + rsf::perturb (checked in
// tests/test_phantom.py against the compiled reference).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/rsfg.h"

namespace {

class Rng {  // rng.hpp:10-60
 public:
  explicit Rng(uint64_t seed) : s_(seed) {}
  uint64_t next() {
    uint64_t z = (s_ += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double u01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * u01(); }
  uint64_t below(uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t v;
    do v = next();
    while (v >= limit);
    return v % n;
  }
  double normal() {
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    double a;
    do a = u01();
    while (a <= 0.0);
    const double b = u01();
    const double rad = std::sqrt(-2.0 * std::log(a));
    const double ang = 2.0 * M_PI * b;
    spare_ = rad * std::sin(ang);
    spare_ok_ = true;
    return rad * std::cos(ang);
  }

 private:
  uint64_t s_;
  bool spare_ok_ = false;
  double spare_ = 0.0;
};

struct V3 {
  double x, y, z;
};
struct Sample {
  V3 p;
  double r;
};

V3 unit(V3 v) {
  const double n = std::sqrt(v.x * v.x + v.y * v.y + v.z * v.z);
  if (n < 1e-12) return {1, 0, 0};
  return {v.x / n, v.y / n, v.z / n};
}

thread_local std::string g_perr;

}  // namespace

struct rsfg_phantom_sample {
  double x, y, z, r;
};

extern "C" {

__attribute__((visibility("default"))) void rsfg_phantom_default(rsfg_phantom_spec* s) {
  if (!s) return;
  std::memset(s, 0, sizeof *s);
  s->nx = 128;
  s->ny = 128;
  s->nz = 128;
  s->n_branches = 12;
  s->radius_min = 2.0;
  s->radius_max = 4.0;
  s->tortuosity = 0.25;
  s->foreground = 200.0f;
  s->background = 50.0f;
  s->rng_seed = 1;
  s->tree_connected = 1;
  s->axial_blur_sigma = 0.0;
  s->noise_sigma = 20.0;
  s->contrast_axis = 0;
  s->contrast_lo = 1.0;
  s->contrast_hi = 1.0;
  s->noise_seed = 7;
}

}  // extern "C"

// PhantomSpec::validate / PerturbSpec::validate (phantom.cpp:12-34) and the
// random-walk centerlines (phantom.cpp:55-112): serial in the RNG, cheap.
// Returns the swept-ball samples in generation order.
int phantom_centerlines(const rsfg_phantom_spec* s, std::vector<Sample>& all_out) {
  const int nx = s->nx, ny = s->ny, nz = s->nz;
  // PhantomSpec::validate / PerturbSpec::validate (phantom.cpp:12-34)
  if (nx <= 0 || ny <= 0 || nz <= 0 || s->n_branches < 0 || s->radius_min < 1.0 ||
      s->radius_max < s->radius_min || s->foreground == s->background || s->tortuosity < 0.0 ||
      s->axial_blur_sigma < 0.0 || s->noise_sigma < 0.0 || !(s->contrast_lo > 0.0) ||
      s->contrast_hi < s->contrast_lo)
    return RSFG_ERR_PARAM;
  const bool flat = nz == 1;
  const double margin = s->radius_max + 2.0;
  if (2.0 * margin >= std::min(nx, ny) || (nz > 1 && 2.0 * margin >= nz)) return RSFG_ERR_PARAM;

  Rng rng(s->rng_seed);
  const double step = 0.5;
  const double lox = margin, hix = nx - 1 - margin, loy = margin, hiy = ny - 1 - margin;
  const double loz = flat ? 0.0 : margin, hiz = flat ? 0.0 : nz - 1 - margin;
  std::vector<Sample>& all = all_out;
  all.clear();
  for (int b = 0; b < s->n_branches; ++b) {
    V3 pos;
    if (s->tree_connected && !all.empty()) {
      pos = all[rng.below(all.size())].p;
    } else {
      // evaluation order of the braced initialiser is left to right
      const double px = rng.uniform(lox, hix);
      const double py = rng.uniform(loy, hiy);
      const double pz = flat ? 0.0 : rng.uniform(loz, hiz);
      pos = {px, py, pz};
    }
    V3 dir;
    if (flat) {
      const double a = rng.uniform(0.0, 2.0 * M_PI);
      dir = {std::cos(a), std::sin(a), 0.0};
    } else {
      const double a = rng.normal(), bb = rng.normal(), c = rng.normal();
      dir = unit({a, bb, c});
    }
    const double r0 = rng.uniform(s->radius_min, s->radius_max);
    const double r1 = rng.uniform(s->radius_min, s->radius_max);
    const double length = rng.uniform(0.4, 0.9) * std::max(nx, ny);
    const int n_steps = std::max(2, static_cast<int>(length / step));
    std::vector<Sample> path;
    path.reserve(n_steps);
    for (int k = 0; k < n_steps; ++k) {
      const double t = static_cast<double>(k) / (n_steps - 1);
      path.push_back({pos, r0 + t * (r1 - r0)});
      const double jx = rng.normal(), jy = rng.normal();
      const double jz = flat ? 0.0 : rng.normal();
      dir = unit({dir.x + s->tortuosity * step * jx, dir.y + s->tortuosity * step * jy,
                  dir.z + s->tortuosity * step * jz});
      const V3 nxt{pos.x + step * dir.x, pos.y + step * dir.y, pos.z + step * dir.z};
      if (nxt.x < lox || nxt.x > hix) dir.x = -dir.x;
      if (nxt.y < loy || nxt.y > hiy) dir.y = -dir.y;
      if (!flat && (nxt.z < loz || nxt.z > hiz)) dir.z = -dir.z;
      pos = {std::clamp(pos.x + step * dir.x, lox, hix), std::clamp(pos.y + step * dir.y, loy, hiy),
             flat ? 0.0 : std::clamp(pos.z + step * dir.z, loz, hiz)};
    }
    all.insert(all.end(), path.begin(), path.end());
  }
  return RSFG_OK;
}

extern "C" {

__attribute__((visibility("default"))) int rsfg_phantom(const rsfg_phantom_spec* s, float* image, float* gt) {
  if (!s || !image) return RSFG_ERR_STATE;
  std::vector<Sample> all;
  if (int rc = phantom_centerlines(s, all)) return rc;
  const int nx = s->nx, ny = s->ny, nz = s->nz;
  const bool flat = nz == 1;

  const size_t n = (size_t)nx * ny * nz;
  std::vector<float> dist(n, std::numeric_limits<float>::max());
  // Order-independent min over samples (the reference rasterises branch by
  // branch, phantom.cpp:113-137; min is exact in any order).
  for (const Sample& q : all) {
      const int x0 = std::max(0, (int)std::floor(q.p.x - q.r - 1.5));
      const int x1 = std::min(nx - 1, (int)std::ceil(q.p.x + q.r + 1.5));
      const int y0 = std::max(0, (int)std::floor(q.p.y - q.r - 1.5));
      const int y1 = std::min(ny - 1, (int)std::ceil(q.p.y + q.r + 1.5));
      const int z0 = flat ? 0 : std::max(0, (int)std::floor(q.p.z - q.r - 1.5));
      const int z1 = flat ? 0 : std::min(nz - 1, (int)std::ceil(q.p.z + q.r + 1.5));
      for (int z = z0; z <= z1; ++z)
        for (int y = y0; y <= y1; ++y)
          for (int x = x0; x <= x1; ++x) {
            const double dx = x - q.p.x, dy = y - q.p.y, dz = z - q.p.z;
            const float d = (float)(std::sqrt(dx * dx + dy * dy + dz * dz) - q.r);
            float& cur = dist[(size_t)x + (size_t)nx * ((size_t)y + (size_t)ny * z)];
            cur = std::min(cur, d);
          }
  }

  std::vector<float> img(n);
  const float f = s->foreground, bgv = s->background;
  for (size_t i = 0; i < n; ++i) {
    const float d = dist[i];
    const float a = std::clamp(0.5f - d, 0.0f, 1.0f);
    img[i] = bgv + (f - bgv) * a;
    if (gt) gt[i] = d < 0.0f ? 1.0f : 0.0f;
  }
  if (s->axial_blur_sigma > 0.0 && !flat) {
    // z-only Gaussian blur with clamp (phantom.cpp:150-166); weights as gaussian_kernel.
    const int r = (int)std::ceil(3.0 * s->axial_blur_sigma);
    std::vector<double> w(2 * r + 1);
    double sum = 0.0;
    for (int i = -r; i <= r; ++i) {
      w[i + r] = std::exp(-((double)i * i) / (2.0 * s->axial_blur_sigma * s->axial_blur_sigma));
      sum += w[i + r];
    }
    for (double& v : w) v /= sum;
    std::vector<float> out(n);
    const size_t plane = (size_t)nx * ny;
    for (int z = 0; z < nz; ++z)
      for (size_t xy = 0; xy < plane; ++xy) {
        double acc = 0.0;
        for (int j = -r; j <= r; ++j) acc += w[j + r] * img[xy + plane * std::clamp(z + j, 0, nz - 1)];
        out[xy + plane * z] = (float)acc;
      }
    img.swap(out);
  }

  // perturb (phantom.cpp:186-214)
  Rng nr(s->noise_seed);
  const double lo = s->contrast_lo, hi = s->contrast_hi;
  auto ramp = [&](int i, int m) { return m <= 1 ? 0.5 * (lo + hi) : lo + (hi - lo) * (double)i / (m - 1); };
  size_t i = 0;
  for (int z = 0; z < nz; ++z)
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x, ++i) {
        double v = img[i];
        if (s->noise_sigma > 0.0) v += s->noise_sigma * nr.normal();
        double m = 1.0;
        if (s->contrast_axis == 1) m = ramp(x, nx);
        if (s->contrast_axis == 2) m = ramp(y, ny);
        if (s->contrast_axis == 3) m = ramp(z, nz);
        image[i] = (float)std::clamp(v * m, 0.0, 255.0);
      }
  return RSFG_OK;
}

}  // extern "C"

// Centerline samples as plain (x, y, z, r) doubles for the device rasteriser.
int rsfg_phantom_samples_host(const rsfg_phantom_spec* s, std::vector<rsfg_phantom_sample>& out) {
  std::vector<Sample> all;
  if (int rc = phantom_centerlines(s, all)) return rc;
  out.resize(all.size());
  for (size_t i = 0; i < all.size(); ++i) out[i] = {all[i].p.x, all[i].p.y, all[i].p.z, all[i].r};
  return RSFG_OK;
}
