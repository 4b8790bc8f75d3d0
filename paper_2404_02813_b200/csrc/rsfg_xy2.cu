// rsfg_xy2.cu -- dispatch of kernel 1's multi-plane TMA variant
// (rsfg_xy2.cuh) over the per-radius-group translation units rsfg_xy2_g*.cu.
#include "rsfg_xy2.cuh"

namespace rsfg {

// Whether xy2's kernel for (r, fields, ty) fits shared memory (setup uses it
// to pick the fast path; large radii with fields=4 can exceed 227 KB).
bool xy2_fits(int r, int fields, int ty) {
  switch (r) {
#define CASE(R)                                                                                     \
  case R:                                                                                           \
    if (ty == 64) return fields == 2 && R <= 18 && XY2<R, 1, 64>::kSmem <= 227 * 1024;              \
    return (fields == 4 ? XY2<R, 2, 32>::kSmem : XY2<R, 1, 32>::kSmem) <= 227 * 1024;
    RSFG_RADII(CASE)
#undef CASE
    default:
      return false;
  }
}

bool xy2_box(int r, int ty, int* bx, int* by) {
  int rc = -2;
#define TRY(N) \
  if (rc == -2) rc = xy2_group_box_##N(r, ty, bx, by);
  RSFG_XY2_GROUPS(TRY)
#undef TRY
  return rc == 1;
}

int launch_xy2(const Geom& g, int fields, int ty, const Taps& t1, float inv_eps, float2* P0, float2* P1,
               int z_begin, int z_end, const XYMaps& m, cudaStream_t st) {
  if (!m.valid) return -1;
  int rc = -2;
#define TRY(N) \
  if (rc == -2) rc = xy2_group_##N(t1.r, ty, g, fields, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
  RSFG_XY2_GROUPS(TRY)
#undef TRY
  return rc == -2 ? -1 : rc;
}

}  // namespace rsfg
