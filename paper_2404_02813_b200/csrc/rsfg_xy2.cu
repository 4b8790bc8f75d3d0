// rsfg_xy2.cu -- dispatch of kernel 1's multi-plane TMA variant
// (rsfg_xy2.cuh) over the per-radius-group translation units rsfg_xy2_g*.cu.
#include "rsfg_xy2.cuh"

namespace rsfg {

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
