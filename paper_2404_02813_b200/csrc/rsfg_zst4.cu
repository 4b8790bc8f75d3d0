// rsfg_zst4.cu -- dispatch of kernel 2's TMA-fed variant (rsfg_zst4.cuh)
// over the per-radius-group translation units rsfg_zst4_g*.cu.
#include "rsfg_zst4.cuh"

namespace rsfg {

bool zst4_box(int r, int fields, int* pbox_z, int* ty) {
  int rc = -2;
#define TRY(N) \
  if (rc == -2) rc = zst4_group_box_##N(r, fields, pbox_z, ty);
  RSFG_ZST4_GROUPS(TRY)
#undef TRY
  return rc == 1;
}

int launch_zst4(const Geom& g, int fields, const Taps& t1, const StepConsts& c, const StepBuffers& b, int z_begin,
                int z_end, const ZMaps& m, cudaStream_t st) {
  if (!m.valid) return -1;
  int rc = -2;
#define TRY(N) \
  if (rc == -2) rc = zst4_group_##N(t1.r, g, fields, t1, c, b, z_begin, z_end, m, st);
  RSFG_ZST4_GROUPS(TRY)
#undef TRY
  return rc == -2 ? -1 : rc;
}

}  // namespace rsfg
