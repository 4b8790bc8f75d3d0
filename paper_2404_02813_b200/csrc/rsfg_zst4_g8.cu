// rsfg_zst4_g8.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [18];
// split across translation units so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {

int zst4_group_box_8(int r, int fields, int* pbox_z, int* ty) {
  switch (r) {
    case 18:
      *pbox_z = Z4<18, 1>::NW;
      *ty = fields == 4 ? Z4<18, 2>::TY : Z4<18, 1>::TY;  // box rows = the launched kernel's tile
      return (fields == 4 ? Z4<18, 2>::kSmem : Z4<18, 1>::kSmem) <= 227 * 1024;
    default:
      return -2;
  }
}

int zst4_group_8(int r, const Geom& g, int fields, const Taps& t1, const StepConsts& c, const StepBuffers& b,
                  int z_begin, int z_end, const ZMaps& m, cudaStream_t st) {
  switch (r) {
    case 18:
      return fields == 4 ? zst4_launch<18, 2>(g, t1, c, b, z_begin, z_end, m, st)
                         : zst4_launch<18, 1>(g, t1, c, b, z_begin, z_end, m, st);
    default:
      return -2;
  }
}

}  // namespace rsfg
