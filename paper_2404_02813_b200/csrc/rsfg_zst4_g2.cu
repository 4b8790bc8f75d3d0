// rsfg_zst4_g2.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [5, 6];
// split across translation units so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {

int zst4_group_box_2(int r, int fields, int* pbox_z, int* ty) {
  switch (r) {
    case 5:
      *pbox_z = Z4<5, 1>::NW;
      *ty = fields == 4 ? Z4<5, 2>::TY : Z4<5, 1>::TY;  // box rows = the launched kernel's tile
      return (fields == 4 ? Z4<5, 2>::kSmem : Z4<5, 1>::kSmem) <= 227 * 1024;
    case 6:
      *pbox_z = Z4<6, 1>::NW;
      *ty = fields == 4 ? Z4<6, 2>::TY : Z4<6, 1>::TY;  // box rows = the launched kernel's tile
      return (fields == 4 ? Z4<6, 2>::kSmem : Z4<6, 1>::kSmem) <= 227 * 1024;
    default:
      return -2;
  }
}

int zst4_group_2(int r, const Geom& g, int fields, const Taps& t1, const StepConsts& c, const StepBuffers& b,
                  int z_begin, int z_end, const ZMaps& m, cudaStream_t st) {
  switch (r) {
    case 5:
      return fields == 4 ? zst4_launch<5, 2>(g, t1, c, b, z_begin, z_end, m, st)
                         : zst4_launch<5, 1>(g, t1, c, b, z_begin, z_end, m, st);
    case 6:
      return fields == 4 ? zst4_launch<6, 2>(g, t1, c, b, z_begin, z_end, m, st)
                         : zst4_launch<6, 1>(g, t1, c, b, z_begin, z_end, m, st);
    default:
      return -2;
  }
}

}  // namespace rsfg
