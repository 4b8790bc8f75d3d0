// rsfg_zst4_g0.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [0, 1, 2];
// split across translation units so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {

int zst4_group_box_0(int r, int fields, int* pbox_z, int* ty) {
  switch (r) {
    case 0:
      *pbox_z = Z4<0, 1>::NW;
      *ty = fields == 4 ? Z4<0, 2>::TY : Z4<0, 1>::TY;  // box rows = the launched kernel's tile
      return (fields == 4 ? Z4<0, 2>::kSmem : Z4<0, 1>::kSmem) <= 227 * 1024;
    case 1:
      *pbox_z = Z4<1, 1>::NW;
      *ty = fields == 4 ? Z4<1, 2>::TY : Z4<1, 1>::TY;  // box rows = the launched kernel's tile
      return (fields == 4 ? Z4<1, 2>::kSmem : Z4<1, 1>::kSmem) <= 227 * 1024;
    case 2:
      *pbox_z = Z4<2, 1>::NW;
      *ty = fields == 4 ? Z4<2, 2>::TY : Z4<2, 1>::TY;  // box rows = the launched kernel's tile
      return (fields == 4 ? Z4<2, 2>::kSmem : Z4<2, 1>::kSmem) <= 227 * 1024;
    default:
      return -2;
  }
}

int zst4_group_0(int r, const Geom& g, int fields, const Taps& t1, const StepConsts& c, const StepBuffers& b,
                  int z_begin, int z_end, const ZMaps& m, cudaStream_t st) {
  switch (r) {
    case 0:
      return fields == 4 ? zst4_launch<0, 2>(g, t1, c, b, z_begin, z_end, m, st)
                         : zst4_launch<0, 1>(g, t1, c, b, z_begin, z_end, m, st);
    case 1:
      return fields == 4 ? zst4_launch<1, 2>(g, t1, c, b, z_begin, z_end, m, st)
                         : zst4_launch<1, 1>(g, t1, c, b, z_begin, z_end, m, st);
    case 2:
      return fields == 4 ? zst4_launch<2, 2>(g, t1, c, b, z_begin, z_end, m, st)
                         : zst4_launch<2, 1>(g, t1, c, b, z_begin, z_end, m, st);
    default:
      return -2;
  }
}

}  // namespace rsfg
