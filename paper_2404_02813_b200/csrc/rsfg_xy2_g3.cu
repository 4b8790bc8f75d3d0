// rsfg_xy2_g3.cu -- xy2 (rsfg_xy2.cuh) instantiations for radii [10, 11];
// split across translation units so the build parallelises.
#include "rsfg_xy2.cuh"

namespace rsfg {

int xy2_group_box_3(int r, int ty, int* bx, int* by) {
  switch (r) {
    case 10:
      *bx = ty == 64 ? XY2<10, 1, 64>::BOXX : XY2<10, 1, 32>::BOXX;
      *by = ty == 64 ? XY2<10, 1, 64>::WY : XY2<10, 1, 32>::WY;
      return 1;
    case 11:
      *bx = ty == 64 ? XY2<11, 1, 64>::BOXX : XY2<11, 1, 32>::BOXX;
      *by = ty == 64 ? XY2<11, 1, 64>::WY : XY2<11, 1, 32>::WY;
      return 1;
    default:
      return -2;
  }
}

int xy2_group_3(int r, int ty, const Geom& g, int fields, const Taps& t1, float inv_eps, float2* P0, float2* P1,
                 int z_begin, int z_end, const XYMaps& m, cudaStream_t st) {
  switch (r) {
    case 10:
      if (ty == 64)  // 64 x 64 tiles: fields=2 only (the fields=4 tile exceeds shared memory)
        return fields == 4 ? -1 : xy2_launch<10, 1, 64>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
      return fields == 4 ? xy2_launch<10, 2, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st)
                         : xy2_launch<10, 1, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
    case 11:
      if (ty == 64)  // 64 x 64 tiles: fields=2 only (the fields=4 tile exceeds shared memory)
        return fields == 4 ? -1 : xy2_launch<11, 1, 64>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
      return fields == 4 ? xy2_launch<11, 2, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st)
                         : xy2_launch<11, 1, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
    default:
      return -2;
  }
}

}  // namespace rsfg
