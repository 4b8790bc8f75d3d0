// rsfg_xy2_g0.cu -- xy2 (rsfg_xy2.cuh) instantiations for radii [0, 1, 2, 3, 4];
// split across translation units so the build parallelises.
#include "rsfg_xy2.cuh"

namespace rsfg {

int xy2_group_box_0(int r, int ty, int* bx, int* by) {
  switch (r) {
    case 0:
      *bx = ty == 64 ? XY2<0, 1, 64>::BOXX : XY2<0, 1, 32>::BOXX;
      *by = ty == 64 ? XY2<0, 1, 64>::WY : XY2<0, 1, 32>::WY;
      return 1;
    case 1:
      *bx = ty == 64 ? XY2<1, 1, 64>::BOXX : XY2<1, 1, 32>::BOXX;
      *by = ty == 64 ? XY2<1, 1, 64>::WY : XY2<1, 1, 32>::WY;
      return 1;
    case 2:
      *bx = ty == 64 ? XY2<2, 1, 64>::BOXX : XY2<2, 1, 32>::BOXX;
      *by = ty == 64 ? XY2<2, 1, 64>::WY : XY2<2, 1, 32>::WY;
      return 1;
    case 3:
      *bx = ty == 64 ? XY2<3, 1, 64>::BOXX : XY2<3, 1, 32>::BOXX;
      *by = ty == 64 ? XY2<3, 1, 64>::WY : XY2<3, 1, 32>::WY;
      return 1;
    case 4:
      *bx = ty == 64 ? XY2<4, 1, 64>::BOXX : XY2<4, 1, 32>::BOXX;
      *by = ty == 64 ? XY2<4, 1, 64>::WY : XY2<4, 1, 32>::WY;
      return 1;
    default:
      return -2;
  }
}

int xy2_group_0(int r, int ty, const Geom& g, int fields, const Taps& t1, float inv_eps, float2* P0, float2* P1,
                 int z_begin, int z_end, const XYMaps& m, cudaStream_t st) {
  switch (r) {
    case 0:
      if (ty == 64)  // 64 x 64 tiles: fields=2 only (the fields=4 tile exceeds shared memory)
        return fields == 4 ? -1 : xy2_launch<0, 1, 64>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
      return fields == 4 ? xy2_launch<0, 2, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st)
                         : xy2_launch<0, 1, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
    case 1:
      if (ty == 64)  // 64 x 64 tiles: fields=2 only (the fields=4 tile exceeds shared memory)
        return fields == 4 ? -1 : xy2_launch<1, 1, 64>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
      return fields == 4 ? xy2_launch<1, 2, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st)
                         : xy2_launch<1, 1, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
    case 2:
      if (ty == 64)  // 64 x 64 tiles: fields=2 only (the fields=4 tile exceeds shared memory)
        return fields == 4 ? -1 : xy2_launch<2, 1, 64>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
      return fields == 4 ? xy2_launch<2, 2, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st)
                         : xy2_launch<2, 1, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
    case 3:
      if (ty == 64)  // 64 x 64 tiles: fields=2 only (the fields=4 tile exceeds shared memory)
        return fields == 4 ? -1 : xy2_launch<3, 1, 64>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
      return fields == 4 ? xy2_launch<3, 2, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st)
                         : xy2_launch<3, 1, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
    case 4:
      if (ty == 64)  // 64 x 64 tiles: fields=2 only (the fields=4 tile exceeds shared memory)
        return fields == 4 ? -1 : xy2_launch<4, 1, 64>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
      return fields == 4 ? xy2_launch<4, 2, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st)
                         : xy2_launch<4, 1, 32>(g, t1, inv_eps, P0, P1, z_begin, z_end, m, st);
    default:
      return -2;
  }
}

}  // namespace rsfg
