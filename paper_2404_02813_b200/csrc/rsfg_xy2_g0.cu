// rsfg_xy2_g0.cu -- xy2 (rsfg_xy2.cuh) instantiations for radii [0, 1, 2, 3, 4];
// one translation unit per radius group so the build parallelises.
#include "rsfg_xy2.cuh"

namespace rsfg {
#define RADII(X) X(0) X(1) X(2) X(3) X(4)
RSFG_XY2_GROUP(0, RADII)
}  // namespace rsfg
