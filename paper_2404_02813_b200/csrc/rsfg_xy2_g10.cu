// rsfg_xy2_g10.cu -- xy2 (rsfg_xy2.cuh) instantiations for radii [21, 22];
// one translation unit per radius group so the build parallelises.
#include "rsfg_xy2.cuh"

namespace rsfg {
#define RADII(X) X(21) X(22)
RSFG_XY2_GROUP(10, RADII)
}  // namespace rsfg
