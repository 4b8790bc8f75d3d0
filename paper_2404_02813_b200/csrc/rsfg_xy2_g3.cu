// rsfg_xy2_g3.cu -- xy2 (rsfg_xy2.cuh) instantiations for radii [10, 11];
// one translation unit per radius group so the build parallelises.
#include "rsfg_xy2.cuh"

namespace rsfg {
#define RADII(X) X(10) X(11)
RSFG_XY2_GROUP(3, RADII)
}  // namespace rsfg
