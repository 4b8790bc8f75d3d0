// rsfg_xy2_g11.cu -- xy2 (rsfg_xy2.cuh) instantiations for radii [23, 24];
// one translation unit per radius group so the build parallelises.
#include "rsfg_xy2.cuh"

namespace rsfg {
#define RADII(X) X(23) X(24)
RSFG_XY2_GROUP(11, RADII)
}  // namespace rsfg
