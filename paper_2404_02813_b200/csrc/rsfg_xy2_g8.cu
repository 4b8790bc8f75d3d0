// rsfg_xy2_g8.cu -- xy2 (rsfg_xy2.cuh) instantiations for radii [16, 17];
// one translation unit per radius group so the build parallelises.
#include "rsfg_xy2.cuh"

namespace rsfg {
#define RADII(X) X(16) X(17)
RSFG_XY2_GROUP(8, RADII)
}  // namespace rsfg
