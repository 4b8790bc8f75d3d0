// rsfg_xy2_g5.cu -- xy2 (rsfg_xy2.cuh) instantiations for radii [15];
// one translation unit per radius group so the build parallelises.
#include "rsfg_xy2.cuh"

namespace rsfg {
#define RADII(X) X(15)
RSFG_XY2_GROUP(5, RADII)
}  // namespace rsfg
