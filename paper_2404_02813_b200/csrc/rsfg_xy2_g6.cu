// rsfg_xy2_g6.cu -- xy2 (rsfg_xy2.cuh) instantiations for radii [18];
// one translation unit per radius group so the build parallelises.
#include "rsfg_xy2.cuh"

namespace rsfg {
#define RADII(X) X(18)
RSFG_XY2_GROUP(6, RADII)
}  // namespace rsfg
