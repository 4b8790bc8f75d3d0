// rsfg_xy2_g7.cu -- xy2 (rsfg_xy2.cuh) instantiations for radii [13, 14];
// one translation unit per radius group so the build parallelises.
#include "rsfg_xy2.cuh"

namespace rsfg {
#define RADII(X) X(13) X(14)
RSFG_XY2_GROUP(7, RADII)
}  // namespace rsfg
