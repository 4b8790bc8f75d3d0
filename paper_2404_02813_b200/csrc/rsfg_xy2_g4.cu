// rsfg_xy2_g4.cu -- xy2 (rsfg_xy2.cuh) instantiations for radii [12];
// one translation unit per radius group so the build parallelises.
#include "rsfg_xy2.cuh"

namespace rsfg {
#define RADII(X) X(12)
RSFG_XY2_GROUP(4, RADII)
}  // namespace rsfg
