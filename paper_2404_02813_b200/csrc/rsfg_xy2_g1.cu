// rsfg_xy2_g1.cu -- xy2 (rsfg_xy2.cuh) instantiations for radii [5, 6, 7, 8];
// one translation unit per radius group so the build parallelises.
#include "rsfg_xy2.cuh"

namespace rsfg {
#define RADII(X) X(5) X(6) X(7) X(8)
RSFG_XY2_GROUP(1, RADII)
}  // namespace rsfg
