// rsfg_xy2_g9.cu -- xy2 (rsfg_xy2.cuh) instantiations for radii [19, 20];
// one translation unit per radius group so the build parallelises.
#include "rsfg_xy2.cuh"

namespace rsfg {
#define RADII(X) X(19) X(20)
RSFG_XY2_GROUP(9, RADII)
}  // namespace rsfg
