// rsfg_zst4_g0.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [0, 1, 2];
// one translation unit per radius group so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {
#define RADII(X) X(0) X(1) X(2)
RSFG_ZST4_GROUP(0, RADII)
}  // namespace rsfg
