// rsfg_zst4_g6.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [10, 11];
// one translation unit per radius group so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {
#define RADII(X) X(10) X(11)
RSFG_ZST4_GROUP(6, RADII)
}  // namespace rsfg
