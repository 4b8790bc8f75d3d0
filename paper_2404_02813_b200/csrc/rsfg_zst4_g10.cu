// rsfg_zst4_g10.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [16, 17];
// one translation unit per radius group so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {
#define RADII(X) X(16) X(17)
RSFG_ZST4_GROUP(10, RADII)
}  // namespace rsfg
