// rsfg_zst4_g1.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [3, 4];
// one translation unit per radius group so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {
#define RADII(X) X(3) X(4)
RSFG_ZST4_GROUP(1, RADII)
}  // namespace rsfg
