// rsfg_zst4_g3.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [7];
// one translation unit per radius group so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {
#define RADII(X) X(7)
RSFG_ZST4_GROUP(3, RADII)
}  // namespace rsfg
