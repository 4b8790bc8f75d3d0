// rsfg_zst4_g5.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [9];
// one translation unit per radius group so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {
#define RADII(X) X(9)
RSFG_ZST4_GROUP(5, RADII)
}  // namespace rsfg
