// rsfg_zst4_g8.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [18];
// one translation unit per radius group so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {
#define RADII(X) X(18)
RSFG_ZST4_GROUP(8, RADII)
}  // namespace rsfg
