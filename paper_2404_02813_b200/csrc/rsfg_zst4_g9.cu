// rsfg_zst4_g9.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [13, 14];
// one translation unit per radius group so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {
#define RADII(X) X(13) X(14)
RSFG_ZST4_GROUP(9, RADII)
}  // namespace rsfg
