// rsfg_zst4_g13.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [23, 24];
// one translation unit per radius group so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {
#define RADII(X) X(23) X(24)
RSFG_ZST4_GROUP(13, RADII)
}  // namespace rsfg
