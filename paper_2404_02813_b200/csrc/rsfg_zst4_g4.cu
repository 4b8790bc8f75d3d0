// rsfg_zst4_g4.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [8];
// one translation unit per radius group so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {
#define RADII(X) X(8)
RSFG_ZST4_GROUP(4, RADII)
}  // namespace rsfg
