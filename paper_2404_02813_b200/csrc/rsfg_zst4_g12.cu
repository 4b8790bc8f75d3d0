// rsfg_zst4_g12.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [21, 22];
// one translation unit per radius group so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {
#define RADII(X) X(21) X(22)
RSFG_ZST4_GROUP(12, RADII)
}  // namespace rsfg
