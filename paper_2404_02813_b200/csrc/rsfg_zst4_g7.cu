// rsfg_zst4_g7.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [12, 15];
// one translation unit per radius group so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {
#define RADII(X) X(12) X(15)
RSFG_ZST4_GROUP(7, RADII)
}  // namespace rsfg
