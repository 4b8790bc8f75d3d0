// rsfg_zst4_g2.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [5, 6];
// one translation unit per radius group so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {
#define RADII(X) X(5) X(6)
RSFG_ZST4_GROUP(2, RADII)
}  // namespace rsfg
