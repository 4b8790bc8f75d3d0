// rsfg_zst4_g11.cu -- zst4 (rsfg_zst4.cuh) instantiations for radii [19, 20];
// one translation unit per radius group so the build parallelises.
#include "rsfg_zst4.cuh"

namespace rsfg {
#define RADII(X) X(19) X(20)
RSFG_ZST4_GROUP(11, RADII)
}  // namespace rsfg
