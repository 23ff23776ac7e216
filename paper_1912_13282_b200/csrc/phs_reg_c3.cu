// Register and tensor-core shape solves instantiated for n=35, degree 2, d=3, 1 family.
#include "phs_mma.cuh"

namespace mf {
MF_INSTANTIATE_REG(35, 2, 3, 1)
MF_INSTANTIATE_MMA(35, 2, 3, 1)
}  // namespace mf
