// Register and tensor-core shape solves instantiated for n=25, degree 2, d=2, 3 families.
#include "phs_mma.cuh"

#include "phs_ns2.cuh"

namespace mf {
MF_INSTANTIATE_REG(25, 2, 2, 3)
MF_INSTANTIATE_MMA(25, 2, 2, 3)
MF_INSTANTIATE_NS(25, 2, 2, 3)
MF_INSTANTIATE_NS2(25, 2, 2, 3)
}  // namespace mf
