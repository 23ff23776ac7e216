// Register and tensor-core shape solves instantiated for n=15, degree 2, d=2, 1 family.
#include "phs_mma.cuh"

#include "phs_ns2.cuh"

namespace mf {
MF_INSTANTIATE_REG(15, 2, 2, 1)
MF_INSTANTIATE_MMA(15, 2, 2, 1)
MF_INSTANTIATE_NS(15, 2, 2, 1)
MF_INSTANTIATE_NS2(15, 2, 2, 1)
}  // namespace mf
