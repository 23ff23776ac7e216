// Shape-solve kernels instantiated for n=35, degree 2, d=3, 1 family (config C3).
#include "phs_split.cuh"

#include "phs_ns2.cuh"

namespace mf {
MF_INSTANTIATE_REG(35, 2, 3, 1)
MF_INSTANTIATE_MMA(35, 2, 3, 1)
MF_INSTANTIATE_SPLIT(35, 2, 3, 1)
MF_INSTANTIATE_NS(35, 2, 3, 1)
MF_INSTANTIATE_NS2(35, 2, 3, 1)
}  // namespace mf
