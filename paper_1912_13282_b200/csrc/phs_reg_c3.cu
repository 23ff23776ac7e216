// Shape-solve kernels instantiated for n=35, degree 2, d=3, 1 family (config C3): the register LU
// (FAST / REPLAY, phs_reg.cuh) and the nullspace HYBRID first pass (phs_ns2.cuh).
#include "phs_ns2.cuh"

namespace mf {
MF_INSTANTIATE_REG(35, 2, 3, 1)
MF_INSTANTIATE_NS2(35, 2, 3, 1)
}  // namespace mf
