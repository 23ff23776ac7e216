// Shape-solve kernels instantiated for n=15, degree 2, d=2, 1 family (configs C1, C4): the register LU
// (FAST / REPLAY, phs_reg.cuh) and the nullspace HYBRID first pass (phs_ns2.cuh).
#include "phs_ns2.cuh"

namespace mf {
MF_INSTANTIATE_REG(15, 2, 2, 1)
MF_INSTANTIATE_NS2(15, 2, 2, 1)
}  // namespace mf
