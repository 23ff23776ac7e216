// Shape-solve kernels instantiated for n=25, degree 2, d=2, 3 families (config C2): the register LU
// (FAST / REPLAY, phs_reg.cuh) and the nullspace HYBRID first pass (phs_ns2.cuh).
#include "phs_ns2.cuh"

namespace mf {
MF_INSTANTIATE_REG(25, 2, 2, 3)
MF_INSTANTIATE_NS2(25, 2, 2, 3)
}  // namespace mf
