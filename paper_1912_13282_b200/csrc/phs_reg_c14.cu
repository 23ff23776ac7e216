// Shape-solve kernels instantiated for n=15, degree 2, d=2, 1 family (configs C1, C4): the register LU
// (FAST / REPLAY, phs_reg.cuh); the nullspace first pass of this shape is in phs_ns2_t*.cu.
#include "phs_reg.cuh"

namespace mf {
MF_INSTANTIATE_REG(15, 2, 2, 1)
}  // namespace mf
