// Shape-solve kernels instantiated for n=35, degree 2, d=3, 1 family (config C3): the register LU
// (FAST / REPLAY, phs_reg.cuh); the nullspace first pass of this shape is in phs_ns2_t*.cu.
#include "phs_reg.cuh"

namespace mf {
MF_INSTANTIATE_REG(35, 2, 3, 1)
}  // namespace mf
