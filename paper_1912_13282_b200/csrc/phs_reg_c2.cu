// Shape-solve kernels instantiated for n=25, degree 2, d=2, 3 families (config C2): the register LU
// (FAST / REPLAY, phs_reg.cuh); the nullspace first pass of this shape is in phs_ns2_t*.cu.
#include "phs_reg.cuh"

namespace mf {
MF_INSTANTIATE_REG(25, 2, 2, 3)
}  // namespace mf
