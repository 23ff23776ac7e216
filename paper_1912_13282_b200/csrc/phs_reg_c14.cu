// Register shape solve instantiated for n=15, degree 2, d=2, 1 family.
#include "phs_reg.cuh"

namespace mf {
MF_INSTANTIATE_REG(15, 2, 2, 1)
}  // namespace mf
