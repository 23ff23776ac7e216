// Register shape solve instantiated for n=35, degree 2, d=3, 1 family.
#include "phs_reg.cuh"

namespace mf {
MF_INSTANTIATE_REG(35, 2, 3, 1)
}  // namespace mf
