// Register shape solve instantiated for n=25, degree 2, d=2, 3 families.
#include "phs_reg.cuh"

namespace mf {
MF_INSTANTIATE_REG(25, 2, 2, 3)
}  // namespace mf
