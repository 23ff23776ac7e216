// Register-resident fast path of the PHS shape solve (filled in below).
#include "common.cuh"
#include "phs_params.cuh"

namespace mf {
// Not specialised for any shape yet: the generic kernel handles everything.
int launch_phs_fast(const PhsArgs&, cudaStream_t, int) { return MF_ERR_UNSUPPORTED; }
}  // namespace mf
