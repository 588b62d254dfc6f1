// trsv_line_k2n.cu -- ldlt_line_kernel instances: 2 system(s) per cluster, plain mode.
#include "trsv_line_impl.cuh"

namespace npcg {
cudaError_t launch_ldlt_k2n(const LineArgs &a, cudaStream_t s) { return launch_ldlt_inst<false, 2>(a, s); }
}  // namespace npcg
