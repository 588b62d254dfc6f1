// trsv_line_k1n.cu -- ldlt_line_kernel instances: 1 system(s) per cluster, plain mode.
#include "trsv_line_impl.cuh"

namespace npcg {
cudaError_t launch_ldlt_k1n(const LineArgs &a, cudaStream_t s) { return launch_ldlt_inst<false, 1>(a, s); }
}  // namespace npcg
