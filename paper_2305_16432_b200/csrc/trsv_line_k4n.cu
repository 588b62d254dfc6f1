// trsv_line_k4n.cu -- ldlt_line_kernel instances: 4 system(s) per cluster, plain mode.
#include "trsv_line_impl.cuh"

namespace npcg {
cudaError_t launch_ldlt_k4n(const LineArgs &a, cudaStream_t s) { return launch_ldlt_inst<false, 4>(a, s); }
}  // namespace npcg
