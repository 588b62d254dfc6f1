// trsv_line_k2p.cu -- ldlt_line_kernel instances: 2 system(s) per cluster, PCG mode.
#include "trsv_line_impl.cuh"

namespace npcg {
cudaError_t launch_ldlt_k2p(const LineArgs &a, cudaStream_t s) { return launch_ldlt_inst<true, 2>(a, s); }
}  // namespace npcg
