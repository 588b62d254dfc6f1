// trsv_line_k1p.cu -- ldlt_line_kernel instances: 1 system(s) per cluster, PCG mode.
#include "trsv_line_impl.cuh"

namespace npcg {
cudaError_t launch_ldlt_k1p(const LineArgs &a, cudaStream_t s) { return launch_ldlt_inst<true, 1>(a, s); }
}  // namespace npcg
