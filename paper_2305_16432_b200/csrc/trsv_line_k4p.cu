// trsv_line_k4p.cu -- ldlt_line_kernel instances: 4 system(s) per cluster, PCG mode.
#include "trsv_line_impl.cuh"

namespace npcg {
cudaError_t launch_ldlt_k4p(const LineArgs &a, cudaStream_t s) { return launch_ldlt_inst<true, 4>(a, s); }
}  // namespace npcg
