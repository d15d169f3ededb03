// tcgen05 tensor-core complex GEMM (placeholder until the sm_100a kernel lands).
#include "kernels.cuh"

namespace rcsg {
bool gemm_tc_supported(const GemmArgs&) { return false; }
void launch_gemm_tc(const GemmArgs&, int, cudaStream_t) {}
}  // namespace rcsg
