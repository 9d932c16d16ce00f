// ffn_gemm_tc.cu — prefill path: tcgen05 grouped GEMM (placeholder until the
// kernel lands; gemm_available() reports false and AUTO routes to the GEMV).
#include "kernels.cuh"

namespace moqe_gpu {
bool gemm_available() { return false; }
int gemm_block_n() { return 128; }
cudaError_t launch_gemm(int, int, const GemmArgs&, const Plan&, cudaStream_t, int) { return cudaErrorNotSupported; }
}  // namespace moqe_gpu
