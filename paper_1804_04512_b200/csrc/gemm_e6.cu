// gemm_e6.cu -- instantiates the tcgen05 GEMM for the EPI_RBM_VIS epilogue (all tile widths, both
// precisions) in its own translation unit; see runtime.cuh gemm_launch_epi.
#define B2N_GEMM_INSTANTIATE
#include "runtime.cuh"

namespace b2n {
template void gemm_launch_epi<EPI_RBM_VIS>(const GemmLaunch&, cudaStream_t);
}  // namespace b2n
