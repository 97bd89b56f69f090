// conv_fwd.cu -- instantiates the implicit-GEMM conv kernel for CONV_FWD (conv.cuh) in its own
// translation unit.
#define B2N_CONV_INSTANTIATE
#include "conv.cuh"

namespace b2n {
template void launch_conv<CONV_FWD>(const ConvParams&, int, bool, int, cudaStream_t);
}  // namespace b2n
