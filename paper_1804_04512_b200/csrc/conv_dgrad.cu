// conv_dgrad.cu -- instantiates the implicit-GEMM conv kernel for CONV_DGRAD (conv.cuh) in its own
// translation unit.
#define B2N_CONV_INSTANTIATE
#include "conv.cuh"

namespace b2n {
template void launch_conv<CONV_DGRAD>(const ConvParams&, int, bool, int, cudaStream_t);
}  // namespace b2n
