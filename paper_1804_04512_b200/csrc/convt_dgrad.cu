// convt_dgrad.cu -- instantiates the halo-tile tensor-core conv kernel (convt.cuh) for backward-data.
#define B2N_CONVT_INSTANTIATE
#include "convt.cuh"

namespace b2n {
template void launch_convt<CT_DGRAD>(const ConvTLaunch&, cudaStream_t);
}  // namespace b2n
