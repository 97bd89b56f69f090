// convt_fwd.cu -- instantiates the halo-tile tensor-core conv kernel (convt.cuh) for the forward pass.
#define B2N_CONVT_INSTANTIATE
#include "convt.cuh"

namespace b2n {
template void launch_convt<CT_FWD>(const ConvTLaunch&, cudaStream_t);
}  // namespace b2n
