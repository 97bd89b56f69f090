// conv.cuh -- implicit-GEMM convolution on tcgen05 (forward + act + 2x2 max-pool + argmax,
// backward-data, backward-weights). Interface used by network.cuh.
#pragma once
#include "runtime.cuh"

namespace b2n {

struct ConvGeom {
    int c = 1, h = 1, w = 1, k = 1, kh = 1, kw = 1, pad = 0, oh = 1, ow = 1;
};

struct ConvFwdLaunch {
    double flops = 0, bytes = 0;
    void run(cudaStream_t) const { throw Error(B2N_ESPEC, "b200nn: conv path not built yet"); }
};
struct ConvBwdLaunch {
    double flops = 0, bytes = 0;
    void run(cudaStream_t, bool) const { throw Error(B2N_ESPEC, "b200nn: conv path not built yet"); }
    int kernels() const { return 0; }
};

inline ConvFwdLaunch plan_conv_fwd(const ConvGeom&, int, const float*, long long, const float*, const float*, int, bool,
                                   float*, long long, uint8_t*, bool) {
    throw Error(B2N_ESPEC, "b200nn: conv path not built yet");
}
inline ConvBwdLaunch plan_conv_bwd(const ConvGeom&, int, const float*, long long, const float*, const float*, int, bool,
                                   const float*, long long, const uint8_t*, const float*, long long, float*, long long,
                                   float*, float*, float*, float*, float*, float*, float, float, float, bool) {
    throw Error(B2N_ESPEC, "b200nn: conv path not built yet");
}

}  // namespace b2n
