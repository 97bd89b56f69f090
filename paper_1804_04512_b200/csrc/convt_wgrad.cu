// convt_wgrad.cu -- the FFMA weight-gradient kernel of the halo-tile conv path (convt.cuh).
#include "convt.cuh"

namespace b2n {

template <int KH, int KW, int NT>
static void launch_wg(const ConvTWLaunch& L, cudaStream_t st) {
    auto k = convt_wgrad_kernel<KH, KW, NT>;
    static bool attr = [&] {
        B2N_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        return true;
    }();
    (void)attr;
    launch_ex(k, dim3(L.grid), dim3(NT), (size_t)L.smem, st, 1u, L.map, L.zmaps[0], L.zmaps[1], L.zmaps[2],
              L.p);
}

void launch_convt_wgrad(const ConvTWLaunch& L, cudaStream_t st) {
    if (L.p.kh == 3 && L.p.kw == 3 && L.nt == 256)
        launch_wg<3, 3, 256>(L, st);
    else if (L.p.kh == 3 && L.p.kw == 3)
        launch_wg<3, 3, 512>(L, st);
    else if (L.p.kh == 5 && L.p.kw == 5)
        launch_wg<5, 5, 256>(L, st);
    else
        throw Error(B2N_EINTERNAL, "convt wgrad: filter size not instantiated");
}

}  // namespace b2n
