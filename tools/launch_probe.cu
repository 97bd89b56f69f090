// launch_probe.cu -- event-timed single graph launches of an (almost) empty kernel vs launch config:
// cluster dims and dynamic shared memory (bring-up tool for the fused RBM step's launch overhead).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/launch_probe tools/launch_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_plain(int* p) { if (threadIdx.x == 0 && p) p[blockIdx.x] = 1; }
__global__ void __cluster_dims__(8, 1, 1) k_cluster(int* p) { if (threadIdx.x == 0 && p) p[blockIdx.x] = 1; }

template <class K>
float time_graph(K kernel, dim3 grid, int smem, cudaStream_t st, float* flush, size_t nflush) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    kernel<<<grid, 256, smem, st>>>(nullptr);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float tot = 0;
    const int n = 200;
    for (int i = 0; i < n + 10; ++i) {
        cudaMemsetAsync(flush, 0, nflush * 4, st);  // a different kernel before, like the bench's L2 flush
        cudaEventRecord(a, st);
        cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (i >= 10) tot += ms;
    }
    return tot / n * 1e3f;
}

int main() {
    cudaStream_t st;
    cudaStreamCreate(&st);
    float* flush;
    const size_t nf = 1 << 20;
    cudaMalloc(&flush, nf * 4);
    for (int smem : {0, 100 * 1024, 226 * 1024}) {
        printf("plain   64 CTAs smem %6d: %6.2f us\n", smem, time_graph(k_plain, dim3(64), smem, st, flush, nf));
        printf("cluster 64 CTAs smem %6d: %6.2f us\n", smem, time_graph(k_cluster, dim3(8, 8), smem, st, flush, nf));
    }
    return 0;
}
