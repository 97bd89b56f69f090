// Micro-probe: cost per iteration of a CTA barrier loop, alone and with an smem load/store chain
// (the shape of the device mt19937 wavefront, csrc/mt19937.cuh).  nvcc -arch=sm_100a -O3 barrier_probe.cu
#include <cstdio>
#include <cstdint>
__global__ void probe(int mode, int iters, long long* out, unsigned* sink) {
    __shared__ __align__(16) uint32_t ring[4096];
    const int t = threadIdx.x;
    for (int i = t; i < 4096; i += blockDim.x) ring[i] = i * 2654435761u;
    __syncthreads();
    uint32_t acc = t, reg = t;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (mode == 1) {  // 2 loads (prefetchable) + 1 store + register chain: plain MT recurrence shape
            const int q = (it * 227 + t) & 2047;
            const uint32_t a = ring[(q + 1424) & 2047], b = ring[(q + 1425) & 2047];
            reg = reg ^ ((((a & 0x80000000u) | (b & 0x7fffffffu)) >> 1) ^ ((b & 1u) ? 0x9908b0dfu : 0u));
            ring[q] = reg;
        } else if (mode == 2) {  // 8 x LDS.128 + 2 x STS.128 per thread (the 3-term, 4-word shape)
            const int A = ((it * 620 + 4 * t) & 2047);
            const uint4* r = reinterpret_cast<const uint4*>(ring + A + 2048 - 1080);
            uint4 x0 = r[0], x1 = r[1], x2 = r[57], x3 = r[58], x4 = r[99], x5 = r[100], x6 = r[114], x7 = r[115];
            uint4 v;
            v.x = x0.x ^ x1.y ^ x2.z ^ x3.w ^ x4.x ^ x5.y ^ x6.z ^ x7.w ^ reg;
            v.y = x0.y ^ x1.z ^ x2.w ^ x3.x ^ x4.y ^ x5.z ^ x6.w ^ x7.x;
            v.z = x0.z ^ x1.w ^ x2.x ^ x3.y ^ x4.z ^ x5.w ^ x6.x ^ x7.y;
            v.w = x0.w ^ x1.x ^ x2.y ^ x3.z ^ x4.w ^ x5.x ^ x6.y ^ x7.z;
            reg = v.x;
            *reinterpret_cast<uint4*>(ring + A) = v;
            *reinterpret_cast<uint4*>(ring + ((A + 2048) & 4095)) = v;
        }
        if (mode == 3) asm volatile("bar.sync 1, 256;" ::: "memory");
        else __syncthreads();
    }
    long long t1 = clock64();
    if (t == 0) out[0] = t1 - t0;
    sink[t] = acc ^ reg;
}
int main() {
    long long* d;
    unsigned* s;
    cudaMalloc(&d, 8);
    cudaMalloc(&s, 4096 * 4);
    const int iters = 2000;
    const int threads[] = {32, 160, 256, 640, 1024};
    for (int mode = 0; mode < 4; ++mode)
        for (int nt : threads) {
            if (mode == 3 && nt != 256) continue;
            if (mode == 2 && nt > 512) continue;
            probe<<<1, nt>>>(mode, 10, d, s);
            probe<<<1, nt>>>(mode, iters, d, s);
            long long h;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("mode %d threads %4d: %.1f clk / iteration\n", mode, nt, (double)h / iters);
        }
    return 0;
}
