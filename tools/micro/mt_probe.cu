// Micro-probe of the device mt19937 wavefront (csrc/mt19937.cuh mt_words_kernel): cycles per 620-word
// chunk with the global store of the words (MODE 0), without it (1), and with the barrier only (2).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t tw(uint32_t a, uint32_t b) {
    return (((a & 0x80000000u) | (b & 0x7fffffffu)) >> 1) ^ ((b & 1u) ? 0x9908b0dfu : 0u);
}
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(uint32_t* wbuf, int chunks, long long* cyc) {
    __shared__ __align__(16) uint32_t ring[4096];
    constexpr int M = 2047;
    const int t = threadIdx.x;
    for (int i = t; i < 4096; i += 256) ring[i] = i * 2654435761u;
    __syncthreads();
    long long t0 = clock64();
    if (t < 160) {
        uint4* wb = reinterpret_cast<uint4*>(wbuf);
        int A = (1080 + 4 * t) & M;
        uint32_t own0 = ring[(460 + 4 * t) & M];
        for (int c = 0; c < chunks; ++c) {
            const long long q = 1080 + 620LL * c + 4 * t;
            if (t < 155) {
                if (MODE < 2) {
                    const uint32_t* r = ring + A + 2048;
                    const uint4 a0 = *reinterpret_cast<const uint4*>(r - 624);
                    const uint32_t b0 = r[-851];
                    const uint2 b1 = *reinterpret_cast<const uint2*>(r - 850);
                    const uint2 b2 = *reinterpret_cast<const uint2*>(r - 848);
                    const uint2 d0 = *reinterpret_cast<const uint2*>(r - 1078);
                    const uint2 d1 = *reinterpret_cast<const uint2*>(r - 1076);
                    const uint32_t d2 = r[-1074];
                    const uint32_t e0 = r[-681];
                    const uint2 e1 = *reinterpret_cast<const uint2*>(r - 680);
                    const uint32_t e2 = r[-678];
                    const uint32_t c0 = a0.x ^ b0 ^ d0.x, c1 = a0.y ^ b1.x ^ d0.y, c2 = a0.z ^ b1.y ^ d1.x,
                                   c3 = a0.w ^ b2.x ^ d1.y, c4 = own0 ^ b2.y ^ d2;
                    uint4 v;
                    v.x = e0 ^ tw(c0, c1);
                    v.y = e1.x ^ tw(c1, c2);
                    v.z = e1.y ^ tw(c2, c3);
                    v.w = e2 ^ tw(c3, c4);
                    own0 = v.x;
                    *reinterpret_cast<uint4*>(ring + A) = v;
                    *reinterpret_cast<uint4*>(ring + A + 2048) = v;
                    if (MODE == 0) wb[q >> 2] = v;
                }
            }
            A = (A + 620) & M;
            asm volatile("bar.sync 1, 160;" ::: "memory");
        }
    }
    __syncthreads();
    if (t == 0) cyc[0] = clock64() - t0;
}
int main() {
    uint32_t* w;
    long long* c;
    cudaMalloc(&w, 200 * 620 * 4 + 4096 * 4);
    cudaMalloc(&c, 8);
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) k<0><<<1, 256>>>(w, 161, c);
            if (mode == 1) k<1><<<1, 256>>>(w, 161, c);
            if (mode == 2) k<2><<<1, 256>>>(w, 161, c);
        }
        long long h;
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("mode %d: %.1f clk / chunk\n", mode, h / 161.0);
    }
    return 0;
}
