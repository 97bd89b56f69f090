// mma_probe.cu -- tcgen05.mma throughput vs operand layout / N / kind on one B200 SM (bring-up tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_probe tools/mma_probe.cu
// Every CTA issues `iters` back-to-back MMAs (single thread) into one TMEM accumulator and reports
// clk per MMA; 148 CTAs run concurrently (one per SM).
#include <cstdio>
#include <cstdint>
#include "../paper_1804_04512_b200/csrc/ptx.cuh"
using namespace b2n;

__device__ __forceinline__ void mma_tf32_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
                 "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n}" ::"r"(d), "l"(a), "l"(b), "r"(idesc) : "memory");
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

struct Cfg { int kind, N, layout, lbo, sbo, a_step, iters, nacc; };

__global__ void probe(Cfg c, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<float*>(s)[i] = c.a_step < 0 ? 0.0f : 0.001f * (float)((i * 2654435761u) >> 20) - 1.0f;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (threadIdx.x < 32) tmem_alloc(&tslot, 256);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (c.nacc == 4 && threadIdx.x < 32) {  // conv-kernel pattern: descriptors from an smem table + row adds
        __shared__ uint64_t tab[16];
        const uint32_t a0 = smem_u32(s), b0 = a0 + 96 * 1024;
        if (threadIdx.x < 8) {
            tab[2 * threadIdx.x] = umma_desc(a0 + threadIdx.x * c.a_step, c.lbo, c.sbo, c.layout);
            tab[2 * threadIdx.x + 1] = umma_desc(b0 + threadIdx.x * 1536, 48 * 16, 128, c.layout);
        }
        __syncwarp();
        const uint32_t idesc = umma_idesc_tf32(128, c.N, 0, 0);
        const unsigned long long t0 = clock64();
        uint64_t add = 0;
        for (int i = 0; i < c.iters; i += 24, add = (add + 130) & 1023) {
            for (int h = 0; h < 4; ++h) {
                for (int ks = 0; ks < 2; ++ks) {
                    const uint64_t da = tab[2 * ks] + add + h * 8, db = tab[2 * ks + 1];
                    mma_tf32_elect(tmem + (3 - h) * 16, da + 520, db, idesc);
                    mma_tf32_elect(tmem + (3 - h) * 16, da, db + 96, idesc);
                    mma_tf32_elect(tmem + (3 - h) * 16, da, db, idesc);
                }
            }
        }
        if (threadIdx.x == 0) mma_commit(&bar);
        mbar_wait(&bar, 0);
        if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    } else if (c.nacc == 3 && threadIdx.x < 32) {  // warp-converged issue, elect.sync per MMA
        const uint32_t a0 = smem_u32(s), b0 = a0 + 96 * 1024;
        const uint32_t idesc = umma_idesc_tf32(128, c.N, 0, 0);
        const uint64_t da = umma_desc(a0, c.lbo, c.sbo, c.layout), db = umma_desc(b0, c.lbo, c.sbo, c.layout);
        __syncwarp();
        const unsigned long long t0 = clock64();
        for (int i = 0; i < c.iters; i += 4) {
            mma_tf32_elect(tmem, da + (uint64_t)(i & 7), db, idesc);
            mma_tf32_elect(tmem, da + 2, db, idesc);
            mma_tf32_elect(tmem, da + (uint64_t)((i + 2) & 7), db, idesc);
            mma_tf32_elect(tmem, da + 6, db, idesc);
        }
        if (threadIdx.x == 0) mma_commit(&bar);
        mbar_wait(&bar, 0);
        if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    } else if (c.nacc < 3 && threadIdx.x == 0) {
        const uint32_t a0 = smem_u32(s), b0 = a0 + 96 * 1024;
        uint32_t idesc;
        if (c.kind == 0) idesc = umma_idesc_tf32(128, c.N, 0, 0);
        else idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(c.N >> 3) << 17) | ((128u >> 4) << 24);
        const uint64_t da = umma_desc(a0, c.lbo, c.sbo, c.layout);
        const uint64_t db = umma_desc(b0, c.lbo, c.sbo, c.layout);
        const unsigned long long t0 = clock64();
        if (c.nacc == 1) {  // loop-invariant operands: the body is the MMA issue alone
            if (c.kind == 0)
                for (int i = 0; i < c.iters; i += 4) {
                    mma_tf32(tmem, da, db, idesc, 1); mma_tf32(tmem, da, db, idesc, 1);
                    mma_tf32(tmem, da, db, idesc, 1); mma_tf32(tmem, da, db, idesc, 1);
                }
            else
                for (int i = 0; i < c.iters; i += 4) {
                    mma_f16(tmem, da, db, idesc, 1); mma_f16(tmem, da, db, idesc, 1);
                    mma_f16(tmem, da, db, idesc, 1); mma_f16(tmem, da, db, idesc, 1);
                }
        } else {  // a descriptor add per MMA (the conv kernels' pattern)
            for (int i = 0; i < c.iters; i += 4) {
                if (c.kind == 0) {
                    mma_tf32(tmem, da + (uint64_t)(i & 7), db, idesc, 1); mma_tf32(tmem, da + 2, db, idesc, 1);
                    mma_tf32(tmem, da + (uint64_t)((i + 2) & 7), db, idesc, 1); mma_tf32(tmem, da + 6, db, idesc, 1);
                } else {
                    mma_f16(tmem, da + (uint64_t)(i & 7), db, idesc, 1); mma_f16(tmem, da + 2, db, idesc, 1);
                    mma_f16(tmem, da + (uint64_t)((i + 2) & 7), db, idesc, 1); mma_f16(tmem, da + 6, db, idesc, 1);
                }
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        const unsigned long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tmem, 256); }
}

int main() {
    unsigned long long* d; cudaMalloc(&d, 148 * 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    // layout codes: 0 = none (interleave), 2 = SW128, 4 = SW64, 6 = SW32
    const char* lname[8] = {"NONE", "SW128B32", "SW128", "?", "SW64", "?", "SW32", "?"};
    struct { int layout, lbo, sbo, a_step; } L[] = {{0, 2080, 128, 16}, {0, 128, 256, 0}, {2, 16, 1024, 32}, {6, 16, 256, 32}, {4, 16, 512, 32}};
    struct { int layout, lbo, sbo, a_step; } P2[] = {{0, 16, 128, 32}, {0, 2080, 128, 16}, {0, 128, 256, 16}};
    for (auto& l : P2)
        for (int N : {16, 48, 96})
            for (int var : {3, 4}) {
                Cfg c{0, N, l.layout, l.lbo, l.sbo, l.a_step, 24 * 96, var};
                probe<<<148, 128, 200 * 1024>>>(c, d);
                unsigned long long h[148];
                cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
                double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
                printf("tf32 NONE lbo=%5d sbo=%4d N=%3d variant=%d : %6.1f clk/MMA (floor %d)\n", l.lbo, l.sbo, N, var,
                       avg / c.iters, N / 2);
            }
    return 0;
}
