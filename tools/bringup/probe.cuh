// probe.cuh -- single-CTA bring-up probe for the TMA -> SWIZZLE_128B smem -> tcgen05.mma -> TMEM
// chain (test infrastructure for the tensor-core path; exported as b2n_debug_probe).
#pragma once
#include "runtime.cuh"

namespace b2n {

// A: 128 x 32 tile (K-major, or MN-major when a_mn), B: 32 x 32 tile; dumps smem and D.
__global__ void __launch_bounds__(192, 1)
    probe_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int a_mn, int b_mn,
                 float* smem_out, float* d_out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* a = smem;
    uint8_t* b = smem + 16384;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 4096);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(slot, 32);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *slot;
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar[0], 16384 + 4096);
        if (!a_mn) tma_load_2d(a, &mapA, &bar[0], 0, 0);
        else for (int j = 0; j < 4; ++j) tma_load_2d(a + j * 4096, &mapA, &bar[0], 32 * j, 0);
        tma_load_2d(b, &mapB, &bar[0], 0, 0);
    }
    mbar_wait(&bar[0], 0);
    for (int i = threadIdx.x; i < (16384 + 4096) / 4; i += blockDim.x) smem_out[i] = reinterpret_cast<float*>(smem)[i];
    __syncthreads();
    if (warp == 1 && lane == 0) {
        tc_fence_after();
        const uint32_t idesc = umma_idesc_tf32(128, 32, a_mn, b_mn);
        for (int kk = 0; kk < 4; ++kk) {
            mma_tf32(tbase, a_mn ? desc_mnmajor(smem_u32(a), kk) : desc_kmajor(smem_u32(a), kk),
                     b_mn ? desc_mnmajor(smem_u32(b), kk) : desc_kmajor(smem_u32(b), kk), idesc, kk > 0);
        }
        mma_commit(&bar[1]);
    }
    if (warp >= 2) {
        mbar_wait(&bar[1], 0);
        tc_fence_after();
        const int q = warp & 3;
        float v[16];
        for (int c = 0; c < 32; c += 16) {
            tmem_ld16(tbase + ((uint32_t)(32 * q) << 16) + c, v);
            for (int i = 0; i < 16; ++i) d_out[(32 * q + lane) * 32 + c + i] = v[i];
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, 32);
    }
}

}  // namespace b2n
