// convt.cuh -- halo-tile convolution kernels (conv_forward / conv_backward + pool, layers.hpp:132-271,
// conv.hpp:180-345) for the B200: the full-resolution conv output and the im2col matrix never exist.
//
// Activations between conv layers use a row-blocked layout, [b][y][c/4][x][4] ("channel quads per
// image row"), so that ONE TMA box {4 ch, P cols, G quads, HR rows} lands an input halo tile in
// shared memory as [row][quad][col][4]: 16-byte pixel rows, exactly the K-major no-swizzle UMMA
// core-matrix layout (8 pixel rows x 16 B). Every filter tap (di, dj) is then just a different
// descriptor start address into the same halo (start + (row*G + quad)*P*16 + dj*16), so the 9 (25)
// taps of a 3x3 (5x5) filter cost no data movement at all:
//
//   convt_mma_kernel<FWD>   : TMA halo -> [lo split] -> tcgen05.mma per (output row, tap, quad pair)
//                              -> TMEM -> bias + act + 2x2 max + first-index argmax -> pooled output
//                              (row-blocked, or NCHW for the layer feeding a dense layer) + code bytes
//   convt_mma_kernel<DGRAD> : the same kernel over dZ = unpool(dP) * act'(P), expanded by producer
//                              warps straight into the halo (never stored), flipped / transposed
//                              weights, pad' = kh - 1 - pad  -> dX (the previous layer's dP)
//   convt_wgrad_kernel      : FFMA direct correlation X halo (TMA) x dZ tile (expanded) into
//                              per-thread register accumulators, fixed-order CTA reduction -> partials
//   convt_wgrad_reduce_kernel: fixed-order sum of the per-CTA partials + sgd_momentum_step
//   convt_repack_kernel     : NCHW network input -> row-blocked (channels padded to 4 with zeros)
// Padding (conv pad, tile edges) is TMA out-of-bounds zero fill; every reduction order is fixed.
#pragma once
#include "conv.cuh"

namespace b2n {

// one activation tensor of the conv stack: row-blocked [b][y][c/4][x][4] or NCHW (network layout)
struct TLayout {
    float* p = nullptr;
    long long bstride = 0;  // floats between images
    int blocked = 1;
    int C = 1, H = 1, W = 1;  // real channels (blocked storage pads to a multiple of 4)
};
__device__ __forceinline__ long long tl_quad(const TLayout& t, int b, int q, int y, int x) {  // blocked
    return (long long)b * t.bstride + (((long long)y * ((t.C + 3) >> 2) + q) * t.W + x) * 4;
}
// 4 consecutive channels [4q, 4q+4) of pixel (y, x); zeros past C
__device__ __forceinline__ float4 tl_load4(const TLayout& t, int b, int q, int y, int x) {
    if (t.blocked) return __ldg(reinterpret_cast<const float4*>(t.p + tl_quad(t, b, q, y, x)));
    float v[4];
    const long long plane = (long long)t.H * t.W;
    const float* base = t.p + (long long)b * t.bstride + (long long)y * t.W + x;
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = 4 * q + j < t.C ? __ldg(base + (4 * q + j) * plane) : 0.0f;
    return make_float4(v[0], v[1], v[2], v[3]);
}

// Source of a layer's dZ = unpool(dP) * act'(P) (pool_backward, layers.hpp:240-271, +
// activation_gradient, layers.hpp:284-298). The pooled-resolution inputs of a tile (dP, P and the
// argmax codes for a window of pooled rows x cols, all channel quads) are staged in shared memory --
// by TMA when dP / P are row-blocked, by thread loads when they are NCHW (the layer feeding a dense
// layer) -- and dZ is expanded from there, never written to HBM.
// The innermost TMA coordinate must be 16-byte aligned, so staging windows start at a pooled column
// that is a multiple of 4 (and are 3 columns wider).
struct DZSrc {
    TLayout dP, P;          // gradient / value of the layer's pooled (or plain) output
    const uint8_t* codes;   // argmax codes, row-blocked bytes [b][py][Kq][PWc][4]
    long long codes_bstride;
    int PWc;                // code rows are padded to a multiple of 4 pooled columns (TMA strides)
    int act, pool;
    int OHz, OWz;           // the layer's conv-output extents (= dZ extents)
    int tma;                // dP / P row-blocked: stage by TMA
    int bh, bw, Kq;         // staging window: pooled rows, cols (multiple of 4), channel quads
};
// staging slot layout: float4 dP | float4 P | uint32 codes, each part 128-byte aligned (TMA destinations)
__host__ __device__ __forceinline__ int zs_off_p(const DZSrc& z) { return (z.bh * z.Kq * z.bw * 16 + 127) & ~127; }
__host__ __device__ __forceinline__ int zs_bytes(const DZSrc& z) {
    return 2 * zs_off_p(z) + ((z.bh * z.Kq * z.bw * 4 + 127) & ~127);
}
__host__ __device__ __forceinline__ uint32_t zs_tx_bytes(const DZSrc& z) {
    return (uint32_t)(z.bh * z.Kq * z.bw * (z.pool ? 36 : 32));
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3, int c4);

// staging slot: float4 dP[bh][Kq][bw] | float4 P[bh][Kq][bw] | uint32 codes[bh][Kq][bw]
__device__ __forceinline__ void zs_issue(const DZSrc& z, const CUtensorMap* mdp, const CUtensorMap* mp,
                                         const CUtensorMap* mc, uint8_t* slot, uint64_t* bar, int b, int sy0, int sx0) {
    const int n = z.bh * z.Kq * z.bw;  // the caller has armed `bar` with zs_tx_bytes(z)
    (void)n;
    tma_load_5d(slot, mdp, bar, 0, sx0, 0, sy0, b);
    tma_load_5d(slot + zs_off_p(z), mp, bar, 0, sx0, 0, sy0, b);
    if (z.pool) tma_load_4d(slot + 2 * zs_off_p(z), mc, bar, sx0, 0, sy0, b);
}
__device__ __forceinline__ void zs_load_sync(const DZSrc& z, uint8_t* slot, int b, int sy0, int sx0, int tid, int nt) {
    const int n = z.bh * z.Kq * z.bw;
    float4* dps = reinterpret_cast<float4*>(slot);
    float4* ps = reinterpret_cast<float4*>(slot + zs_off_p(z));
    uint32_t* cs = reinterpret_cast<uint32_t*>(slot + 2 * zs_off_p(z));
    const int PH = z.dP.H, PW = z.dP.W;
    for (int i = tid; i < n; i += nt) {
        const int sr = i / (z.Kq * z.bw), rem = i - sr * (z.Kq * z.bw), q = rem / z.bw, sc = rem - q * z.bw;
        const int py = sy0 + sr, px = sx0 + sc;
        float4 g = make_float4(0.f, 0.f, 0.f, 0.f), v = g;
        uint32_t cw = 0;
        if ((unsigned)py < (unsigned)PH && (unsigned)px < (unsigned)PW) {
            g = tl_load4(z.dP, b, q, py, px);
            v = tl_load4(z.P, b, q, py, px);
            if (z.pool)
                cw = __ldg(reinterpret_cast<const uint32_t*>(z.codes + (long long)b * z.codes_bstride +
                                                             (((long long)py * z.Kq + q) * z.PWc + px) * 4));
        }
        dps[i] = g;
        ps[i] = v;
        cs[i] = cw;
    }
}
// dZ quad q at conv-output pixel (Y, X) from a staging slot anchored at pooled (sy0, sx0); zero
// outside the map (the dgrad's implicit padding)
__device__ __forceinline__ float4 zs_dz(const DZSrc& z, const uint8_t* slot, int sy0, int sx0, int q, int Y, int X) {
    if ((unsigned)Y >= (unsigned)z.OHz || (unsigned)X >= (unsigned)z.OWz) return make_float4(0.f, 0.f, 0.f, 0.f);
    const int sr = (z.pool ? Y >> 1 : Y) - sy0, sc = (z.pool ? X >> 1 : X) - sx0;
    const int idx = (sr * z.Kq + q) * z.bw + sc;
    const float4 g = reinterpret_cast<const float4*>(slot)[idx];
    const float4 y = reinterpret_cast<const float4*>(slot + zs_off_p(z))[idx];
    float d[4] = {act_grad(z.act, g.x, y.x), act_grad(z.act, g.y, y.y), act_grad(z.act, g.z, y.z),
                  act_grad(z.act, g.w, y.w)};
    if (z.pool) {
        const uint32_t cw = reinterpret_cast<const uint32_t*>(slot + 2 * zs_off_p(z))[idx];
        const uint32_t want = (uint32_t)((Y & 1) * 2 + (X & 1));
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (((cw >> (8 * j)) & 0xFFu) != want) d[j] = 0.0f;
    }
    return make_float4(d[0], d[1], d[2], d[3]);
}

enum ConvTMode : int { CT_FWD = 0, CT_DGRAD = 1 };

struct ConvTParams {
    // the correlation this launch computes: input Hin x Win, Cp = 4*G channels, kh x kw, pad
    int B, Cp, G, Hin, Win, kh, kw, pad, OH, OW;
    int N;             // real output channels
    int R, Wt, P, HR;  // output rows / cols per tile, halo cols / rows
    int tiles_x, tiles_y, ntiles;
    int ksteps, stages;
    int halo_bytes, stage_bytes, w_bytes;  // smem carve-up (host-computed)
    // epilogue
    int act, pool;
    const float* bias;  // FWD
    TLayout out;        // FWD: pooled (or full) output; DGRAD: dX (row-blocked)
    uint8_t* codes;     // FWD + pool: argmax codes, row-blocked bytes [b][py][k/4][PWc][4]
    long long codes_bstride;
    int codes_pw;       // PWc: pooled columns per code row, padded to a multiple of 4
    // weights W[k][c][kh][kw] of the LAYER (k = wk_K real kernels, c = wk_C real channels)
    const float* wk;
    int wk_K, wk_C;
    // DGRAD producer: dZ of the layer, staged + expanded on the fly (two staging slots)
    DZSrc z;
    int zslot_bytes;
};

// K step s (8 tf32 = two 16-byte chunks kc) -> correlation input channel / tap of element j of chunk kc
__device__ __forceinline__ bool ct_kdecode(const ConvTParams& p, int s, int kc, int j, int& cin, int& di, int& dj) {
    if (p.G >= 2) {
        const int GP = (p.G + 1) >> 1, tap = s / GP, gp = s - tap * GP;
        di = tap / p.kw;
        dj = tap - di * p.kw;
        const int q = 2 * gp + kc;
        cin = 4 * q + j;
        return q < p.G;
    }
    const int DJP = (p.kw + 1) >> 1;
    di = s / DJP;
    dj = 2 * (s - di * DJP) + kc;
    cin = j;
    return dj < p.kw;
}
// byte offset of K step s for output row r inside the halo, and the K-chunk stride (LBO)
__device__ __forceinline__ uint32_t ct_aoff(const ConvTParams& p, int r, int s, uint32_t& lbo) {
    if (p.G >= 2) {
        const int GP = (p.G + 1) >> 1, tap = s / GP, gp = s - tap * GP;
        const int di = tap / p.kw, dj = tap - di * p.kw;
        lbo = (uint32_t)p.P * 16;
        return (uint32_t)((((r + di) * p.G + 2 * gp) * p.P + dj) * 16);
    }
    const int DJP = (p.kw + 1) >> 1;
    const int di = s / DJP, djp = s - di * DJP;
    lbo = 16;  // the second K chunk is the same row one pixel on: tap dj + 1
    return (uint32_t)(((r + di) * p.P + 2 * djp) * 16);
}

constexpr uint32_t kLayoutNone = 0;
__device__ __forceinline__ uint64_t desc_none(uint32_t addr, uint32_t lbo) { return umma_desc(addr, lbo, 128, kLayoutNone); }

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}

__device__ __forceinline__ void ct_tile(const ConvTParams& p, int t, int& b, int& y0, int& x0) {
    const int per = p.tiles_x * p.tiles_y;
    b = t / per;
    const int rem = t - b * per;
    const int ty = rem / p.tiles_x;
    y0 = ty * p.R;
    x0 = (rem - ty * p.tiles_x) * p.Wt;
}

template <int MODE, bool X3>
struct CtRoles {
    static constexpr int kEpi0 = 2;                               // warps 2..5: epilogue
    static constexpr int kProd0 = 6;                              // warps 6..: lo split / dZ expansion
    static constexpr int kProdWarps = MODE == CT_DGRAD ? 8 : (X3 ? 4 : 0);
    static constexpr int kThreads = 32 * (kProd0 + kProdWarps);
};

template <int NK, int MODE, bool X3>
__global__ void __launch_bounds__(CtRoles<MODE, X3>::kThreads, 1)
    convt_mma_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapZdP,
                     const __grid_constant__ CUtensorMap mapZP, const __grid_constant__ CUtensorMap mapZc,
                     const ConvTParams p) {
    using Roles = CtRoles<MODE, X3>;
    constexpr int kMaxStages = 4;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* wsm = smem + p.stages * p.stage_bytes;  // weights hi | lo
    uint64_t* full = reinterpret_cast<uint64_t*>(wsm + 2 * p.w_bytes);
    uint64_t* ready = full + kMaxStages;
    uint64_t* empty = ready + kMaxStages;
    uint64_t* tfull = empty + kMaxStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
    uint64_t* zfull = reinterpret_cast<uint64_t*>(tslot + 2);  // DGRAD staging slots
    uint64_t* zempty = zfull + 2;
    uint64_t* dtab = zempty + 2;  // per K step: A descriptor (row 0, stage 0), B descriptor
    uint8_t* zst = reinterpret_cast<uint8_t*>(dtab + 2 * p.ksteps);  // 2 staging slots (DGRAD)
    zst = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(zst) + 127) & ~uintptr_t(127));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = p.stages;
    const int acc_cols = p.R * NK;
    uint32_t tcols = 32;
    while (tcols < (uint32_t)(2 * acc_cols)) tcols <<= 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], MODE == CT_DGRAD ? 32 * Roles::kProdWarps : 1);
            mbar_init(&ready[s], 32 * Roles::kProdWarps);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 128);
            mbar_init(&zfull[a], 1);
            mbar_init(&zempty[a], 32 * Roles::kProdWarps);
        }
        fence_barrier_init();
        if (MODE == CT_FWD) tma_prefetch(&mapX);
    }
    if (warp == 1) tmem_alloc(tslot, tcols);
    // zero the slack behind every halo buffer once (the MMA rows past the tile width read it)
    for (int s = 0; s < S; ++s)
        for (int h = 0; h < (X3 ? 2 : 1); ++h) {
            float4* z = reinterpret_cast<float4*>(smem + s * p.stage_bytes + h * (p.stage_bytes / 2) + p.halo_bytes);
            const int n = (X3 ? p.stage_bytes / 2 : p.stage_bytes) - p.halo_bytes;
            for (int i = threadIdx.x; i < n / 16; i += blockDim.x) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    pdl_wait();  // weights and inputs are written by earlier kernels of the step
    {  // weights, K-major no-swizzle: [kstep][kc][n][4]
        const int total = p.ksteps * 2 * NK * 4;
        for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
            const int j = idx & 3, n = (idx >> 2) % NK, kc = (idx / (4 * NK)) & 1, s = idx / (8 * NK);
            int cin, di, dj;
            float v = 0.0f;
            if (ct_kdecode(p, s, kc, j, cin, di, dj) && n < p.N) {
                if (MODE == CT_FWD) {
                    if (cin < p.wk_C) v = __ldg(p.wk + (((long long)n * p.wk_C + cin) * p.kh + di) * p.kw + dj);
                } else if (cin < p.wk_K) {  // flipped, transposed: Wf[n=c][k][di][dj] = W[k][c][kh-1-di][kw-1-dj]
                    v = __ldg(p.wk + (((long long)cin * p.wk_C + n) * p.kh + (p.kh - 1 - di)) * p.kw + (p.kw - 1 - dj));
                }
            }
            const int off = s * (2 * NK * 16) + kc * (NK * 16) + n * 16 + j * 4;
            *reinterpret_cast<float*>(wsm + off) = v;
            if (X3) *reinterpret_cast<float*>(wsm + p.w_bytes + off) = split_lo1(v);
        }
    }
    for (int ks = threadIdx.x; ks < p.ksteps; ks += blockDim.x) {  // descriptors, built once
        uint32_t lbo;
        const uint32_t ao = ct_aoff(p, 0, ks, lbo);
        dtab[2 * ks] = desc_none(smem_u32(smem) + ao, lbo);
        dtab[2 * ks + 1] = desc_none(smem_u32(wsm) + (uint32_t)(ks * (2 * NK * 16)), NK * 16);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tslot;
    const int half = X3 ? p.stage_bytes / 2 : 0;  // lo halo offset inside a stage

    if (warp == 0) {
        if (MODE == CT_FWD && lane == 0) {  // ---------------- TMA producer
            int it = 0;
            for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
                const int s = it % S;
                mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
                int b, y0, x0;
                ct_tile(p, t, b, y0, x0);
                mbar_arrive_expect_tx(&full[s], (uint32_t)p.halo_bytes);
                tma_load_5d(smem + s * p.stage_bytes, &mapX, &full[s], 0, x0 - p.pad, 0, y0 - p.pad, b);
            }
        } else if (MODE == CT_DGRAD && lane == 0 && p.z.tma) {  // ---------------- dP / P / codes staging
            int it = 0;
            for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
                const int zs = it & 1;
                mbar_wait(&zempty[zs], ((it >> 1) & 1) ^ 1);
                int b, y0, x0;
                ct_tile(p, t, b, y0, x0);
                const int Y0 = y0 - p.pad, X0 = x0 - p.pad;
                mbar_arrive_expect_tx(&zfull[zs], zs_tx_bytes(p.z));
                zs_issue(p.z, &mapZdP, &mapZP, &mapZc, zst + zs * p.zslot_bytes, &zfull[zs], b,
                         p.z.pool ? Y0 >> 1 : Y0, (p.z.pool ? X0 >> 1 : X0) & ~3);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            // descriptor arithmetic only touches the 14-bit start-address field (smem < 256 KB)
            const uint32_t idesc = umma_idesc_tf32(128, NK, 0, 0);
            const uint64_t a_lo_add = (uint64_t)(half >> 4), b_lo_add = (uint64_t)(p.w_bytes >> 4);
            const uint64_t row_add = (uint64_t)((p.G >= 2 ? p.G * p.P * 16 : p.P * 16) >> 4);
            int it = 0;
            for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
                const int s = it % S, buf = it & 1;
                mbar_wait(&tempty[buf], ((it >> 1) & 1) ^ 1);
                mbar_wait((MODE == CT_FWD && X3) ? &ready[s] : &full[s], (it / S) & 1);
                tc_fence_after();
                uint64_t a_add = (uint64_t)((s * p.stage_bytes) >> 4);
                for (int r = 0; r < p.R; ++r, a_add += row_add) {
                    const uint32_t tacc = tmem_base + (uint32_t)(buf * acc_cols + r * NK);
#pragma unroll 2
                    for (int ks = 0; ks < p.ksteps; ++ks) {
                        const uint64_t dah = dtab[2 * ks] + a_add, dbh = dtab[2 * ks + 1];
                        if (X3) {
                            mma_tf32(tacc, dah + a_lo_add, dbh, idesc, ks != 0);
                            mma_tf32(tacc, dah, dbh + b_lo_add, idesc, 1);
                            mma_tf32(tacc, dah, dbh, idesc, 1);
                        } else {
                            mma_tf32(tacc, dah, dbh, idesc, ks != 0);
                        }
                    }
                }
                mma_commit(&empty[s]);
                mma_commit(&tfull[buf]);
            }
            pdl_trigger();
        }
    } else if (warp >= Roles::kProd0) {
        const int pt = threadIdx.x - 32 * Roles::kProd0;
        constexpr int NP = 32 * Roles::kProdWarps;
        int it = 0;
        for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
            const int s = it % S;
            uint8_t* hi = smem + s * p.stage_bytes;
            if (MODE == CT_FWD) {  // ---------------- lo split of the TMA-landed halo
                mbar_wait(&full[s], (it / S) & 1);
                const uint32_t src = smem_u32(hi), dst = src + half;
                for (int i = pt * 16; i < p.halo_bytes; i += NP * 16) {
                    float x0, x1, x2, x3;
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(x0), "=f"(x1), "=f"(x2), "=f"(x3)
                                 : "r"(src + i));
                    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dst + i), "f"(split_lo1(x0)),
                                 "f"(split_lo1(x1)), "f"(split_lo1(x2)), "f"(split_lo1(x3))
                                 : "memory");
                }
                fence_proxy_async_smem();
                mbar_arrive(&ready[s]);
            } else {  // ---------------- dZ halo expansion (hi + lo) from the staged pooled tile
                int b, y0, x0;
                ct_tile(p, t, b, y0, x0);
                const int Y0 = y0 - p.pad, X0 = x0 - p.pad;
                const int sy0 = p.z.pool ? Y0 >> 1 : Y0, sx0 = (p.z.pool ? X0 >> 1 : X0) & ~3;
                const int zs = it & 1;
                uint8_t* slot = zst + zs * p.zslot_bytes;
                if (p.z.tma) {
                    mbar_wait(&zfull[zs], (it >> 1) & 1);
                } else {
                    zs_load_sync(p.z, slot, b, sy0, sx0, pt, NP);
                    asm volatile("bar.sync 1, %0;" ::"r"(NP) : "memory");
                }
                mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
                const int chunks = p.HR * p.G * p.P;
                for (int i = pt; i < chunks; i += NP) {
                    const int row = i / (p.G * p.P), rem = i - row * (p.G * p.P);
                    const int q = rem / p.P, col = rem - q * p.P;
                    const float4 d = zs_dz(p.z, slot, sy0, sx0, q, Y0 + row, X0 + col);
                    *reinterpret_cast<float4*>(hi + (long long)i * 16) = d;
                    if (X3)
                        *reinterpret_cast<float4*>(hi + half + (long long)i * 16) =
                            make_float4(split_lo1(d.x), split_lo1(d.y), split_lo1(d.z), split_lo1(d.w));
                }
                fence_proxy_async_smem();
                mbar_arrive(&full[s]);
                if (p.z.tma)
                    mbar_arrive(&zempty[zs]);
                else
                    asm volatile("bar.sync 1, %0;" ::"r"(NP) : "memory");
            }
        }
    } else {  // ---------------- epilogue: warps 2..5 -> TMEM lane quadrant warp % 4
        const int q = warp & 3;
        const int L = 32 * q + lane;
        const int Kq = (p.out.C + 3) >> 2;  // output channel quads actually stored
        int it = 0;
        for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
            const int buf = it & 1;
            mbar_wait(&tfull[buf], (it >> 1) & 1);
            tc_fence_after();
            int b, y0, x0;
            ct_tile(p, t, b, y0, x0);
            const int x = x0 + L;
            const bool xok = L < p.Wt && x < p.OW;
            const uint32_t trow = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * acc_cols);
            const int step = p.pool ? 2 : 1;
            for (int r = 0; r < p.R; r += step) {
                float v0[NK], v1[NK];
#pragma unroll
                for (int c0 = 0; c0 < NK; c0 += 8) {
                    float tt[8];
                    tmem_ld8(trow + r * NK + c0, tt);
#pragma unroll
                    for (int i = 0; i < 8; ++i) v0[c0 + i] = tt[i];
                }
                if (p.pool) {
#pragma unroll
                    for (int c0 = 0; c0 < NK; c0 += 8) {
                        float tt[8];
                        tmem_ld8(trow + (r + 1) * NK + c0, tt);
#pragma unroll
                        for (int i = 0; i < 8; ++i) v1[c0 + i] = tt[i];
                    }
                }
                const int y = y0 + r;
                if (MODE == CT_FWD) {
#pragma unroll
                    for (int n = 0; n < NK; ++n) {
                        const float bn = n < p.N ? __ldg(p.bias + n) : 0.0f;
                        v0[n] = n < p.N ? apply_act(p.act, v0[n] + bn) : 0.0f;  // layers.hpp:138-146 + act
                        if (p.pool) v1[n] = n < p.N ? apply_act(p.act, v1[n] + bn) : 0.0f;
                    }
                }
                if (p.pool) {
                    // 2x2 window: (y, x) (y, x+1) (y+1, x) (y+1, x+1) = codes 0..3, first maximum wins
                    const bool wok = xok && y + 1 < p.OH;
                    const int py = y >> 1, px = x >> 1;
                    const bool writer = wok && (lane & 1) == 0;
#pragma unroll
                    for (int g = 0; g < NK / 4; ++g) {
                        float o[4];
                        uint32_t cw = 0;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int n = 4 * g + j;
                            const float a1 = __shfl_xor_sync(0xffffffffu, v0[n], 1);
                            const float a3 = __shfl_xor_sync(0xffffffffu, v1[n], 1);
                            float best = v0[n];
                            uint32_t code = 0;
                            if (a1 > best) best = a1, code = 1;
                            if (v1[n] > best) best = v1[n], code = 2;
                            if (a3 > best) best = a3, code = 3;
                            o[j] = best;
                            cw |= code << (8 * j);
                        }
                        if (writer && g < Kq) {
                            if (p.out.blocked) {
                                *reinterpret_cast<float4*>(p.out.p + tl_quad(p.out, b, g, py, px)) =
                                    make_float4(o[0], o[1], o[2], o[3]);
                            } else {
                                float* base = p.out.p + (long long)b * p.out.bstride + (long long)py * p.out.W + px;
#pragma unroll
                                for (int j = 0; j < 4; ++j)
                                    if (4 * g + j < p.out.C) base[(long long)(4 * g + j) * p.out.H * p.out.W] = o[j];
                            }
                            *reinterpret_cast<uint32_t*>(p.codes + (long long)b * p.codes_bstride +
                                                         (((long long)py * Kq + g) * p.codes_pw + px) * 4) = cw;
                        }
                    }
                } else if (xok && y < p.OH) {
#pragma unroll
                    for (int g = 0; g < NK / 4; ++g) {
                        if (g >= Kq) break;
                        if (p.out.blocked) {
                            *reinterpret_cast<float4*>(p.out.p + tl_quad(p.out, b, g, y, x)) =
                                make_float4(v0[4 * g], v0[4 * g + 1], v0[4 * g + 2], v0[4 * g + 3]);
                        } else {
                            float* base = p.out.p + (long long)b * p.out.bstride + (long long)y * p.out.W + x;
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                if (4 * g + j < p.out.C) base[(long long)(4 * g + j) * p.out.H * p.out.W] = v0[4 * g + j];
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[buf]);
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, tcols);
    }
}

// ------------------------------------------------------------------ weight gradient (FFMA, exact fp32)
struct ConvTWParams {
    int B, Cp, G, H, W, kh, kw, pad, OH, OW;  // layer geometry (input H x W, Cp channels; conv output OH x OW)
    int K, Kp, C;                             // real kernels, padded, real channels
    int R, Wt, P, HR, tiles_x, tiles_y, ntiles;
    int halo_bytes, slot_bytes;               // X halo; one (halo | dZ staging) slot
    DZSrc z;
    float* ws;  // per-CTA partials [cta][Kp*Cp*kh*kw + Kp]
    int ws_stride;
};

constexpr int kWgThreads = 256;
constexpr int kWgChunk = 16;  // output columns per sliding-window run

// Thread (stream st, channel c, kernel quad kq) owns dW[4kq..4kq+3][c][.][.] over the pixel runs of its
// stream. Per tile the X halo and the pooled dP / P / codes arrive by TMA into a double-buffered slot
// (the next tile's loads fly while this one computes); dZ is expanded from the slot into smem.
template <int KH, int KW>
__global__ void __launch_bounds__(kWgThreads, 1)
    convt_wgrad_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapZdP,
                       const __grid_constant__ CUtensorMap mapZP, const __grid_constant__ CUtensorMap mapZc,
                       const ConvTWParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* slots[2] = {smem, smem + p.slot_bytes};  // [X halo | dZ staging]
    const int hb = (p.halo_bytes + 127) & ~127;
    float* dz = reinterpret_cast<float*>(smem + 2 * p.slot_bytes);  // [R][Kq][Wt][4]
    const int Kq = p.Kp >> 2;
    const int dz_floats = p.R * p.Kp * p.Wt;
    uint64_t* full = reinterpret_cast<uint64_t*>(dz + dz_floats);
    float* red = reinterpret_cast<float*>(full + 4);  // CTA reduction scratch

    const int TPS = p.C * Kq;
    const int streams = kWgThreads / TPS;
    const int st = threadIdx.x / TPS, w = threadIdx.x - st * TPS;
    const int c = w % p.C, kq = w / p.C;
    const bool active = st < streams;
    constexpr int T = KH * KW;
    float acc[4][T];
    float bacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < T; ++i) acc[j][i] = 0.0f;

    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_barrier_init();
        tma_prefetch(&mapX);
    }
    __syncthreads();
    pdl_wait();
    auto tile_of = [&](int t, int& b, int& y0, int& x0) {
        const int per = p.tiles_x * p.tiles_y;
        b = t / per;
        const int rem = t - b * per, ty = rem / p.tiles_x;
        y0 = ty * p.R;
        x0 = (rem - ty * p.tiles_x) * p.Wt;
    };
    auto issue = [&](int t, int sl) {
        int b, y0, x0;
        tile_of(t, b, y0, x0);
        mbar_arrive_expect_tx(&full[sl], (uint32_t)p.halo_bytes + (p.z.tma ? zs_tx_bytes(p.z) : 0u));
        tma_load_5d(slots[sl], &mapX, &full[sl], 0, x0 - p.pad, 0, y0 - p.pad, b);
        if (p.z.tma)
            zs_issue(p.z, &mapZdP, &mapZP, &mapZc, slots[sl] + hb, &full[sl], b, p.z.pool ? y0 >> 1 : y0,
                     (p.z.pool ? x0 >> 1 : x0) & ~3);
    };
    if (threadIdx.x == 0 && (int)blockIdx.x < p.ntiles) issue(blockIdx.x, 0);
    int it = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
        const int sl = it & 1;
        int b, y0, x0;
        tile_of(t, b, y0, x0);
        const int sy0 = p.z.pool ? y0 >> 1 : y0, sx0 = (p.z.pool ? x0 >> 1 : x0) & ~3;
        uint8_t* zslot = slots[sl] + hb;
        mbar_wait(&full[sl], (it >> 1) & 1);
        if (!p.z.tma) {
            zs_load_sync(p.z, zslot, b, sy0, sx0, threadIdx.x, kWgThreads);
            __syncthreads();
        }
        for (int i = threadIdx.x; i < p.R * Kq * p.Wt; i += kWgThreads) {  // dZ of the tile
            const int r = i / (Kq * p.Wt), rem = i - r * (Kq * p.Wt), q = rem / p.Wt, xx = rem - q * p.Wt;
            const int Y = y0 + r, X = x0 + xx;
            reinterpret_cast<float4*>(dz)[i] = zs_dz(p.z, zslot, sy0, sx0, q, Y, X);
        }
        __syncthreads();  // dz ready; the other slot (previous tile) is free
        if (threadIdx.x == 0 && t + (int)gridDim.x < p.ntiles) issue(t + gridDim.x, sl ^ 1);
        if (active) {
            const float* hx = reinterpret_cast<const float*>(slots[sl]);
            const int cq = c >> 2, cj = c & 3;
            const int runs_per_row = (p.Wt + kWgChunk - 1) / kWgChunk;
            for (int u = st; u < p.R * runs_per_row; u += streams) {
                const int r = u / runs_per_row, xb = (u - r * runs_per_row) * kWgChunk;
                const int xe = min(min(p.Wt, xb + kWgChunk), p.OW - x0);
                if (y0 + r >= p.OH || xb >= xe) continue;
                float win[KH][KW];
#pragma unroll
                for (int di = 0; di < KH; ++di)
#pragma unroll
                    for (int dj = 0; dj < KW - 1; ++dj)
                        win[di][dj + 1] = hx[(((r + di) * p.G + cq) * p.P + xb + dj) * 4 + cj];
                for (int xx = xb; xx < xe; ++xx) {
#pragma unroll
                    for (int di = 0; di < KH; ++di) {
#pragma unroll
                        for (int dj = 0; dj < KW - 1; ++dj) win[di][dj] = win[di][dj + 1];
                        win[di][KW - 1] = hx[(((r + di) * p.G + cq) * p.P + xx + KW - 1) * 4 + cj];
                    }
                    const float4 d4 = reinterpret_cast<const float4*>(dz)[(r * Kq + kq) * p.Wt + xx];
                    const float dd[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
#pragma unroll
                        for (int di = 0; di < KH; ++di)
#pragma unroll
                            for (int dj = 0; dj < KW; ++dj)
                                acc[j][di * KW + dj] = fmaf(dd[j], win[di][dj], acc[j][di * KW + dj]);
                        bacc[j] += dd[j];
                    }
                }
            }
        }
        __syncthreads();  // slot and dz consumed
    }
    pdl_trigger();
    // fixed-order reduction over the streams of this CTA, then one partial row per CTA
    const int nval = 4 * T + 4;
    if (active)
        for (int j = 0; j < 4; ++j) {
            for (int i = 0; i < T; ++i) red[((long long)st * TPS + w) * nval + j * T + i] = acc[j][i];
            red[((long long)st * TPS + w) * nval + 4 * T + j] = bacc[j];
        }
    __syncthreads();
    float* out = p.ws + (long long)blockIdx.x * p.ws_stride;
    const int nk = p.Kp * p.Cp * T;
    for (int idx = threadIdx.x; idx < nk + p.Kp; idx += kWgThreads) {
        int ww = -1, slotv = 0;
        if (idx < nk) {  // idx = ((k * Cp + c) * T + tap)
            const int k = idx / (p.Cp * T), rem = idx - k * (p.Cp * T), cc = rem / T, tap = rem - cc * T;
            if (cc < p.C) {
                ww = (k >> 2) * p.C + cc;
                slotv = (k & 3) * T + tap;
            }
        } else {  // bias of kernel k: the c == 0 threads' dZ sums
            const int k = idx - nk;
            ww = (k >> 2) * p.C;
            slotv = 4 * T + (k & 3);
        }
        float sum = 0.0f;
        if (ww >= 0)
            for (int q = 0; q < streams; ++q) sum += red[((long long)q * TPS + ww) * nval + slotv];
        out[idx] = sum;
    }
}

// sum of the per-CTA partials in CTA order (warp-parallel, fixed shuffle tree) + the optimizer step
// on kernels and bias (sgd_momentum_step, optim.hpp:69-80) or a plain gradient store (DP split mode)
static __global__ void convt_wgrad_reduce_kernel(const float* __restrict__ ws, int nctas, int ws_stride, int K, int Kp,
                                                 int C, int Cp, int T, float* kern, float* kvel, float* bias,
                                                 float* bvel, float* gk, float* gb, int fused, float lr, float mom,
                                                 float wd) {
    pdl_wait();
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = K * C * T + K;
    if (wid >= nw) return;
    int src;
    float *pp, *vv, *gg;
    if (wid < K * C * T) {  // W[k][c][tap] (dense, real C)
        const int k = wid / (C * T), rem = wid - k * (C * T), c = rem / T, tap = rem - c * T;
        src = (k * Cp + c) * T + tap;
        pp = kern + wid;
        vv = kvel + wid;
        gg = gk + wid;
    } else {
        const int k = wid - K * C * T;
        src = Kp * Cp * T + k;
        pp = bias + k;
        vv = bvel + k;
        gg = gb + k;
    }
    float s = 0.0f;
    for (int q = lane; q < nctas; q += 32) s += ws[(long long)q * ws_stride + src];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane) return;
    if (fused) {
        const float g = s + wd * *pp;
        const float v = mom * *vv - lr * g;
        *vv = v;
        *pp = *pp + v;
    } else {
        *gg = s;
    }
}

// NCHW (C real channels, per-image pitch ld) -> row-blocked [b][y][Cp/4][x][4], zero channels past C
static __global__ void convt_repack_kernel(const float* __restrict__ x, long long ld, int B, int C, int H, int W,
                                           float* __restrict__ out, long long obstride) {
    pdl_wait();
    const int G = (C + 3) >> 2;
    const long long n = (long long)B * H * G * W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int xx = (int)(i % W);
        long long r = i / W;
        const int q = (int)(r % G);
        r /= G;
        const int y = (int)(r % H);
        const int b = (int)(r / H);
        const float* src = x + (long long)b * ld + (long long)y * W + xx;
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = 4 * q + j < C ? __ldg(src + (long long)(4 * q + j) * H * W) : 0.0f;
        *reinterpret_cast<float4*>(out + (long long)b * obstride + ((long long)(y * G + q) * W + xx) * 4) =
            make_float4(v[0], v[1], v[2], v[3]);
    }
}

// ------------------------------------------------------------------ host planning
// 5-D map over a row-blocked tensor: dims {4 ch, W, G quads, H, B}; box {4, P, G, HR, 1}; OOB -> 0
inline CUtensorMap make_map_blocked(const float* base, int B, int G, int H, int W, long long bstride, int P, int HR) {
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (bstride & 3))
        throw Error(B2N_EINTERNAL, "row-blocked activation must be 16-byte aligned");
    if (P > 256 || HR > 256 || G > 256) throw Error(B2N_ESHAPE, "conv halo box exceeds the TMA box limits");
    CUtensorMap m;
    cuuint64_t dims[5] = {4, (cuuint64_t)W, (cuuint64_t)G, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t strides[4] = {16, (cuuint64_t)W * 16, (cuuint64_t)G * W * 16, (cuuint64_t)bstride * 4};
    cuuint32_t box[5] = {4, (cuuint32_t)P, (cuuint32_t)G, (cuuint32_t)HR, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(B2N_ECUDA, "cuTensorMapEncodeTiled (5-D halo) failed: " + std::to_string((int)r));
    return m;
}

// 4-D map over the row-blocked argmax code rows, elements = uint32 (one code byte per channel of a quad)
inline CUtensorMap make_map_codes(const uint8_t* base, int B, int Kq, int PH, int PWc, long long bstride_bytes, int bw,
                                  int bh) {
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (bstride_bytes & 15) || (PWc & 3))
        throw Error(B2N_EINTERNAL, "argmax code rows must be 16-byte aligned");
    CUtensorMap m;
    cuuint64_t dims[4] = {(cuuint64_t)PWc, (cuuint64_t)Kq, (cuuint64_t)PH, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)PWc * 4, (cuuint64_t)Kq * PWc * 4, (cuuint64_t)bstride_bytes};
    cuuint32_t box[4] = {(cuuint32_t)bw, (cuuint32_t)Kq, (cuuint32_t)bh, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<uint8_t*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(B2N_ECUDA, "cuTensorMapEncodeTiled (codes) failed: " + std::to_string((int)r));
    return m;
}
// staging maps of a dZ source for its window (z.bh x z.bw); zeroed when staged by thread loads
inline void dz_maps(const DZSrc& z, int B, CUtensorMap out[3]) {
    std::memset(out, 0, 3 * sizeof(CUtensorMap));
    if (!z.tma) return;
    out[0] = make_map_blocked(z.dP.p, B, z.Kq, z.dP.H, z.dP.W, z.dP.bstride, z.bw, z.bh);
    out[1] = make_map_blocked(z.P.p, B, z.Kq, z.P.H, z.P.W, z.P.bstride, z.bw, z.bh);
    if (z.pool) out[2] = make_map_codes(z.codes, B, z.Kq, z.dP.H, z.PWc, z.codes_bstride, z.bw, z.bh);
}

// tile shape for an OH x OW correlation output: Wt <= 128 columns, R (even) rows, 2*R*NK TMEM columns <= 512
inline void ct_tile_shape(int OH, int OW, int NK, int& R, int& Wt) {
    Wt = std::min(OW, 128);
    if (Wt & 1) ++Wt;
    R = (128 + Wt - 1) / Wt;
    R = std::max(2, (R + 1) & ~1);
    const int ohe = (OH + 1) & ~1;
    R = std::min(R, std::max(2, ohe));
    while (2 * R * NK > 512 && R > 2) R -= 2;
}

inline int ct_nk(int n) {
    if (n <= 8) return 8;
    if (n <= 16) return 16;
    if (n <= 32) return 32;
    throw Error(B2N_ESHAPE, "b200nn conv: at most 32 kernels / channels per layer on the tensor-core path");
}

struct ConvTLaunch {
    ConvTParams p;
    CUtensorMap map;
    CUtensorMap zmaps[3];  // DGRAD: dP, P, codes staging maps
    int mode = CT_FWD, nk = 16, grid = 1, smem = 0;
    bool x3 = true;
    double flops = 0, bytes = 0;
    void run(cudaStream_t st) const;
};

// correlation plan shared by FWD and DGRAD
inline ConvTLaunch plan_convt(int mode, int B, int Cp, int Hin, int Win, int kh, int kw, int pad, int N, bool x3,
                              const DZSrc* z = nullptr) {
    ConvTLaunch L;
    ConvTParams& p = L.p;
    std::memset(&p, 0, sizeof(p));
    L.mode = mode;
    L.x3 = x3;
    L.nk = ct_nk(N);
    p.B = B;
    p.Cp = Cp;
    p.G = Cp / 4;
    p.Hin = Hin;
    p.Win = Win;
    p.kh = kh;
    p.kw = kw;
    p.pad = pad;
    p.OH = Hin + 2 * pad - kh + 1;
    p.OW = Win + 2 * pad - kw + 1;
    p.N = N;
    ct_tile_shape(p.OH, p.OW, L.nk, p.R, p.Wt);
    p.P = p.Wt + kw - 1;
    p.HR = p.R + kh - 1;
    p.tiles_x = (p.OW + p.Wt - 1) / p.Wt;
    p.tiles_y = (p.OH + p.R - 1) / p.R;
    p.ntiles = B * p.tiles_x * p.tiles_y;
    p.ksteps = p.G >= 2 ? kh * kw * ((p.G + 1) / 2) : kh * ((kw + 1) / 2);
    p.halo_bytes = p.HR * p.G * p.P * 16;
    // MMA rows past the tile width read at most (kw + 128) * 16 bytes beyond the halo (ct_aoff)
    const int slack = (kw + 129) * 16;
    const int one = (p.halo_bytes + slack + 127) & ~127;
    p.stage_bytes = one * (x3 ? 2 : 1);
    p.w_bytes = p.ksteps * 2 * L.nk * 16;
    std::memset(L.zmaps, 0, sizeof(L.zmaps));
    if (z) {  // DGRAD: pooled window covering the dZ halo rows / cols of a tile
        p.z = *z;
        p.z.bh = z->pool ? p.HR / 2 + 1 : p.HR;
        p.z.bw = ((z->pool ? p.P / 2 + 1 : p.P) + 6) & ~3;  // window start is aligned down to 4 (TMA: 16 B)
        p.zslot_bytes = (zs_bytes(p.z) + 127) & ~127;
        dz_maps(p.z, B, L.zmaps);
    }
    const int fixed = 2 * p.w_bytes + 1024 + 256 + p.ksteps * 16 + 128 + 2 * p.zslot_bytes;
    const int budget = 220 * 1024;
    p.stages = std::min(4, (budget - fixed) / p.stage_bytes);
    if (p.stages < 2) throw Error(B2N_ESHAPE, "b200nn conv: halo tile does not fit shared memory");
    L.smem = p.stages * p.stage_bytes + fixed;
    L.grid = std::min(p.ntiles, sm_count());
    L.flops = 2.0 * B * p.OH * p.OW * N * (double)Cp * kh * kw;
    return L;
}

template <int NK, int MODE, bool X3>
inline void launch_convt_inst(const ConvTLaunch& L, cudaStream_t st) {
    auto k = convt_mma_kernel<NK, MODE, X3>;
    static int attr_set = 0;
    if (attr_set < L.smem) {
        B2N_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr_set = 227 * 1024;
    }
    launch_ex(k, dim3(L.grid), dim3(CtRoles<MODE, X3>::kThreads), (size_t)L.smem, st, 1u, L.map, L.zmaps[0],
              L.zmaps[1], L.zmaps[2], L.p);
}
template <int MODE>
void launch_convt(const ConvTLaunch& L, cudaStream_t st);
#ifndef B2N_CONVT_INSTANTIATE
extern template void launch_convt<CT_FWD>(const ConvTLaunch&, cudaStream_t);
extern template void launch_convt<CT_DGRAD>(const ConvTLaunch&, cudaStream_t);
#else
template <int MODE>
void launch_convt(const ConvTLaunch& L, cudaStream_t st) {
    switch (L.nk) {
        case 8: L.x3 ? launch_convt_inst<8, MODE, true>(L, st) : launch_convt_inst<8, MODE, false>(L, st); break;
        case 16: L.x3 ? launch_convt_inst<16, MODE, true>(L, st) : launch_convt_inst<16, MODE, false>(L, st); break;
        default: L.x3 ? launch_convt_inst<32, MODE, true>(L, st) : launch_convt_inst<32, MODE, false>(L, st); break;
    }
}
#endif
inline void ConvTLaunch::run(cudaStream_t st) const {
    if (mode == CT_FWD)
        launch_convt<CT_FWD>(*this, st);
    else
        launch_convt<CT_DGRAD>(*this, st);
}

struct ConvTWLaunch {
    ConvTWParams p;
    CUtensorMap map;
    CUtensorMap zmaps[3];
    int grid = 1, smem = 0;
    std::shared_ptr<DevMem> ws;
    float *kern = nullptr, *kvel = nullptr, *bias = nullptr, *bvel = nullptr, *gk = nullptr, *gb = nullptr;
    float lr = 0, mom = 0, wd = 0;
    double flops = 0, bytes = 0;
    void run(cudaStream_t st, bool fused) const;
};

void launch_convt_wgrad(const ConvTWLaunch& L, cudaStream_t st);

// weight gradient over the forward plan's tiles (same X halo map): ws = one partial row per CTA
inline ConvTWLaunch plan_convt_wgrad(const ConvTLaunch& f, int K, int C, const DZSrc& z0) {
    ConvTWLaunch L;
    ConvTWParams& p = L.p;
    std::memset(&p, 0, sizeof(p));
    const ConvTParams& q = f.p;
    p.B = q.B;
    p.Cp = q.Cp;
    p.G = q.G;
    p.H = q.Hin;
    p.W = q.Win;
    p.kh = q.kh;
    p.kw = q.kw;
    p.pad = q.pad;
    p.OH = q.OH;
    p.OW = q.OW;
    p.K = K;
    p.Kp = (K + 3) & ~3;
    p.C = C;
    p.R = q.R;
    p.Wt = q.Wt;
    p.P = q.P;
    p.HR = q.HR;
    p.tiles_x = q.tiles_x;
    p.tiles_y = q.tiles_y;
    p.ntiles = q.ntiles;
    p.halo_bytes = q.halo_bytes;
    p.z = z0;
    p.z.bh = z0.pool ? q.R / 2 : q.R;
    p.z.bw = ((z0.pool ? q.Wt / 2 : q.Wt) + 6) & ~3;  // window start is aligned down to 4 (TMA: 16 B)
    if (!((p.kh == 3 && p.kw == 3) || (p.kh == 5 && p.kw == 5)))
        throw Error(B2N_EINTERNAL, "convt wgrad: only 3x3 and 5x5 filters are instantiated");
    const int T = p.kh * p.kw;
    const int TPS = C * (p.Kp / 4);
    if (TPS > kWgThreads) throw Error(B2N_ESHAPE, "convt wgrad: channels x kernel quads exceed one CTA");
    const int streams = kWgThreads / TPS;
    p.ws_stride = (p.Kp * p.Cp * T + p.Kp + 3) & ~3;
    p.slot_bytes = (((p.halo_bytes + 127) & ~127) + zs_bytes(p.z) + 1023) & ~1023;
    L.map = f.map;
    dz_maps(p.z, p.B, L.zmaps);
    L.grid = std::min(p.ntiles, sm_count());
    L.smem = 1024 + 2 * p.slot_bytes + p.R * p.Kp * p.Wt * 4 + 64 + streams * TPS * (4 * T + 4) * 4;
    if (L.smem > 227 * 1024) throw Error(B2N_ESHAPE, "convt wgrad: tile does not fit shared memory");
    L.ws = std::make_shared<DevMem>();
    L.ws->alloc((size_t)L.grid * p.ws_stride * 4);
    p.ws = L.ws->as<float>();
    const double opix = (double)p.B * p.OH * p.OW;
    L.flops = 2.0 * opix * K * ((double)C * T + 1);
    const double pooled = (double)p.B * K * (z0.pool ? (p.OH / 2) * (p.OW / 2) : p.OH * p.OW);
    L.bytes = (double)p.B * p.H * p.W * C * 4 + pooled * 9 + (double)K * (C * T + 1) * 16;
    return L;
}

inline void ConvTWLaunch::run(cudaStream_t st, bool fused) const {
    launch_convt_wgrad(*this, st);
    const int T = p.kh * p.kw;
    const int nw = p.K * p.C * T + p.K;
    launch_ex(convt_wgrad_reduce_kernel, dim3((nw * 32 + 255) / 256), dim3(256), 0, st, 1u, (const float*)p.ws, grid,
              p.ws_stride, p.K, p.Kp, p.C, p.Cp, T, kern, kvel, bias, bvel, gk, gb, fused ? 1 : 0, lr, mom, wd);
}

}  // namespace b2n
