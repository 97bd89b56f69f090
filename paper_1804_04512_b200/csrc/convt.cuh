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

// the same for the two conv-output rows Ye (even) and Ye + 1 of one pooled row at column X: one
// read of the pooled cell (dP, P, codes) and one act' per channel feed both (pooled layers only)
__device__ __forceinline__ void zs_dz2(const DZSrc& z, const uint8_t* slot, int sy0, int sx0, int q, int Ye, int X,
                                       float4& d0, float4& d1) {
    d0 = d1 = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool vx = (unsigned)X < (unsigned)z.OWz;
    const bool v0 = vx && (unsigned)Ye < (unsigned)z.OHz, v1 = vx && (unsigned)(Ye + 1) < (unsigned)z.OHz;
    if (!(v0 || v1)) return;
    const int idx = (((Ye >> 1) - sy0) * z.Kq + q) * z.bw + ((X >> 1) - sx0);
    const float4 g = reinterpret_cast<const float4*>(slot)[idx];
    const float4 y = reinterpret_cast<const float4*>(slot + zs_off_p(z))[idx];
    const uint32_t cw = reinterpret_cast<const uint32_t*>(slot + 2 * zs_off_p(z))[idx];
    const float a[4] = {act_grad(z.act, g.x, y.x), act_grad(z.act, g.y, y.y), act_grad(z.act, g.z, y.z),
                        act_grad(z.act, g.w, y.w)};
    const uint32_t w0 = (uint32_t)(X & 1), w1 = w0 + 2u;
    float e0[4], e1[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t c = (cw >> (8 * j)) & 0xFFu;
        e0[j] = v0 && c == w0 ? a[j] : 0.0f;
        e1[j] = v1 && c == w1 ? a[j] : 0.0f;
    }
    d0 = make_float4(e0[0], e0[1], e0[2], e0[3]);
    d1 = make_float4(e1[0], e1[1], e1[2], e1[3]);
}

enum ConvTMode : int { CT_FWD = 0, CT_DGRAD = 1 };
constexpr int kCtMaxKSteps = 16;  // K steps per halo row: kw * ceil(quads / 2) (or ceil(kw / 2) for one quad)

struct ConvTParams {
    // the correlation this launch computes: input Hin x Win, Cp = 4*G channels, kh x kw, pad
    int B, Cp, G, Hin, Win, kh, kw, pad, OH, OW;
    int N;             // real output channels
    int R, Wt, P, HR;  // output rows / cols per tile, halo cols / rows
    int tiles_x, tiles_y, ntiles;
    int ksteps, slots, stages;  // K steps per halo row, TMEM row slots per buffer
    int halo_bytes;             // fp32 halo [HR][G][P][4]
    int h_bytes;                // one halo buffer incl. the slack MMA rows past the tile read
    int stage_bytes, w_bytes;       // smem carve-up (host-computed)
    int stack;                      // 3xTF32 with B hi|lo interleaved along N: 2 MMAs per K step (below)
    const float* x;     // FWD input, row-blocked [b][y][G][Win][4]
    long long x_bstride;
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
    // FWD + pool, 3xTF32: exact resolution of the pooling decisions the tensor-core rounding could flip
    // (ct_fix_window). fix_list = per-CTA item lists ([grid][fix_cap]), null disables it; fix_cb = the
    // rigorous per-term bound of |Z_tc - Z_ref| / sum|k x| for this layer's chain length (host-computed)
    unsigned* fix_list;
    long long fix_cap;
    float fix_cb;
    unsigned long long* trace;  // bring-up: per-tile role timestamps of CTA 0 (clock64), null in production
    int dbg;                    // bring-up bisection (B2N_CT_DBG): 1 no lo split, 2 no epilogue work, 4 no halo copy
};
#define CT_TRACE(it, ev)                                                                  \
    do {                                                                                  \
        if (p.trace && blockIdx.x == 0 && (it) < 64 && p.trace[(it) * 8 + (ev)] == 0)        \
            p.trace[(it) * 8 + (ev)] = clock64();                                                \
    } while (0)

// K step s of a halo row (tf32, K = 8 = two 16-byte chunks kc of 4 channels) -> correlation input
// channel / tap column of element j (0..3) of chunk kc. G >= 2 quads: s = (dj, quad pair), the two
// chunks are quads 2gp and 2gp+1 (a plane apart); G == 1: s = tap pair, the second chunk is the same
// quad one pixel on (tap dj + 1). The filter row di is not part of K: it is stacked along N.
__device__ __forceinline__ bool ct_kdecode(const ConvTParams& p, int s, int kc, int j, int& cin, int& dj) {
    if (p.G >= 2) {
        const int GP = (p.G + 1) >> 1;
        dj = s / GP;
        const int q = 2 * (s - dj * GP) + kc;
        cin = 4 * q + j;
        return q < p.G;
    }
    dj = 2 * s + kc;
    cin = j;
    return dj < p.kw;
}
// byte offset of K step s inside a halo row, and the K-chunk stride (LBO)
__device__ __forceinline__ uint32_t ct_aoff(const ConvTParams& p, int s, uint32_t& lbo) {
    if (p.G >= 2) {
        const int GP = (p.G + 1) >> 1, dj = s / GP, gp = s - dj * GP;
        lbo = (uint32_t)p.P * 16;
        return (uint32_t)((2 * gp * p.P + dj) * 16);
    }
    lbo = 16;  // the second K chunk is the same row one pixel on: tap dj + 1
    return (uint32_t)(2 * s * 16);
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

// 1-D bulk copy global -> shared (sizes / addresses multiples of 16 B), completing on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// Input halo rows [ys, ys + HR) x cols [xs, xs + P) of a row-blocked tensor [b][y][G][W][4] into smem
// [HR][G][P][4]: one bulk copy per (row, quad) of the in-range columns (a ~P*16-byte contiguous run),
// zeros for the padding. A whole warp calls it: lanes zero-fill, lane 0 arms `bar` and issues the
// copies. (A 5-D TMA box would have a 16-byte innermost extent: thousands of tiny TMA lines.)
__device__ __forceinline__ void halo_load_warp(const float* base, long long bstride, int G, int H, int W, int b, int ys,
                                               int xs, int HR, int P, uint8_t* dst, uint64_t* bar, int lane) {
    const int xa = max(xs, 0), xe = min(xs + P, W);
    const int ncol = xe - xa;
    const int lz = ncol > 0 ? xa - xs : P;            // zero columns on the left (all when no overlap)
    const int rz = ncol > 0 ? xs + P - xe : 0;        // zero columns on the right
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int row = lane; row < HR * G; row += 32) {
        const int hr = row / G;
        float4* d = reinterpret_cast<float4*>(dst + (long long)row * P * 16);
        const int y = ys + hr;
        if ((unsigned)y >= (unsigned)H || ncol <= 0) {
            for (int c = 0; c < P; ++c) d[c] = z4;
        } else {
            for (int c = 0; c < lz; ++c) d[c] = z4;
            for (int c = P - rz; c < P; ++c) d[c] = z4;
        }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
        const int y_lo = max(ys, 0), y_hi = min(ys + HR, H);
        const int rows = ncol > 0 && y_hi > y_lo ? (y_hi - y_lo) * G : 0;
        mbar_arrive_expect_tx(bar, (uint32_t)(rows * ncol * 16));
        for (int y = y_lo; rows && y < y_hi; ++y)
            for (int g = 0; g < G; ++g)
                bulk_g2s(dst + ((long long)((y - ys) * G + g) * P + lz) * 16,
                         base + (long long)b * bstride + (((long long)y * G + g) * W + xa) * 4, (uint32_t)ncol * 16, bar);
    }
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
    static constexpr int kEpi0 = 2;                               // warps 2..9: epilogue
    static constexpr int kProd0 = 10;                             // warps 10..: lo split / dZ expansion
    static constexpr int kProdWarps = MODE == CT_DGRAD ? 8 : 4;
    static constexpr int kThreads = 32 * (kProd0 + kProdWarps);
};

// warp-converged MMA issue: the whole warp runs the loop, one elected lane issues (a lone divergent
// issuing thread costs ~2x per tcgen05.mma, measured)
__device__ __forceinline__ void mma_tf32_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
        "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc)
        : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
        "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar))
        : "memory");
}
// zero 16 consecutive TMEM columns of this warp's 32 lanes
__device__ __forceinline__ void tmem_zero16(uint32_t taddr) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
        "r"(0u)
        : "memory");
}
__device__ __forceinline__ void tmem_zero8(uint32_t taddr) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(0u)
                 : "memory");
}
__device__ __forceinline__ void tmem_zero4(uint32_t taddr) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" ::"r"(taddr), "r"(0u) : "memory");
}
template <int N>
__device__ __forceinline__ void tmem_zeron(uint32_t taddr) {
    if constexpr (N == 4) tmem_zero4(taddr);
    else if constexpr (N == 8) tmem_zero8(taddr);
    else
#pragma unroll
        for (int c = 0; c < N; c += 16) tmem_zero16(taddr + c);
}

// Epilogue of one warp over all tiles of the CTA: TMEM lane quadrant q (pixels 32q..32q+31 of each
// tile row), channels [hsel*NK/2, (hsel+1)*NK/2). Specialised on activation / pooling / output layout.
// FWD: bias + act (layers.hpp:138-146, :278-282), then the 2x2 max with the reference's first-index
// tie rule over window order (0,0) (0,1) (1,0) (1,1) (layers.hpp:228-232) -> pooled value + code byte.
//
// Exact pooling decisions (FWD + pool, 3xTF32, p.fix_list set). The reference computes every conv
// output as ONE fp32 fma chain over (c, di, dj) plus the bias (conv.hpp:62-119, layers.hpp:138-146);
// the tensor-core value differs from it by at most tau = fix_cb * sum|k x| (+ the bias-add rounding),
// and sum|k x| <= ||k||_1 * max|x| over the tile's input halo (measured by the lo-split warps). A window
// whose first-index argmax -- or, for relu, whether the routed value is > 0 -- is not decided with that
// margin is appended to the CTA's fix list; the CTA recomputes it at its end with the reference's own
// chain (ct_fix_window), so pooled codes and relu' are the reference's, not a rounding artefact.
template <int NK, int ACT, bool POOL, bool BLOCKED, int MODE>
__device__ __forceinline__ void ct_epilogue(const ConvTParams& p, uint32_t tmem_base, int bufcols, uint64_t* tfull,
                                            uint64_t* tempty, int q, int hsel, int lane, const float* xmr,
                                            unsigned* fixcnt) {
    constexpr int NH = NK / 2;   // channels of this warp
    constexpr int NQ = (NH + 3) / 4;
    const int c_lo = hsel * NH;
    const int L = 32 * q + lane;
    const uint32_t tq = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)c_lo;
    const int SW = p.stack ? 2 * NK : NK;  // row-slot width: [a.b_hi + a_lo.b_hi | a_hi.b_lo] when stacked
    // output row r of buffer buf accumulates in row slot HR-1-r (see convt_mma_kernel); zero the real
    // slots of both buffers once, then after every drain
    auto zero_rows = [&](int buf) {
        for (int r = 0; r < p.R; ++r) {
            tmem_zeron<NH>(tq + (uint32_t)(buf * bufcols + (p.HR - 1 - r) * SW));
            if (p.stack) tmem_zeron<NH>(tq + (uint32_t)(buf * bufcols + (p.HR - 1 - r) * SW + NK));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    };
    zero_rows(0);
    zero_rows(1);
    tc_fence_before();
    mbar_arrive(&tempty[0]);
    mbar_arrive(&tempty[1]);
    const int Kq = (p.out.C + 3) >> 2;  // channel quads actually stored
    float bias_r[NH];
#pragma unroll
    for (int j = 0; j < NH; ++j) bias_r[j] = (MODE == CT_FWD && c_lo + j < p.N) ? __ldg(p.bias + c_lo + j) : 0.0f;
    // fix_cb * ||k_j||_1 per channel of this warp (0: no fix-up)
    constexpr bool kFix = MODE == CT_FWD && POOL;
    const bool fix = kFix && p.fix_list != nullptr;
    float tk[NH];
#pragma unroll
    for (int j = 0; j < NH; ++j) {
        float a = 0.0f;
        if (fix && c_lo + j < p.N)
            for (int i = 0; i < p.wk_C * p.kh * p.kw; ++i) a += fabsf(__ldg(p.wk + (long long)(c_lo + j) * p.wk_C * p.kh * p.kw + i));
        tk[j] = p.fix_cb * a * 1.0001f;  // the float sum of |k| may round low by < 1e-4 relative
    }
    unsigned* flist = fix ? p.fix_list + (long long)blockIdx.x * p.fix_cap : nullptr;
    const long long plane = (long long)p.out.H * p.out.W;  // NCHW channel stride
    const long long qstride = (long long)p.out.W * 4;      // blocked quad stride (floats)
    int it = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
        const int buf = it & 1;
        mbar_wait_sleep(&tfull[buf], (it >> 1) & 1);
        tc_fence_after();
        if (q == 0 && hsel == 0 && lane == 0) CT_TRACE(it, 5);
        int b, y0, x0;
        ct_tile(p, t, b, y0, x0);
        const int x = x0 + L;
        const bool xok = L < p.Wt && x < p.OW;
        const uint32_t tcol = tq + (uint32_t)(buf * bufcols + (p.HR - 1) * SW);  // slot of row 0; row r at -r*SW
        float* ob = p.out.p + (long long)b * p.out.bstride;
        for (int r = 0; r < (p.dbg & 2 ? 0 : p.R); r += POOL ? 2 : 1) {
            float v0[NH], v1[NH];
            tmem_ldn<NH>(tcol - r * SW, v0);
            if (POOL) tmem_ldn<NH>(tcol - (r + 1) * SW, v1);
            if (p.stack) {  // fold the a_hi.b_lo half of each slot
                float w0[NH], w1[NH];
                tmem_ldn<NH>(tcol - r * SW + NK, w0);
                if (POOL) tmem_ldn<NH>(tcol - (r + 1) * SW + NK, w1);
#pragma unroll
                for (int j = 0; j < NH; ++j) {
                    v0[j] += w0[j];
                    if (POOL) v1[j] += w1[j];
                }
            }
            const int y = y0 + r;
#pragma unroll
            for (int j = 0; j < NH; ++j) {  // pre-activations Z = chain + bias (layers.hpp:138-146)
                v0[j] += bias_r[j];
                if (POOL) v1[j] += bias_r[j];
            }
            if (!POOL) {
#pragma unroll
                for (int j = 0; j < NH; ++j) v0[j] = apply_act(ACT, v0[j]);
            }
            if (POOL) {
                const bool writer = xok && y + 1 < p.OH && (lane & 1) == 0;
                const int py = y >> 1, px = x >> 1;
                float* orow = BLOCKED ? ob + (long long)py * Kq * qstride + (long long)px * 4 : ob + (long long)py * p.out.W + px;
                uint8_t* crow = p.codes + (long long)b * p.codes_bstride + (((long long)py * Kq) * p.codes_pw + px) * 4;
                float xm = 0.0f;
                if (fix) {
                    const float* xr = xmr + (it & 7) * 4;
                    xm = fmaxf(fmaxf(xr[0], xr[1]), fmaxf(xr[2], xr[3]));
                }
#pragma unroll
                for (int g = 0; g < NQ; ++g) {
                    float o[4];
                    uint32_t cw = 0;
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        const int j = 4 * g + jj;
                        // window order (0,0) (0,1) (1,0) (1,1) (layers.hpp:228-232)
                        const float z[4] = {v0[j], __shfl_xor_sync(0xffffffffu, v0[j], 1), v1[j],
                                            __shfl_xor_sync(0xffffffffu, v1[j], 1)};
                        float a[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) a[i] = apply_act(ACT, z[i]);
                        float best = a[0], zb = z[0];
                        uint32_t code = 0;
#pragma unroll
                        for (int i = 1; i < 4; ++i)
                            if (a[i] > best) best = a[i], zb = z[i], code = (uint32_t)i;
                        o[jj] = best;
                        cw |= code << (8 * jj);
                        if (kFix && fix) {
                            // is the decision (and, for relu, the routed value's sign) certain within tau?
                            const float tau = tk[j] * xm;
                            bool doubt = false;
                            if (ACT == ACT_RELU) {
                                const float tw = tau + fabsf(zb) * 2.4e-7f;
                                const float lo_w = fmaxf(zb - tw, 0.0f), hi_w = fmaxf(zb + tw, 0.0f);
                                doubt = lo_w == 0.0f && hi_w > 0.0f;
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    const float hi = fmaxf(z[i] + tau + fabsf(z[i]) * 2.4e-7f, 0.0f);
                                    if ((uint32_t)i < code ? hi >= lo_w : ((uint32_t)i > code && hi > lo_w)) doubt = true;
                                }
                            } else {
                                // sigmoid: |da| <= |dz| / 4 + a few ulps of the two implementations' expf
                                const float sc = ACT == ACT_SIGMOID ? 0.25f : 1.0f;
                                const float lo_w = best - (sc * tau + fabsf(best) * 4.8e-7f);
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    const float hi = a[i] + sc * tau + fabsf(a[i]) * 4.8e-7f;
                                    if ((uint32_t)i < code ? hi >= lo_w : ((uint32_t)i > code && hi > lo_w)) doubt = true;
                                }
                            }
                            doubt = (doubt || (p.dbg & 8)) && writer && c_lo + j < p.N;
                            const unsigned m = __ballot_sync(0xffffffffu, doubt);
                            if (m) {
                                const int leader = __ffs(m) - 1;
                                unsigned base = 0;
                                if (lane == leader) base = atomicAdd(fixcnt, (unsigned)__popc(m));
                                base = __shfl_sync(0xffffffffu, base, leader);
                                if (doubt)
                                    flist[base + __popc(m & ((1u << lane) - 1u))] =
                                        (((unsigned)it * p.R + r) * p.Wt + L) * NK + c_lo + j;
                            }
                        }
                    }
                    const int gq = (c_lo >> 2) + g;
                    if (writer && gq < Kq) {
                        if (BLOCKED) {
                            *reinterpret_cast<float4*>(orow + gq * qstride) = make_float4(o[0], o[1], o[2], o[3]);
                        } else {
#pragma unroll
                            for (int jj = 0; jj < 4; ++jj)
                                if (4 * gq + jj < p.out.C) orow[(4 * gq + jj) * plane] = o[jj];
                        }
                        *reinterpret_cast<uint32_t*>(crow + (long long)gq * p.codes_pw * 4) = cw;
                    }
                }
            } else if (xok && y < p.OH) {
                float* orow = BLOCKED ? ob + (long long)y * Kq * qstride + (long long)x * 4 : ob + (long long)y * p.out.W + x;
#pragma unroll
                for (int g = 0; g < NQ; ++g) {
                    const int gq = (c_lo >> 2) + g;
                    if (gq >= Kq) break;
                    if (BLOCKED) {
                        *reinterpret_cast<float4*>(orow + gq * qstride) =
                            make_float4(v0[4 * g], v0[4 * g + 1], v0[4 * g + 2], v0[4 * g + 3]);
                    } else {
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj)
                            if (4 * gq + jj < p.out.C) orow[(4 * gq + jj) * plane] = v0[4 * g + jj];
                    }
                }
            }
        }
        if (!(p.dbg & 2)) zero_rows(buf);
        tc_fence_before();
        if (q == 0 && hsel == 0 && lane == 0) CT_TRACE(it, 6);
        mbar_arrive(&tempty[buf]);
    }
}

// the K steps of one halo row, unrolled: KW taps x GP quad pairs (GP = 0: one quad, tap pairs)
template <int KW, int GP, bool X3>
__device__ __forceinline__ void ct_mma_row(uint32_t tacc, uint64_t a_row, uint64_t b_base, uint64_t b_step,
                                           uint64_t two_p, uint64_t a_lo_add, uint64_t b_lo_add, uint32_t idesc,
                                           bool stk) {
    constexpr int NS = GP ? KW * GP : (KW + 1) / 2;
#pragma unroll
    for (int ks = 0; ks < NS; ++ks) {
        const uint64_t dah = a_row + (GP ? (uint64_t)(ks / GP) + (uint64_t)(ks % GP) * two_p : (uint64_t)(2 * ks));
        const uint64_t dbh = b_base + (uint64_t)ks * b_step;
        if (X3 && stk) {  // B1 = [hi | lo], B2 = [hi | 0] per filter row: a_hi.B1 + a_lo.B2
            mma_tf32_elect(tacc, dah, dbh, idesc);
            mma_tf32_elect(tacc, dah + a_lo_add, dbh + b_lo_add, idesc);
            continue;
        }
        if (X3) {
            mma_tf32_elect(tacc, dah + a_lo_add, dbh, idesc);
            mma_tf32_elect(tacc, dah, dbh + b_lo_add, idesc);
        }
        mma_tf32_elect(tacc, dah, dbh, idesc);
    }
}

// One pooling window of the forward recomputed exactly as the reference does (ct_epilogue's fix list):
// Z = fl(fma chain over (c, di, dj) in that order from 0) + bias (conv.hpp:62-119 / :215-273,
// layers.hpp:138-146; zero padding contributes exact zeros), the activation, then the first-index 2x2
// max (layers.hpp:228-232). Rewrites the pooled value and the code byte. Item = ((it*R + r)*Wt + L)*NK + k.
__device__ __forceinline__ void ct_fix_window(const ConvTParams& p, unsigned item, int NK) {
    const int k = (int)(item % (unsigned)NK);
    unsigned rest = item / (unsigned)NK;
    const int L = (int)(rest % (unsigned)p.Wt);
    rest /= (unsigned)p.Wt;
    const int r = (int)(rest % (unsigned)p.R);
    const int it = (int)(rest / (unsigned)p.R);
    int b, y0, x0;
    ct_tile(p, (int)blockIdx.x + it * (int)gridDim.x, b, y0, x0);
    const int Y = y0 + r, X = x0 + L;  // window origin (even, even)
    const int C = p.wk_C, KH = p.kh, KW = p.kw;
    const float* wk = p.wk + (long long)k * C * KH * KW;
    const float* xb = p.x + (long long)b * p.x_bstride;
    const float bias = __ldg(p.bias + k);
    float a[4];
#pragma unroll 1
    for (int w = 0; w < 4; ++w) {
        const int y = Y + (w >> 1), x = X + (w & 1);
        float acc = 0.0f;
        for (int c = 0; c < C; ++c)
            for (int di = 0; di < KH; ++di) {
                const int iy = y + di - p.pad;
                for (int dj = 0; dj < KW; ++dj) {
                    const int ix = x + dj - p.pad;
                    if ((unsigned)iy < (unsigned)p.Hin && (unsigned)ix < (unsigned)p.Win)
                        acc = fmaf(__ldg(wk + (c * KH + di) * KW + dj),
                                   __ldg(xb + (((long long)iy * p.G + (c >> 2)) * p.Win + ix) * 4 + (c & 3)), acc);
                }
            }
        a[w] = apply_act(p.act, acc + bias);
    }
    float best = a[0];
    int code = 0;
    for (int i = 1; i < 4; ++i)
        if (a[i] > best) best = a[i], code = i;
    const int py = Y >> 1, px = X >> 1, Kq = (p.out.C + 3) >> 2;
    float* ob = p.out.p + (long long)b * p.out.bstride;
    if (p.out.blocked)
        ob[(((long long)py * Kq + (k >> 2)) * p.out.W + px) * 4 + (k & 3)] = best;
    else
        ob[((long long)k * p.out.H + py) * p.out.W + px] = best;
    p.codes[(long long)b * p.codes_bstride + (((long long)py * Kq + (k >> 2)) * p.codes_pw + px) * 4 + (k & 3)] =
        (uint8_t)code;
}

// Correlation over row-blocked halo tiles on the tensor cores (3xTF32: a.b = ah.bh + ah.bl + al.bh with
// the hardware's tf32 truncation making the raw value the hi part, fp32 accumulate, ~1e-7 relative). Per tile (R output rows x Wt columns) and per halo row
// h, each MMA reads the halo row ONCE and multiplies it with all kh filter rows stacked along N
// (N = kh * NK). Output row r's accumulator lives in TMEM row slot (HR - 1 - r), so the MMA of halo row h
// lands its kh products on rows h, h-1, .., h-kh+1 -- exactly the rows that need them. Slots are zeroed
// by the epilogue after it drains them, so every MMA accumulates.
//   warp 0      : FWD halo producer (bulk copies + edge zeros) | DGRAD dP/P/codes staging (TMA)
//   warp 1      : TMEM allocation + MMA issue (warp-converged, elect.sync)
//   warps 2..9  : epilogue (two warps per TMEM lane quadrant, half the channels each)
//   warps 10..  : FWD lo split of the landed halo | DGRAD dZ expansion into hi / lo halo planes
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
    uint64_t* dtab = zempty + 2;  // per K step: A descriptor (halo row 0, stage 0), B descriptor
    float* xmr = reinterpret_cast<float*>(dtab + 2 * p.ksteps);  // [8 tiles][4 producer warps] max|x| of a halo
    unsigned* fixcnt = reinterpret_cast<unsigned*>(xmr + 32);     // items in this CTA's fix list
    uint8_t* zst = reinterpret_cast<uint8_t*>(xmr + 64);  // 2 staging slots (DGRAD)
    zst = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(zst) + 127) & ~uintptr_t(127));

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = p.stages;
    const int bufcols = p.slots * (p.stack ? 2 * NK : NK);
    // one CTA per SM (shared memory): it takes all of TMEM, whose base is then column 0 -- a compile-time
    // constant, so the MMA warp's accumulator addresses stay in uniform registers
    constexpr uint32_t tcols = 512;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], MODE == CT_DGRAD ? 32 * Roles::kProdWarps : 1);
            mbar_init(&ready[s], 32 * Roles::kProdWarps);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 256);
            mbar_init(&zfull[a], 1);
            mbar_init(&zempty[a], 32 * Roles::kProdWarps);
        }
        *fixcnt = 0u;
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tslot, tcols);
    // zero the halo buffers once: the slack behind them is read by MMA rows past the tile width
    for (int i = threadIdx.x; i < S * p.stage_bytes / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0u, 0u, 0u, 0u);
    pdl_wait();  // weights and inputs are written by earlier kernels of the step
    {  // weights, K-major no-swizzle: [kstep][kc][n][4] with n = di*NK + k, or (stacked) di*2NK + part*NK + k:
        // array 1 = hi | lo, array 2 = hi | 0 (the lo part of array 1 takes the place of array 2's zeros)
        const int SWb = p.stack ? 2 * NK : NK;
        const int NN = p.kh * SWb;
        const int total = p.ksteps * 2 * NN * 4;
        for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
            const int j = idx & 3, n = (idx >> 2) % NN, kc = (idx / (4 * NN)) & 1, s = idx / (8 * NN);
            const int di = n / SWb, part = (n - di * SWb) / NK, nn = n - di * SWb - part * NK;
            int cin, dj;
            float v = 0.0f;
            if (ct_kdecode(p, s, kc, j, cin, dj) && nn < p.N) {
                if (MODE == CT_FWD) {
                    if (cin < p.wk_C) v = __ldg(p.wk + (((long long)nn * p.wk_C + cin) * p.kh + di) * p.kw + dj);
                } else if (cin < p.wk_K) {  // flipped, transposed: Wf[n=c][k][di][dj] = W[k][c][kh-1-di][kw-1-dj]
                    v = __ldg(p.wk + (((long long)cin * p.wk_C + nn) * p.kh + (p.kh - 1 - di)) * p.kw + (p.kw - 1 - dj));
                }
            }
            const int off = s * (2 * NN * 16) + kc * (NN * 16) + n * 16 + j * 4;
            if (p.stack) {
                *reinterpret_cast<float*>(wsm + off) = part ? split_lo1(v) : v;
                *reinterpret_cast<float*>(wsm + p.w_bytes + off) = part ? 0.0f : v;
            } else {
                *reinterpret_cast<float*>(wsm + off) = v;
                *reinterpret_cast<float*>(wsm + p.w_bytes + off) = split_lo1(v);
            }
        }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (*tslot != 0u) __trap();  // the MMA issue below assumes TMEM base column 0
    constexpr uint32_t tmem_base = 0u;

    if (warp == 0) {
        if (MODE == CT_FWD) {  // ---------------- halo producer (bulk copies + edge zeros)
            int it = 0;
            for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
                const int s = it % S;
                mbar_wait_sleep(&empty[s], ((it / S) & 1) ^ 1);
                if (lane == 0) CT_TRACE(it, 0);
                int b, y0, x0;
                ct_tile(p, t, b, y0, x0);
                if (p.dbg & 4) {
                    if (lane == 0) mbar_arrive(&full[s]);
                } else {
                    halo_load_warp(p.x, p.x_bstride, p.G, p.Hin, p.Win, b, y0 - p.pad, x0 - p.pad, p.HR, p.P,
                                   smem + s * p.stage_bytes, &full[s], lane);
                }
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
    } else if (warp == 1) {  // ---------------- MMA issue (whole warp, elected lane)
        // descriptor arithmetic only touches the 14-bit start-address field (smem < 256 KB)
        const int SWm = p.stack ? 2 * NK : NK;
        const uint32_t idesc = umma_idesc_tf32(128, p.kh * SWm, 0, 0);
        const uint64_t a_lo_add = (uint64_t)(p.h_bytes >> 4), b_lo_add = (uint64_t)(p.w_bytes >> 4);
        const uint64_t row_add = (uint64_t)((p.G * p.P * 16) >> 4);
        const uint64_t a_base = desc_none(smem_u32(smem), p.G >= 2 ? (uint32_t)p.P * 16 : 16u);
        const uint64_t b_base = desc_none(smem_u32(wsm), (uint32_t)(p.kh * SWm * 16));
        const uint64_t b_step = (uint64_t)((2 * p.kh * SWm * 16) >> 4);
        int it = 0;
        for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
            const int s = it % S, buf = it & 1;
            mbar_wait(&tempty[buf], (it >> 1) & 1);  // slots drained and re-zeroed
            mbar_wait(MODE == CT_FWD ? &ready[s] : &full[s], (it / S) & 1);
            tc_fence_after();
            if (lane == 0) CT_TRACE(it, 3);
            // descriptors by running adds on the start-address field (no per-MMA memory loads):
            // K step (dj, quad pair gp) starts at (2*gp*P + dj) * 16 bytes into the halo row, or at
            // 2*s*16 for a single quad (tap pairs); its weights at s * kh*NK*32 bytes
            uint64_t a_row = a_base + (uint64_t)((s * p.stage_bytes) >> 4);
            for (int h = 0; h < p.HR; ++h, a_row += row_add) {
                // halo row h feeds output rows h - di (di = 0..kh-1) = row slots HR-1-h .. HR-1-h+kh-1
                const uint32_t tacc = tmem_base + (uint32_t)(buf * bufcols + (p.HR - 1 - h) * SWm);
                uint64_t dbh = b_base;
                const uint64_t two_p = (uint64_t)(2 * p.P);
                // the common shapes run fully unrolled (independent descriptor adds interleave)
                if (p.kw == 3 && p.G == 4) {
                    ct_mma_row<3, 2, X3>(tacc, a_row, b_base, b_step, two_p, a_lo_add, b_lo_add, idesc, p.stack != 0);
                } else if (p.kw == 3 && p.G == 1) {
                    ct_mma_row<3, 0, X3>(tacc, a_row, b_base, b_step, two_p, a_lo_add, b_lo_add, idesc, p.stack != 0);
                } else if (p.kw == 5 && p.G == 1) {
                    ct_mma_row<5, 0, X3>(tacc, a_row, b_base, b_step, two_p, a_lo_add, b_lo_add, idesc, p.stack != 0);
                } else if (p.kw == 5 && (p.G == 3 || p.G == 4)) {
                    ct_mma_row<5, 2, X3>(tacc, a_row, b_base, b_step, two_p, a_lo_add, b_lo_add, idesc, p.stack != 0);
                } else if (p.kw == 5 && p.G == 2) {
                    ct_mma_row<5, 1, X3>(tacc, a_row, b_base, b_step, two_p, a_lo_add, b_lo_add, idesc, p.stack != 0);
                } else if (p.kw == 3 && p.G == 2) {
                    ct_mma_row<3, 1, X3>(tacc, a_row, b_base, b_step, two_p, a_lo_add, b_lo_add, idesc, p.stack != 0);
                } else if (p.G >= 2) {
                    const int GP = (p.G + 1) >> 1;
                    for (int dj = 0; dj < p.kw; ++dj) {
                        uint64_t dah = a_row + (uint64_t)dj;
                        for (int gp = 0; gp < GP; ++gp, dah += (uint64_t)(2 * p.P), dbh += b_step) {
                            if (X3 && p.stack) {
                                mma_tf32_elect(tacc, dah, dbh, idesc);
                                mma_tf32_elect(tacc, dah + a_lo_add, dbh + b_lo_add, idesc);
                                continue;
                            }
                            if (X3) {
                                mma_tf32_elect(tacc, dah + a_lo_add, dbh, idesc);
                                mma_tf32_elect(tacc, dah, dbh + b_lo_add, idesc);
                            }
                            mma_tf32_elect(tacc, dah, dbh, idesc);
                        }
                    }
                } else {
                    uint64_t dah = a_row;
                    for (int ks = 0; ks < p.ksteps; ++ks, dah += 2, dbh += b_step) {
                        if (X3 && p.stack) {
                            mma_tf32_elect(tacc, dah, dbh, idesc);
                            mma_tf32_elect(tacc, dah + a_lo_add, dbh + b_lo_add, idesc);
                            continue;
                        }
                        if (X3) {
                            mma_tf32_elect(tacc, dah + a_lo_add, dbh, idesc);
                            mma_tf32_elect(tacc, dah, dbh + b_lo_add, idesc);
                        }
                        mma_tf32_elect(tacc, dah, dbh, idesc);
                    }
                }
            }
            if (lane == 0) CT_TRACE(it, 4);
            mma_commit_elect(&empty[s]);
            mma_commit_elect(&tfull[buf]);
        }
        if (lane == 0) pdl_trigger();
    } else if (warp >= Roles::kProd0) {
        const int pt = threadIdx.x - 32 * Roles::kProd0;
        constexpr int NP = 32 * Roles::kProdWarps;
        const int chunks = p.HR * p.G * p.P;  // 16-byte quads of one halo
        int it = 0;
        for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
            const int s = it % S;
            uint8_t* hi = smem + s * p.stage_bytes;
            uint8_t* lo = hi + p.h_bytes;
            if (MODE == CT_FWD) {  // ---------------- lo = x - tf32(x) of the landed halo (the raw halo is hi)
                mbar_wait_sleep(&full[s], (it / S) & 1);
                if (pt == 0) CT_TRACE(it, 1);
                if (X3 && !(p.dbg & 1)) {
                    const float4* src = reinterpret_cast<const float4*>(hi);
                    float am = 0.0f;  // max|x| of the halo: bounds sum|k x| for the exact-decision test
                    for (int i = pt; i < chunks; i += NP) {
                        const float4 a = src[i];
                        am = fmaxf(am, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
                        reinterpret_cast<float4*>(lo)[i] =
                            make_float4(split_lo1(a.x), split_lo1(a.y), split_lo1(a.z), split_lo1(a.w));
                    }
                    if (p.fix_list) {
#pragma unroll
                        for (int o = 16; o; o >>= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
                        // ring of 8: the producer of tile it + 8 waits (through the stage / TMEM buffer
                        // barriers) for the epilogue of tile it + 2
                        if ((pt & 31) == 0) xmr[(it & 7) * 4 + (pt >> 5)] = am;
                    }
                }
                fence_proxy_async_smem();
                if (pt == 0) CT_TRACE(it, 2);
                mbar_arrive(&ready[s]);
            } else {  // ---------------- dZ halo expansion (hi + lo) from the staged pooled tile
                int b, y0, x0;
                ct_tile(p, t, b, y0, x0);
                const int Y0 = y0 - p.pad, X0 = x0 - p.pad;
                const int sy0 = p.z.pool ? Y0 >> 1 : Y0, sx0 = (p.z.pool ? X0 >> 1 : X0) & ~3;
                const int zs = it & 1;
                uint8_t* slot = zst + zs * p.zslot_bytes;
                if (p.z.tma) {
                    mbar_wait_sleep(&zfull[zs], (it >> 1) & 1);
                } else {
                    zs_load_sync(p.z, slot, b, sy0, sx0, pt, NP);
                    asm volatile("bar.sync 1, %0;" ::"r"(NP) : "memory");
                }
                mbar_wait_sleep(&empty[s], ((it / S) & 1) ^ 1);
                auto put = [&](int i, const float4& d) {
                    reinterpret_cast<float4*>(hi)[i] = d;
                    if (X3)
                        reinterpret_cast<float4*>(lo)[i] =
                            make_float4(split_lo1(d.x), split_lo1(d.y), split_lo1(d.z), split_lo1(d.w));
                };
                const int GP = p.G * p.P;
                if (p.z.pool) {  // by pooled row: both conv rows of a pooled cell from one read of it
                    const int pr0 = Y0 >> 1;  // floor (Y0 = -pad on the top tile)
                    const int prn = ((Y0 + p.HR - 1) >> 1) - pr0 + 1;
                    for (int rem = pt; rem < GP; rem += NP) {  // (quad, col) fixed per thread, walk the rows
                        const int q = rem / p.P, X = X0 + rem - q * p.P;
                        for (int a = 0; a < prn; ++a) {
                            const int Ye = 2 * (pr0 + a), r0 = Ye - Y0;  // halo rows r0 (may be -1), r0 + 1
                            float4 d0, d1;
                            zs_dz2(p.z, slot, sy0, sx0, q, Ye, X, d0, d1);
                            if (r0 >= 0) put(r0 * GP + rem, d0);
                            if (r0 + 1 < p.HR) put((r0 + 1) * GP + rem, d1);
                        }
                    }
                } else {
                    for (int i = pt; i < chunks; i += NP) {
                        const int row = i / GP, rem = i - row * GP;
                        const int q = rem / p.P, col = rem - q * p.P;
                        put(i, zs_dz(p.z, slot, sy0, sx0, q, Y0 + row, X0 + col));
                    }
                }
                fence_proxy_async_smem();
                mbar_arrive(&full[s]);
                if (p.z.tma)
                    mbar_arrive(&zempty[zs]);
                else
                    asm volatile("bar.sync 1, %0;" ::"r"(NP) : "memory");
            }
        }
    } else {  // ---------------- epilogue: warps 2..9, two per TMEM lane quadrant (warp % 4), half the channels each
        const int q = warp & 3;
        const int hsel = (warp - Roles::kEpi0) >> 2;
        if (MODE == CT_DGRAD) {
            ct_epilogue<NK, ACT_NONE, false, true, MODE>(p, tmem_base, bufcols, tfull, tempty, q, hsel, lane, xmr, fixcnt);
        } else {
            const int sel = (p.act == ACT_SIGMOID ? 2 : p.act == ACT_RELU ? 1 : 0) * 4 + (p.pool ? 2 : 0) +
                            (p.out.blocked ? 1 : 0);
            switch (sel) {
                case 3: ct_epilogue<NK, ACT_NONE, true, true, MODE>(p, tmem_base, bufcols, tfull, tempty, q, hsel, lane, xmr, fixcnt); break;
                case 2: ct_epilogue<NK, ACT_NONE, true, false, MODE>(p, tmem_base, bufcols, tfull, tempty, q, hsel, lane, xmr, fixcnt); break;
                case 7: ct_epilogue<NK, ACT_RELU, true, true, MODE>(p, tmem_base, bufcols, tfull, tempty, q, hsel, lane, xmr, fixcnt); break;
                case 6: ct_epilogue<NK, ACT_RELU, true, false, MODE>(p, tmem_base, bufcols, tfull, tempty, q, hsel, lane, xmr, fixcnt); break;
                case 11: ct_epilogue<NK, ACT_SIGMOID, true, true, MODE>(p, tmem_base, bufcols, tfull, tempty, q, hsel, lane, xmr, fixcnt); break;
                case 10: ct_epilogue<NK, ACT_SIGMOID, true, false, MODE>(p, tmem_base, bufcols, tfull, tempty, q, hsel, lane, xmr, fixcnt); break;
                case 1: ct_epilogue<NK, ACT_NONE, false, true, MODE>(p, tmem_base, bufcols, tfull, tempty, q, hsel, lane, xmr, fixcnt); break;
                case 0: ct_epilogue<NK, ACT_NONE, false, false, MODE>(p, tmem_base, bufcols, tfull, tempty, q, hsel, lane, xmr, fixcnt); break;
                case 5: ct_epilogue<NK, ACT_RELU, false, true, MODE>(p, tmem_base, bufcols, tfull, tempty, q, hsel, lane, xmr, fixcnt); break;
                case 4: ct_epilogue<NK, ACT_RELU, false, false, MODE>(p, tmem_base, bufcols, tfull, tempty, q, hsel, lane, xmr, fixcnt); break;
                case 9: ct_epilogue<NK, ACT_SIGMOID, false, true, MODE>(p, tmem_base, bufcols, tfull, tempty, q, hsel, lane, xmr, fixcnt); break;
                default: ct_epilogue<NK, ACT_SIGMOID, false, false, MODE>(p, tmem_base, bufcols, tfull, tempty, q, hsel, lane, xmr, fixcnt); break;
            }
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, tcols);
    }
    if (MODE == CT_FWD && p.fix_list) {  // the CTA's doubtful windows, recomputed in the reference's order
        const unsigned n = *fixcnt;
        const unsigned* fl = p.fix_list + (long long)blockIdx.x * p.fix_cap;
        for (unsigned i = threadIdx.x; i < n; i += blockDim.x) ct_fix_window(p, fl[i], NK);
    }
}

// ------------------------------------------------------------------ weight gradient (FFMA, exact fp32)
struct ConvTWParams {
    int B, Cp, G, H, W, kh, kw, pad, OH, OW;  // layer geometry (input H x W, Cp channels; conv output OH x OW)
    int K, Kp, C;                             // real kernels, padded, real channels
    int R, Wt, P, HR, tiles_x, tiles_y, ntiles;
    int halo_bytes, slot_bytes;               // X halo; one (halo | dZ staging) slot
    const float* x;                           // layer input, row-blocked
    long long x_bstride;
    DZSrc z;
    float* ws;  // per-CTA partials [cta][Kp*Cp*kh*kw + Kp]
    int ws_stride;
    int chunk;  // output columns per sliding-window run (enough runs per tile for every stream)
};

constexpr int kWgChunk = 16;  // output columns per sliding-window run
// kernels per thread of the weight-gradient kernel for a filter size (the thread count NT is a
// template parameter: 512 = one CTA per SM, 256 = two; 5x5 runs 256 threads, one CTA per SM)
template <int KH, int KW>
struct WgCfg {
    static constexpr int KG = KH * KW <= 9 ? 8 : 4;  // register accumulators
};

// Thread (stream st, channel c, kernel group kg) owns dW[KG*kg .. KG*kg+KG)[c][.][.] over the pixel runs
// of its stream: per output pixel KH loads of the X window (sliding along the row) + KG/4 float4 loads
// of dZ feed KG*KH*KW FMAs. Per tile the X halo and the pooled dP / P / codes arrive by bulk copy / TMA
// into a double-buffered slot (the next tile's loads fly while this one computes); dZ is expanded from
// the slot into smem, and the bias gradient (sum of dZ) is accumulated there, per thread in a fixed
// quad, reduced in fixed order at the end.
template <int KH, int KW, int NT>
__global__ void __launch_bounds__(NT, NT <= 256 && KH * KW <= 9 ? 2 : 1)
    convt_wgrad_kernel(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapZdP,
                       const __grid_constant__ CUtensorMap mapZP, const __grid_constant__ CUtensorMap mapZc,
                       const ConvTWParams p) {
    constexpr int KG = WgCfg<KH, KW>::KG, T = KH * KW;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* slots[2] = {smem, smem + p.slot_bytes};  // [X halo | dZ staging]
    const int hb = (p.halo_bytes + 127) & ~127;
    float* dz = reinterpret_cast<float*>(smem + 2 * p.slot_bytes);  // [R][Kq][Wt][4]
    const int Kq = p.Kp >> 2;
    const int dz_floats = p.R * p.Kp * p.Wt;
    uint64_t* full = reinterpret_cast<uint64_t*>(dz + dz_floats);
    float* red = reinterpret_cast<float*>(smem);  // CTA reduction scratch, reuses the slots after the tile loop

    const int ngrp = (p.Kp + KG - 1) / KG;  // kernel groups
    const int TPS = p.C * ngrp;
    const int streams = NT / TPS;
    const int st = threadIdx.x / TPS, w = threadIdx.x - st * TPS;
    const int c = w % p.C, kg = w / p.C;
    const bool active = st < streams;
    float acc[KG][T];
#pragma unroll
    for (int j = 0; j < KG; ++j)
#pragma unroll
        for (int i = 0; i < T; ++i) acc[j][i] = 0.0f;
    // bias: thread t always expands quad bq = t % Kq (fixed assignment -> deterministic order)
    const int bq = threadIdx.x % Kq;
    float4 bsum = make_float4(0.f, 0.f, 0.f, 0.f);

    if (threadIdx.x == 0) {  // two arrivals per fill: the dZ staging arm and the halo arm
        mbar_init(&full[0], p.z.tma ? 2 : 1);
        mbar_init(&full[1], p.z.tma ? 2 : 1);
        fence_barrier_init();
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
    auto issue = [&](int t, int sl) {  // warp 0: X halo (bulk copies) + dZ staging (TMA) on full[sl]
        int b, y0, x0;
        tile_of(t, b, y0, x0);
        const int lane = threadIdx.x & 31;
        if (lane == 0 && p.z.tma) {
            mbar_arrive_expect_tx(&full[sl], zs_tx_bytes(p.z));
            zs_issue(p.z, &mapZdP, &mapZP, &mapZc, slots[sl] + hb, &full[sl], b, p.z.pool ? y0 >> 1 : y0,
                     (p.z.pool ? x0 >> 1 : x0) & ~3);
        }
        halo_load_warp(p.x, p.x_bstride, p.G, p.H, p.W, b, y0 - p.pad, x0 - p.pad, p.HR, p.P, slots[sl], &full[sl],
                       lane);
    };
    if (threadIdx.x < 32 && (int)blockIdx.x < p.ntiles) issue(blockIdx.x, 0);
    const int npx = p.R * p.Wt;
    int it = 0;
    for (int t = blockIdx.x; t < p.ntiles; t += gridDim.x, ++it) {
        const int sl = it & 1;
        int b, y0, x0;
        tile_of(t, b, y0, x0);
        const int sy0 = p.z.pool ? y0 >> 1 : y0, sx0 = (p.z.pool ? x0 >> 1 : x0) & ~3;
        uint8_t* zslot = slots[sl] + hb;
        // the other slot was released by the previous tile's closing barrier: its next fill flies
        // during this whole tile (dZ expansion + FMAs)
        if (threadIdx.x < 32 && t + (int)gridDim.x < p.ntiles) issue(t + gridDim.x, sl ^ 1);
        mbar_wait(&full[sl], (it >> 1) & 1);
        if (!p.z.tma) {
            zs_load_sync(p.z, zslot, b, sy0, sx0, threadIdx.x, NT);
            __syncthreads();
        }
        if (threadIdx.x < (NT / Kq) * Kq && p.z.pool) {  // pooled: rows in pairs, one read per pooled cell
            const int step = NT / Kq;
            int a = (threadIdx.x / Kq) / p.Wt, xx = threadIdx.x / Kq - a * p.Wt;
            for (int pi = threadIdx.x / Kq; pi < npx / 2; pi += step) {
                float4 d0, d1;
                zs_dz2(p.z, zslot, sy0, sx0, bq, y0 + 2 * a, x0 + xx, d0, d1);
                reinterpret_cast<float4*>(dz)[(2 * a * Kq + bq) * p.Wt + xx] = d0;
                reinterpret_cast<float4*>(dz)[((2 * a + 1) * Kq + bq) * p.Wt + xx] = d1;
                bsum.x += d0.x + d1.x;
                bsum.y += d0.y + d1.y;
                bsum.z += d0.z + d1.z;
                bsum.w += d0.w + d1.w;
                for (xx += step; xx >= p.Wt; xx -= p.Wt) ++a;
            }
        } else if (threadIdx.x < (NT / Kq) * Kq) {
            const int step = NT / Kq;
            int r = (threadIdx.x / Kq) / p.Wt, xx = threadIdx.x / Kq - r * p.Wt;
            for (int pi = threadIdx.x / Kq; pi < npx; pi += step) {  // dZ of the tile, quad bq
                const int Y = y0 + r, X = x0 + xx;
                float4 d = make_float4(0.f, 0.f, 0.f, 0.f);
                if (Y < p.OH && X < p.OW) d = zs_dz(p.z, zslot, sy0, sx0, bq, Y, X);
                reinterpret_cast<float4*>(dz)[(r * Kq + bq) * p.Wt + xx] = d;
                bsum.x += d.x;
                bsum.y += d.y;
                bsum.z += d.z;
                bsum.w += d.w;
                for (xx += step; xx >= p.Wt; xx -= p.Wt) ++r;
            }
        }
        __syncthreads();  // dz ready
        if (active) {
            const float* hx = reinterpret_cast<const float*>(slots[sl]);
            const int cq = c >> 2, cj = c & 3;
            const int runs_per_row = (p.Wt + p.chunk - 1) / p.chunk;
            for (int u = st; u < p.R * runs_per_row; u += streams) {
                const int r = u / runs_per_row, xb = (u - r * runs_per_row) * p.chunk;
                const int xe = min(min(p.Wt, xb + p.chunk), p.OW - x0);
                if (y0 + r >= p.OH || xb >= xe) continue;
                float win[KH][KW];
                const float* hrow = hx + (((r * p.G + cq) * p.P + xb) * 4 + cj);
                const int rstride = p.G * p.P * 4;
#pragma unroll
                for (int di = 0; di < KH; ++di)
#pragma unroll
                    for (int dj = 0; dj < KW - 1; ++dj) win[di][dj + 1] = hrow[di * rstride + dj * 4];
                const float4* dzr = reinterpret_cast<const float4*>(dz) + (r * Kq + kg * (KG / 4)) * p.Wt;
                for (int xx = xb; xx < xe; ++xx) {
                    const float* hcol = hrow + (xx - xb + KW - 1) * 4;
#pragma unroll
                    for (int di = 0; di < KH; ++di) {
#pragma unroll
                        for (int dj = 0; dj < KW - 1; ++dj) win[di][dj] = win[di][dj + 1];
                        win[di][KW - 1] = hcol[di * rstride];
                    }
                    float dd[KG];
#pragma unroll
                    for (int g = 0; g < KG / 4; ++g) {
                        const float4 d4 = dzr[g * p.Wt + xx];
                        dd[4 * g] = d4.x, dd[4 * g + 1] = d4.y, dd[4 * g + 2] = d4.z, dd[4 * g + 3] = d4.w;
                    }
#pragma unroll
                    for (int j = 0; j < KG; ++j)
#pragma unroll
                        for (int di = 0; di < KH; ++di)
#pragma unroll
                            for (int dj = 0; dj < KW; ++dj)
                                acc[j][di * KW + dj] = fmaf(dd[j], win[di][dj], acc[j][di * KW + dj]);
                }
            }
        }
        __syncthreads();  // slot and dz consumed
    }
    pdl_trigger();
    // fixed-order reductions: streams of the CTA, bias over the threads of each quad; one row per CTA
    const int nval = KG * T;
    if (active)
        for (int j = 0; j < KG; ++j)
            for (int i = 0; i < T; ++i) red[((long long)st * TPS + w) * nval + j * T + i] = acc[j][i];
    float* bred = red + (long long)streams * TPS * nval;  // [NT][4]
    reinterpret_cast<float4*>(bred)[threadIdx.x] = bsum;
    __syncthreads();
    float* out = p.ws + (long long)blockIdx.x * p.ws_stride;
    const int nk = p.Kp * p.Cp * T;
    for (int idx = threadIdx.x; idx < nk + p.Kp; idx += NT) {
        float sum = 0.0f;
        if (idx < nk) {  // idx = ((k * Cp + c) * T + tap)
            const int k = idx / (p.Cp * T), rem = idx - k * (p.Cp * T), cc = rem / T, tap = rem - cc * T;
            if (cc < p.C && k / KG < ngrp) {
                const int ww = (k / KG) * p.C + cc, slotv = (k % KG) * T + tap;
                for (int q = 0; q < streams; ++q) sum += red[((long long)q * TPS + ww) * nval + slotv];
            }
        } else {  // bias of kernel k: threads with bq == k / 4, in thread order
            const int k = idx - nk, q4 = k >> 2, j = k & 3;
            for (int tt = q4; tt < (NT / Kq) * Kq; tt += Kq) sum += bred[tt * 4 + j];
        }
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
    // NCHW -> row-blocked quads. Vector path: a thread takes 4 consecutive pixels of one image row (one
    // float4 load per plane, a 4x4 transpose, 4 float4 stores); the CTA covers blockDim / (W / 4) rows
    // per iteration. Index math once per thread, not per element.
    pdl_wait();
    const int G = (C + 3) >> 2;
    const long long plane = (long long)H * W;
    const long long rows = (long long)B * H;
    const bool vec = (W & 3) == 0 && (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                     W / 4 <= (int)blockDim.x;
    if (vec) {
        const int w4 = W / 4, per = blockDim.x / w4;
        const int x4 = threadIdx.x % w4, sub = threadIdx.x / w4;
        if (sub >= per) return;
        for (long long row = (long long)blockIdx.x * per + sub; row < rows; row += (long long)gridDim.x * per) {
            const int b = (int)(row / H), y = (int)(row - (long long)b * H);
            const float* src = x + (long long)b * ld + (long long)y * W;
            float* dst = out + (long long)b * obstride + (long long)y * G * W * 4;
            for (int q = 0; q < G; ++q) {
                float4 v[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    v[j] = 4 * q + j < C ? __ldg(reinterpret_cast<const float4*>(src + (4 * q + j) * plane) + x4)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                float4* d = reinterpret_cast<float4*>(dst + ((long long)q * W + 4 * x4) * 4);
                d[0] = make_float4(v[0].x, v[1].x, v[2].x, v[3].x);
                d[1] = make_float4(v[0].y, v[1].y, v[2].y, v[3].y);
                d[2] = make_float4(v[0].z, v[1].z, v[2].z, v[3].z);
                d[3] = make_float4(v[0].w, v[1].w, v[2].w, v[3].w);
            }
        }
        return;
    }
    for (long long row = blockIdx.x; row < rows; row += gridDim.x) {
        const int b = (int)(row / H), y = (int)(row - (long long)b * H);
        const float* src = x + (long long)b * ld + (long long)y * W;
        float* dst = out + (long long)b * obstride + (long long)y * G * W * 4;
        for (int q = 0; q < G; ++q)
            for (int xx = threadIdx.x; xx < W; xx += blockDim.x) {
                float v[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) v[j] = 4 * q + j < C ? __ldg(src + (4 * q + j) * plane + xx) : 0.0f;
                *reinterpret_cast<float4*>(dst + ((long long)q * W + xx) * 4) = make_float4(v[0], v[1], v[2], v[3]);
            }
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
inline void ct_tile_shape(int B, int OH, int OW, int NK, int kh, int& R, int& Wt) {
    Wt = std::min(OW, 128);
    if (Wt & 1) ++Wt;
    // >= 512 output pixels per tile: halo rows are re-read (R + kh - 1) / R times
    R = (512 + Wt - 1) / Wt;
    R = std::max(2, (R + 1) & ~1);
    const int ohe = (OH + 1) & ~1;
    R = std::min(R, std::max(2, ohe));
    // two TMEM buffers of (R + 2(kh-1)) row slots of NK columns
    while (2 * (R + 2 * (kh - 1)) * NK > 512 && R > 2) R -= 2;
    // small maps: optionally shrink R until there are per_sm tiles per SM (B2N_CT_TILES_PER_SM). Off by
    // default: measured, the taller tiles win (MNIST / CIFAR conv1 dgrad 28.7 / 55.0 -> 24.7 / 48.8 us)
    // -- a tile's pipeline latency, not the SM count, bounds these small layers
    const long long tx = (OW + Wt - 1) / Wt;
    static const int per_sm = std::getenv("B2N_CT_TILES_PER_SM") ? std::atoi(std::getenv("B2N_CT_TILES_PER_SM")) : 0;
    while (R > 2 && (long long)B * tx * ((OH + R - 1) / R) < (long long)per_sm * sm_count()) R -= 2;
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
    std::shared_ptr<DevMem> fix;  // exact-decision item lists (convt_enable_fix)
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
    if (kh * L.nk > 256) throw Error(B2N_ESHAPE, "b200nn conv: kh x kernels exceeds one MMA (N <= 256)");
    if (2 * (2 + 2 * (kh - 1)) * L.nk > 512) throw Error(B2N_ESHAPE, "b200nn conv: accumulators exceed TMEM");
    // 3x3 / <= 16 kernels: B hi|lo interleaved along N (2 MMAs per K step, double-width row slots) when
    // a tile of >= 4 rows (or the whole map) still fits shared memory with the doubled weights
    p.stack = x3 && kh == 3 && L.nk <= 16 && !std::getenv("B2N_CT_NOSTACK");
    for (int attempt = 0; attempt < 2; ++attempt) {
    ct_tile_shape(B, p.OH, p.OW, p.stack ? 2 * L.nk : L.nk, kh, p.R, p.Wt);
    bool fits = true;
    for (;;) {  // the tallest tile whose 2 halo stages (hi + lo) fit next to the weights / staging
        const int P_ = p.Wt + kw - 1, HR_ = p.R + kh - 1, G_ = Cp / 4;
        const int hb = (HR_ * G_ * P_ * 16 + (kw + 129) * 16 + 127) & ~127;
        const int ks = G_ >= 2 ? kw * ((G_ + 1) / 2) : (kw + 1) / 2;
        int zb = 0;
        if (z) {
            DZSrc zz = *z;
            zz.bh = z->pool ? HR_ / 2 + 1 : HR_;
            zz.bw = ((z->pool ? P_ / 2 + 1 : P_) + 6) & ~3;
            zb = (zs_bytes(zz) + 127) & ~127;
        }
        const int need = 2 * (2 * hb) + 2 * (ks * 2 * kh * (p.stack ? 2 : 1) * L.nk * 16) + 1024 + 256 + ks * 16 + 384 + 2 * zb;
        if (need <= 227 * 1024) break;
        if (p.R <= 2) {
            fits = false;
            break;
        }
        p.R -= 2;
    }
    const int ohe = (p.OH + 1) & ~1;
    if (!p.stack || (fits && (p.R >= 4 || p.R >= ohe))) break;
    p.stack = 0;  // fall back to 3 MMAs per K step with single-width slots
    }
    p.P = p.Wt + kw - 1;
    p.HR = p.R + kh - 1;
    p.slots = p.HR + kh - 1;
    p.tiles_x = (p.OW + p.Wt - 1) / p.Wt;
    p.tiles_y = (p.OH + p.R - 1) / p.R;
    p.ntiles = B * p.tiles_x * p.tiles_y;
    p.ksteps = p.G >= 2 ? kw * ((p.G + 1) / 2) : (kw + 1) / 2;
    if (p.ksteps > kCtMaxKSteps) throw Error(B2N_ESHAPE, "b200nn conv: filter width x channel quads too large");
    p.halo_bytes = p.HR * p.G * p.P * 16;
    // MMA rows past the tile width read at most (kw + 128) * 16 bytes beyond the halo (ct_aoff)
    p.h_bytes = (p.halo_bytes + (kw + 129) * 16 + 127) & ~127;
    p.stage_bytes = 2 * p.h_bytes;
    p.w_bytes = p.ksteps * 2 * kh * (p.stack ? 2 : 1) * L.nk * 16;
    std::memset(L.zmaps, 0, sizeof(L.zmaps));
    if (z) {  // DGRAD: pooled window covering the dZ halo rows / cols of a tile
        p.z = *z;
        p.z.bh = z->pool ? p.HR / 2 + 1 : p.HR;
        p.z.bw = ((z->pool ? p.P / 2 + 1 : p.P) + 6) & ~3;  // window start is aligned down to 4 (TMA: 16 B)
        p.zslot_bytes = (zs_bytes(p.z) + 127) & ~127;
        dz_maps(p.z, B, L.zmaps);
    }
    const int fixed = 2 * p.w_bytes + 1024 + 256 + p.ksteps * 16 + 384 + 2 * p.zslot_bytes;
    const int budget = 227 * 1024;
    p.stages = std::min(4, (budget - fixed) / p.stage_bytes);
    if (p.stages < 2) throw Error(B2N_ESHAPE, "b200nn conv: halo tile does not fit shared memory");
    L.smem = p.stages * p.stage_bytes + fixed;
    L.grid = std::min(p.ntiles, sm_count());
    L.flops = 2.0 * B * p.OH * p.OW * N * (double)Cp * kh * kw;
    p.trace = TraceRegistry::get().next();
    if (const char* e = std::getenv("B2N_CT_DBG")) p.dbg = std::atoi(e);
    return L;
}

// Exact pooling decisions for a FWD + pool plan (3xTF32 only): one item list per CTA, sized for every
// window x channel of its tiles. The bound per chain term: the tf32 split drops <= 3 * 2^-20 |k x| per
// product; the tensor core's fp32 accumulation (products exact, sums aligned to the largest term and
// truncated: <= 9 ulps of it per 8-term MMA, up to 3 MMAs per K step) <= 7 n 2^-24 sum|k x|; the
// reference's sequential fma chain <= n 2^-24 sum|k x| (n = Cp * kh * kw terms).
inline void convt_enable_fix(ConvTLaunch& L, std::shared_ptr<DevMem>& mem) {
    ConvTParams& p = L.p;
    if (!L.x3 || !p.pool || L.mode != CT_FWD) return;
    const long long per_cta = (p.ntiles + L.grid - 1) / L.grid;
    p.fix_cap = per_cta * (p.R / 2) * ((p.Wt + 1) / 2) * L.nk;
    if (((long long)per_cta * p.R * p.Wt * L.nk) >> 32) throw Error(B2N_ESHAPE, "conv fix-up items exceed 32 bits");
    mem = std::make_shared<DevMem>();
    mem->alloc((size_t)L.grid * p.fix_cap * 4);
    p.fix_list = mem->as<unsigned>();
    const double n = (double)p.Cp * p.kh * p.kw;
    p.fix_cb = (float)(3.0 * std::ldexp(1.0, -20) + 8.0 * n * std::ldexp(1.0, -24));
    if (const char* e = std::getenv("B2N_CT_FIXSCALE")) p.fix_cb *= (float)std::atof(e);
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
    int grid = 1, smem = 0, nt = 512;  // nt: threads per CTA (256 -> two CTAs per SM)
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
    p.Wt = q.Wt;
    p.P = q.P;
    p.tiles_x = q.tiles_x;
    p.x = q.x;
    p.x_bstride = q.x_bstride;
    p.z = z0;
    p.z.bw = ((z0.pool ? q.Wt / 2 : q.Wt) + 6) & ~3;  // window start is aligned down to 4 (TMA: 16 B)
    if (!((p.kh == 3 && p.kw == 3) || (p.kh == 5 && p.kw == 5)))
        throw Error(B2N_EINTERNAL, "convt wgrad: only 3x3 and 5x5 filters are instantiated");
    const int T = p.kh * p.kw;
    const int KG = T <= 9 ? 8 : 4;  // WgCfg
    const int TPS = C * ((p.Kp + KG - 1) / KG);
    int NT = T <= 9 ? 512 : 256;
    if (TPS > NT) throw Error(B2N_ESHAPE, "convt wgrad: channels x kernel groups exceed one CTA");
    auto smem_for = [&](int R, int nt) {
        DZSrc zz = p.z;
        zz.bh = z0.pool ? R / 2 : R;
        const int halo = (R + p.kh - 1) * p.G * p.P * 16;
        const int slot = (((halo + 127) & ~127) + zs_bytes(zz) + 1023) & ~1023;
        const int red_bytes = (nt / TPS) * TPS * KG * T * 4 + nt * 16;
        return 1024 + std::max(2 * slot + R * p.Kp * p.Wt * 4 + 64, red_bytes);
    };
    // its own tile height: as many output rows as fit (compute per tile must hide the next tile's loads)
    auto rows_for = [&](int nt, int cap) {
        int R = std::min(std::max(2, (p.OH + 1) & ~1), 16);
        while (R > 2 && smem_for(R, nt) > cap) R -= 2;
        return R;
    };
    p.R = rows_for(NT, 200 * 1024);
    // 3x3 filters: two 256-thread CTAs per SM when a tile fits half the shared memory (B2N_CONVT_WG_R2MIN:
    // the least tile height taken, default 2; B2N_CONVT_WG_WIDE: always one 512-thread CTA) --
    // one CTA's per-tile barrier and dZ expansion overlap the other's FMAs
    if (T <= 9 && TPS <= 256 && !std::getenv("B2N_CONVT_WG_WIDE")) {
        const int R2 = rows_for(256, 112 * 1024);
        static const int r2min = std::getenv("B2N_CONVT_WG_R2MIN") ? std::atoi(std::getenv("B2N_CONVT_WG_R2MIN")) : 2;
        if (R2 >= r2min && smem_for(R2, 256) <= 112 * 1024) {
            NT = 256;
            p.R = R2;
        }
    }
    const int streams = NT / TPS;
    p.HR = p.R + p.kh - 1;
    p.tiles_y = (p.OH + p.R - 1) / p.R;
    p.ntiles = p.B * p.tiles_x * p.tiles_y;
    p.halo_bytes = p.HR * p.G * p.P * 16;
    p.z.bh = z0.pool ? p.R / 2 : p.R;
    p.chunk = std::max(2, std::min(kWgChunk, (p.R * p.Wt + streams - 1) / streams));
    p.ws_stride = (p.Kp * p.Cp * T + p.Kp + 3) & ~3;
    p.slot_bytes = (((p.halo_bytes + 127) & ~127) + zs_bytes(p.z) + 1023) & ~1023;
    L.map = f.map;
    dz_maps(p.z, p.B, L.zmaps);
    L.nt = NT;
    L.grid = std::min(p.ntiles, (NT <= 256 && T <= 9 ? 2 : 1) * sm_count());
    L.smem = smem_for(p.R, NT);
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
