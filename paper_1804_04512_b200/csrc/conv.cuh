// conv.cuh -- convolution layers as implicit-GEMM tcgen05 kernels (conv_forward / conv_backward,
// layers.hpp:132-193, conv.hpp:180-345) with the layer's activation and 2x2 max-pool fused.
//
// One persistent, warp-specialised kernel template, three modes:
//   FWD   : M = output pixels (ordered so the 4 pixels of each pooling window are 4 consecutive
//           rows / TMEM lanes), N = kernels, K = c*kh*kw. Epilogue: bias + act, 2x2 max with the
//           reference's first-index tie rule (layers.hpp:228-232) via lane shuffles, writes only the
//           pooled activation and a 1-byte argmax code -- the full-resolution conv output never
//           reaches HBM.
//   DGRAD : M = input pixels, N = input channels, K = kernels*kh*kw; the A operand is gathered from
//           dZ (pool_backward + activation_gradient), i.e. the padded-valid full conv
//           (conv.hpp:337-345) as an implicit GEMM. Skipped for the first layer (its dx is dead).
//   WGRAD : M = patch index (c,di,dj) plus a ones row (-> bias gradient), N = kernels, K = output
//           pixels split across CTAs; per-CTA partial tiles are reduced in fixed order by
//           conv_wgrad_reduce_kernel, which also applies the SGD-momentum step (deterministic).
// Roles (416 threads): warps 0-7 gather A (and per-block B) tiles into 128 B-swizzled smem with the
// 3xTF32 lo split (all loads of a thread issued before its 16 B smem stores), warp 8 allocates TMEM
// and issues tcgen05.mma, warps 9-12 drain a double-buffered TMEM accumulator through the epilogue.
// Backward first materialises dZ = unpool(dpool) * act' once (conv_dz_kernel) so the dgrad / wgrad
// gathers are single loads.
#pragma once
#include "runtime.cuh"

namespace b2n {

struct ConvGeom {
    int c = 1, h = 1, w = 1, k = 1, kh = 1, kw = 1, pad = 0, oh = 1, ow = 1;
};

enum ConvMode : int { CONV_FWD = 0, CONV_DGRAD = 1, CONV_WGRAD = 2 };

struct ConvParams {
    ConvGeom g;
    int B;           // local batch
    int act;         // activation following the conv
    int pool;        // 2x2 max-pool fused
    int ph, pw;      // pooled extents (== oh, ow without pool)
    // tensors (fp32, NCHW per image with the given per-image pitch)
    const float* x;  // layer input
    long long ldx;
    const float* wk;    // kernels (k, c, kh, kw) dense
    const float* bias;  // (k)
    float* y;           // pooled activation output
    long long ldy;
    uint8_t* arg;       // argmax codes, dense per image (k*ph*pw)
    const float* dy;    // gradient of the pooled output (D)
    long long lddy;
    float* dx;          // DGRAD output (previous layer's D)
    long long lddx;
    float* ws;          // WGRAD partials [item][128][32]
    const float* dz;    // DGRAD / WGRAD: unpooled pre-activation gradient [B][K][OH][OW]
    // work decomposition
    int items;       // total work items
    int kblocks;     // K blocks per item
    int ckk;         // c*kh*kw
    int kkk;         // k*kh*kw
    int mtiles_w;    // WGRAD: M' tiles
    int chunk_px;    // WGRAD: output pixels per item (multiple of 32)
    int chunks;      // WGRAD: pixel chunks
    long long npix;  // rows of the GEMM view (pixels)
    // convolutional-RBM epilogue extensions (crbm.cuh); zero for the network layers
    const double* u;       // FWD: Bernoulli uniforms [B][K][OH][OW] -> ys = (u < (double)y)
    float* ys;             // FWD: sampled hidden states, dense [B][K][OH][OW]
    int neg_out;           // FWD: store -y (the negative phase of the weight statistics)
    const float* dg_bias;  // DGRAD: dx = act(acc + dg_bias[c]) (crbm_visible_preact + unit mean)
    int dg_act;
    float* vstat_f;        // DGRAD: per (item, warp, channel) sum of (x - dx) (p.x = v0) ...
    double* vstat_d;       // ... and sum of (x - dx)^2 in double (sq_diff_per_row)
};

constexpr int kGatherWarps = 8;
constexpr int kConvThreads = 32 * (kGatherWarps + 1 + 4);  // gather | MMA | 4 epilogue warps = 416
constexpr int kConvStages = 4;

template <int NP, int MODE, bool X3>
struct ConvCfg {
    static constexpr int A_BYTES = 128 * 32 * 4;
    static constexpr int B_BYTES = MODE == CONV_WGRAD ? 32 * 32 * 4 : 0;  // per-stage B only for WGRAD
    static constexpr int STAGE_BYTES = (A_BYTES + B_BYTES) * (X3 ? 2 : 1);
    static constexpr int NPAD = MODE == CONV_WGRAD ? 32 : NP;
    static constexpr int TMEM_COLS = 2 * NPAD <= 32 ? 32 : 2 * NPAD <= 64 ? 64 : 128;
    static constexpr int KMAX = 320;                                    // c*kh*kw or k*kh*kw padded
    static constexpr int WB_BYTES = MODE == CONV_WGRAD ? 0 : NP * KMAX * 4 * (X3 ? 2 : 1);  // static B
    static constexpr int SMEM = kConvStages * STAGE_BYTES + WB_BYTES + KMAX * 8 + 1024 + 512;
};

__device__ __forceinline__ float split_lo1(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// K-major SW128 byte offset of (row, k) inside a 32-wide K block (16 B chunks XOR row%8)
__device__ __forceinline__ uint32_t kmaj_off(int row, int k) {
    return (row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 2) ^ (row & 7)) & 7) << 4) + (k & 3) * 4;
}
// MN-major SW128_BASE32B byte offset of (mn, k) in boxes of 32 MN x 32 K rows (32 B chunks XOR k%4)
__device__ __forceinline__ uint32_t mnmaj_off(int mn, int k) {
    return (mn >> 5) * 4096 + k * 128 + (((((mn & 31) >> 3) ^ (k & 3)) & 3) << 5) + (mn & 7) * 4;
}

__device__ __forceinline__ void sts4(uint8_t* base, uint32_t off, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(base) + off), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

__device__ __forceinline__ float act_grad(int act, float g, float y) {
    if (act == ACT_SIGMOID) return g * y * (1.0f - y);  // layers.hpp:294
    if (act == ACT_RELU) return y > 0.0f ? g : 0.0f;
    return g;
}

// decode a GEMM row of the FWD view into an output pixel; pool order puts a window on 4 rows
__device__ __forceinline__ bool fwd_pixel(const ConvParams& p, long long row, int& b, int& oy, int& ox) {
    b = oy = ox = 0;
    if (row >= p.npix) return false;
    if (p.pool) {
        const long long win = row >> 2;
        const int w = (int)(row & 3);
        const int per = p.ph * p.pw;
        b = (int)(win / per);
        const int rem = (int)(win - (long long)b * per);
        const int py = rem / p.pw;
        oy = 2 * py + (w >> 1);
        ox = 2 * (rem - py * p.pw) + (w & 1);
    } else {
        const int per = p.g.oh * p.g.ow;
        b = (int)(row / per);
        const int rem = (int)(row - (long long)b * per);
        oy = rem / p.g.ow;
        ox = rem - oy * p.g.ow;
    }
    return true;
}

template <int NP, int MODE, bool X3>
__global__ void __launch_bounds__(kConvThreads, 1) conv_tc_kernel(const ConvParams p) {
    using Cfg = ConvCfg<NP, MODE, X3>;
    constexpr int S = kConvStages;
    constexpr int NPAD = Cfg::NPAD;
    constexpr int MMA_WARP = kGatherWarps;
    constexpr int NG = 32 * kGatherWarps;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stages = smem;
    uint8_t* wb = smem + S * Cfg::STAGE_BYTES;  // static B (weights) hi | lo, K-major per 32-k block
    int2* ktab = reinterpret_cast<int2*>(wb + Cfg::WB_BYTES);  // per-k (offset, di<<16|dj)
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(ktab) + Cfg::KMAX * 8);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const ConvGeom& g = p.g;
    const int HW = g.h * g.w, OHW = g.oh * g.ow;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], NG);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 128);
        }
        fence_barrier_init();
    }
    if (warp == MMA_WARP) tmem_alloc(tslot, Cfg::TMEM_COLS);
    pdl_wait();  // weights / inputs below are written by earlier kernels of the step
    // per-k gather offsets: FWD/WGRAD patch index (c,di,dj) -> c*H*W + di*W + dj;
    // DGRAD (kk,di,dj) -> kk*OH*OW - di*OW - dj (relative to the (iy+pad, ix+pad) position of dZ)
    const int Kdim = MODE == CONV_DGRAD ? p.kkk : p.ckk;
    for (int k = threadIdx.x; k < Cfg::KMAX; k += blockDim.x) {
        int off = 0, didj = 0;
        if (k < Kdim) {
            const int khw = g.kh * g.kw;
            const int ch = k / khw, r = k % khw, di = r / g.kw, dj = r % g.kw;
            off = MODE == CONV_DGRAD ? ch * OHW - di * g.ow - dj : ch * HW + di * g.w + dj;
            didj = (di << 16) | dj;
        }
        ktab[k] = make_int2(off, didj);
    }
    if (MODE != CONV_WGRAD) {  // the static weight operand, K-major, hi and lo
        const int kb_total = (Kdim + 31) / 32;
        for (int idx = threadIdx.x; idx < NP * kb_total * 32; idx += blockDim.x) {
            const int n = idx / (kb_total * 32), k = idx % (kb_total * 32);
            float v = 0.0f;
            if (k < Kdim && n < (MODE == CONV_FWD ? g.k : g.c)) {
                if (MODE == CONV_FWD) {
                    v = p.wk[(long long)n * p.ckk + k];
                } else {  // Wt[n=c][k=(kk,di,dj)] = W[kk][c][di][dj]
                    const int khw = g.kh * g.kw, kk = k / khw, r = k % khw;
                    v = p.wk[((long long)kk * g.c + n) * khw + r];
                }
            }
            uint8_t* blk = wb + (k >> 5) * (NP * 128);
            *reinterpret_cast<float*>(blk + kmaj_off(n, k & 31)) = v;
            if (X3) *reinterpret_cast<float*>(blk + Cfg::WB_BYTES / 2 + kmaj_off(n, k & 31)) = split_lo1(v);
        }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tslot;

    if (warp < kGatherWarps) {
        // ===================== gather producers (256 threads): loads first, then 16 B smem stores
        const int t = threadIdx.x;
        int it = 0;
        for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
            // per-item row decode (FWD / DGRAD: one GEMM row per thread pair)
            const int r = t & 127, half = t >> 7;
            int b = 0, oy = 0, ox = 0;
            bool ok = false;
            const float* base = p.x;
            if (MODE == CONV_FWD) {
                ok = fwd_pixel(p, (long long)item * 128 + r, b, oy, ox);
                base = p.x + (long long)b * p.ldx + (long long)(oy - g.pad) * g.w + (ox - g.pad);
            } else if (MODE == CONV_DGRAD) {
                const long long row = (long long)item * 128 + r;
                ok = row < p.npix;
                if (ok) {
                    b = (int)(row / HW);
                    const int rem = (int)(row - (long long)b * HW);
                    oy = rem / g.w;  // (iy, ix) of the input pixel
                    ox = rem - oy * g.w;
                }
                base = p.dz + (long long)b * g.k * OHW + (long long)(oy + g.pad) * g.ow + (ox + g.pad);
            }
            for (int kb = 0; kb < p.kblocks; ++kb, ++it) {
                const int s = it % S;
                mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
                uint8_t* a = stages + s * Cfg::STAGE_BYTES;
                uint8_t* alo = a + Cfg::A_BYTES + Cfg::B_BYTES;
                if (MODE == CONV_FWD || MODE == CONV_DGRAD) {
                    float v[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int k = kb * 32 + half * 16 + i;
                        const int2 e = ktab[k];
                        const int di = e.y >> 16, dj = e.y & 0xFFFF;
                        bool in = ok && k < Kdim;
                        if (MODE == CONV_FWD) {
                            if (g.pad) in = in && (unsigned)(oy - g.pad + di) < (unsigned)g.h &&
                                           (unsigned)(ox - g.pad + dj) < (unsigned)g.w;
                        } else {
                            in = in && (unsigned)(oy + g.pad - di) < (unsigned)g.oh &&
                                 (unsigned)(ox + g.pad - dj) < (unsigned)g.ow;
                        }
                        v[i] = in ? __ldg(base + e.x) : 0.0f;
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t o = kmaj_off(r, half * 16 + 4 * j);
                        sts4(a, o, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                        if (X3)
                            sts4(alo, o, split_lo1(v[4 * j]), split_lo1(v[4 * j + 1]), split_lo1(v[4 * j + 2]),
                                 split_lo1(v[4 * j + 3]));
                    }
                } else {  // WGRAD: A'[K'=pixel][M'=patch], B'[K'=pixel][N'=kernel], MN-major
                    const int mt = item / p.chunks, ch = item % p.chunks;
                    const int kp = t & 31, grp = t >> 5;
                    const long long px = (long long)ch * p.chunk_px + kb * 32 + kp;
                    const bool pok = px < p.npix && kb * 32 + kp < p.chunk_px;
                    int pb = 0, py = 0, pxx = 0;
                    if (pok) {
                        pb = (int)(px / OHW);
                        const int rem = (int)(px - (long long)pb * OHW);
                        py = rem / g.ow;
                        pxx = rem - py * g.ow;
                    }
                    const float* xb = p.x + (long long)pb * p.ldx + (long long)(py - g.pad) * g.w + (pxx - g.pad);
                    float v[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int j = mt * 128 + grp * 16 + i;
                        float val = 0.0f;
                        if (pok) {
                            if (j < p.ckk) {
                                const int2 e = ktab[j];
                                const int di = e.y >> 16, dj = e.y & 0xFFFF;
                                const bool in = !g.pad || ((unsigned)(py - g.pad + di) < (unsigned)g.h &&
                                                          (unsigned)(pxx - g.pad + dj) < (unsigned)g.w);
                                if (in) val = __ldg(xb + e.x);
                            } else if (j == p.ckk) {
                                val = 1.0f;  // ones row: its product with dZ is the bias gradient
                            }
                        }
                        v[i] = val;
                    }
                    const float* dzp = p.dz + (long long)pb * g.k * OHW + (long long)py * g.ow + pxx;
                    float d[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int n = grp * 4 + i;
                        d[i] = (pok && n < g.k) ? __ldg(dzp + (long long)n * OHW) : 0.0f;
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t o = mnmaj_off(grp * 16 + 4 * j, kp);
                        sts4(a, o, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                        if (X3)
                            sts4(alo, o, split_lo1(v[4 * j]), split_lo1(v[4 * j + 1]), split_lo1(v[4 * j + 2]),
                                 split_lo1(v[4 * j + 3]));
                    }
                    const uint32_t ob = Cfg::A_BYTES + mnmaj_off(grp * 4, kp);
                    sts4(a, ob, d[0], d[1], d[2], d[3]);
                    if (X3) sts4(alo, ob, split_lo1(d[0]), split_lo1(d[1]), split_lo1(d[2]), split_lo1(d[3]));
                }
                fence_proxy_async_smem();
                mbar_arrive(&full[s]);
            }
        }
    } else if (warp == MMA_WARP) {
        // ===================== MMA issuer
        if (lane == 0) {
            const uint32_t idesc =
                MODE == CONV_WGRAD ? umma_idesc_tf32(128, NPAD, 1, 1) : umma_idesc_tf32(128, NPAD, 0, 0);
            const uint32_t wb_hi = smem_u32(wb), wb_lo = wb_hi + Cfg::WB_BYTES / 2;
            int it = 0, ai = 0;
            for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++ai) {
                const int acc = ai & 1;
                mbar_wait(&tempty[acc], ((ai >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t tacc = tmem_base + acc * NPAD;
                for (int kb = 0; kb < p.kblocks; ++kb, ++it) {
                    const int s = it % S;
                    mbar_wait(&full[s], (it / S) & 1);
                    tc_fence_after();
                    const uint32_t a_hi = smem_u32(stages + s * Cfg::STAGE_BYTES);
                    const uint32_t a_lo = a_hi + Cfg::A_BYTES + Cfg::B_BYTES;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        uint64_t dah, dal, dbh, dbl;
                        if (MODE == CONV_WGRAD) {
                            dah = desc_mnmajor(a_hi, kk);
                            dal = desc_mnmajor(a_lo, kk);
                            dbh = desc_mnmajor(a_hi + Cfg::A_BYTES, kk);
                            dbl = desc_mnmajor(a_lo + Cfg::A_BYTES, kk);
                        } else {
                            dah = desc_kmajor(a_hi, kk);
                            dal = desc_kmajor(a_lo, kk);
                            dbh = desc_kmajor(wb_hi + kb * (NP * 128), kk);
                            dbl = desc_kmajor(wb_lo + kb * (NP * 128), kk);
                        }
                        const uint32_t accum = (kb | kk) != 0;
                        if (X3) {
                            mma_tf32(tacc, dal, dbh, idesc, accum);
                            mma_tf32(tacc, dah, dbl, idesc, 1);
                            mma_tf32(tacc, dah, dbh, idesc, 1);
                        } else {
                            mma_tf32(tacc, dah, dbh, idesc, accum);
                        }
                    }
                    mma_commit(&empty[s]);
                }
                mma_commit(&tfull[acc]);
            }
            pdl_trigger();  // all MMAs issued: the next kernel may launch
        }
    } else {
        // ===================== epilogue (4 warps -> TMEM quadrants warp%4)
        const int q = warp & 3;
        const int r = 32 * q + lane;
        int ai = 0;
        for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++ai) {
            const int acc = ai & 1;
            mbar_wait(&tfull[acc], (ai >> 1) & 1);
            tc_fence_after();
            float v[NPAD];
            const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + acc * NPAD;
            if (NPAD == 8) {
                float t8[8];
                tmem_ld8(taddr, t8);
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = t8[i];
            } else {
#pragma unroll
                for (int c0 = 0; c0 < NPAD; c0 += 16) {
                    float t16[16];
                    tmem_ld16(taddr + c0, t16);
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[c0 + i] = t16[i];
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty[acc]);  // accumulator drained into registers
            if (MODE == CONV_FWD) {
                const long long row = (long long)item * 128 + r;
                int b = 0, oy = 0, ox = 0;
                const bool ok = fwd_pixel(p, row, b, oy, ox);
#pragma unroll
                for (int n = 0; n < NPAD; ++n) {
                    float val = n < g.k ? apply_act(p.act, v[n] + p.bias[n]) : 0.0f;  // layers.hpp:138-146 + act
                    if (p.pool) {
                        // 2x2 max over lanes r..r+3 (window order = row-major (dy,dx)); first max wins
                        int code = r & 3;
                        float bv = ok ? val : -INFINITY;
#pragma unroll
                        for (int o = 1; o <= 2; o <<= 1) {
                            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
                            const int oc = __shfl_xor_sync(0xffffffffu, code, o);
                            if (ov > bv || (ov == bv && oc < code)) {
                                bv = ov;
                                code = oc;
                            }
                        }
                        if (ok && (r & 3) == 0 && n < g.k) {
                            const long long pi = ((long long)n * p.ph + (oy >> 1)) * p.pw + (ox >> 1);
                            p.y[(long long)b * p.ldy + pi] = bv;
                            p.arg[(long long)b * g.k * p.ph * p.pw + pi] = (uint8_t)code;
                        }
                    } else if (ok && n < g.k) {
                        p.y[(long long)b * p.ldy + ((long long)n * g.oh + oy) * g.ow + ox] = p.neg_out ? -val : val;
                        if (p.u) {  // unit_sample_inplace (energy.hpp:59-61) on the supplied draw
                            const long long ui = (((long long)b * g.k + n) * g.oh + oy) * g.ow + ox;
                            p.ys[ui] = p.u[ui] < (double)val ? 1.0f : 0.0f;
                        }
                    }
                }
            } else if (MODE == CONV_DGRAD) {
                const long long row = (long long)item * 128 + r;
                const bool rok = row < p.npix;
                const int b = rok ? (int)(row / HW) : 0, rem = rok ? (int)(row % HW) : 0;
#pragma unroll
                for (int n = 0; n < NPAD; ++n) {
                    if (n >= g.c) break;  // uniform
                    float val = v[n];
                    if (p.dg_bias) val = apply_act(p.dg_act, val + p.dg_bias[n]);
                    if (rok) p.dx[(long long)b * p.lddx + (long long)n * HW + rem] = val;
                    if (p.vstat_f) {  // visible-bias and reconstruction partials of this warp's 32 rows
                        float d = 0.0f;
                        double dd = 0.0;
                        if (rok) {
                            const float x0 = p.x[(long long)b * p.ldx + (long long)n * HW + rem];
                            d = x0 - val;
                            const double e = (double)x0 - (double)val;
                            dd = e * e;
                        }
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            d += __shfl_xor_sync(0xffffffffu, d, o);
                            dd += __shfl_xor_sync(0xffffffffu, dd, o);
                        }
                        if (lane == 0) {
                            const long long si = ((long long)item * 4 + q) * g.c + n;
                            p.vstat_f[si] = d;
                            p.vstat_d[si] = dd;
                        }
                    }
                }
            } else {  // WGRAD partial tile: rows = patch index, cols = kernels
                float* dst = p.ws + (long long)item * 128 * 32 + r * 32;
#pragma unroll
                for (int n = 0; n < 32; n += 4)
                    *reinterpret_cast<float4*>(dst + n) = make_float4(v[n], v[n + 1], v[n + 2], v[n + 3]);
            }
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == MMA_WARP) {
        tc_fence_after();
        tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
}

// dZ = unpool(dpool) * act'(y): pool_backward (layers.hpp:240-271) + activation_gradient
// (layers.hpp:284-298) materialised once per layer (dense [B][K][OH][OW]) so the dgrad / wgrad
// gathers read it with one load. One thread per pooled element, float2 stores.
static __global__ void conv_dz_kernel(const ConvParams p, float* __restrict__ dz) {
    pdl_wait();
    const long long per = (long long)p.g.k * p.ph * p.pw;
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= (long long)p.B * per) return;
    const long long b = idx / per, pi = idx - b * per;
    const float gv = p.dy[b * p.lddy + pi], yv = p.y[b * p.ldy + pi];
    const float d = act_grad(p.act, gv, yv);
    if (p.pool) {
        const int k = (int)(pi / (p.ph * p.pw)), rem = (int)(pi % (p.ph * p.pw));
        const int py = rem / p.pw, px = rem % p.pw;
        const int code = p.arg[b * per + pi];
        float* o = dz + ((b * p.g.k + k) * p.g.oh + 2 * py) * (long long)p.g.ow + 2 * px;
        *reinterpret_cast<float2*>(o) = make_float2(code == 0 ? d : 0.0f, code == 1 ? d : 0.0f);
        *reinterpret_cast<float2*>(o + p.g.ow) = make_float2(code == 2 ? d : 0.0f, code == 3 ? d : 0.0f);
    } else {
        dz[b * per + pi] = d;
    }
}

// fixed-order reduction of the WGRAD partials (chunk groups summed by 8 thread groups, then the 8
// group sums in order) + the optimizer step on kernels and bias (sgd_momentum_step,
// optim.hpp:69-80) or a plain gradient store (data-parallel split mode). One block per patch row.
static __global__ void conv_wgrad_reduce_kernel(const float* __restrict__ ws, int chunks, int ckk, int kout, int mtiles,
                                         float* kern, float* kvel, float* bias, float* bvel, float* gk, float* gb,
                                         int fused, float lr, float mom, float wd) {
    pdl_wait();
    const int j = blockIdx.x;  // patch row (c,di,dj) or the bias row ckk
    const int mt = j / 128, r = j % 128;
    const int n = threadIdx.x & 31, grp = threadIdx.x >> 5;
    __shared__ float part[8][32];
    float acc = 0.0f;
    for (int ch = grp; ch < chunks; ch += 8) acc += ws[((long long)(mt * chunks + ch) * 128 + r) * 32 + n];
    part[grp][n] = acc;
    __syncthreads();
    if (grp != 0 || n >= kout) return;
    float s = part[0][n];
    for (int q = 1; q < 8; ++q) s += part[q][n];
    float* pp = j < ckk ? kern + (long long)n * ckk + j : bias + n;
    float* vv = j < ckk ? kvel + (long long)n * ckk + j : bvel + n;
    float* gg = j < ckk ? gk + (long long)n * ckk + j : gb + n;
    if (fused) {
        const float gr = s + wd * *pp;
        const float vel = mom * *vv - lr * gr;
        *vv = vel;
        *pp = *pp + vel;
    } else {
        *gg = s;
    }
    (void)mtiles;
}

// ------------------------------------------------------------------ host planning
struct ConvFwdLaunch {
    ConvParams p;
    int np = 8;
    bool x3 = true;
    int grid = 1;
    double flops = 0, bytes = 0;
    void run(cudaStream_t st) const;
};

struct ConvBwdLaunch {
    ConvParams pd, pw;  // dgrad (if has_dgrad), wgrad
    bool has_dgrad = false;
    int np_d = 8;
    bool x3 = true;
    int grid_d = 1, grid_w = 1;
    std::shared_ptr<DevMem> ws, dz;
    float *kern, *kvel, *bias, *bvel, *gk, *gb;
    float lr, mom, wd;
    double flops = 0, bytes = 0;
    void run(cudaStream_t st, bool fused) const;
    int kernels() const { return has_dgrad ? 4 : 3; }
};

template <int NP, int MODE, bool X3>
inline void launch_conv_inst(const ConvParams& p, int grid, cudaStream_t st) {
    using Cfg = ConvCfg<NP, MODE, X3>;
    static bool attr = [] {
        B2N_CUDA(cudaFuncSetAttribute(conv_tc_kernel<NP, MODE, X3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      Cfg::SMEM));
        return true;
    }();
    (void)attr;
    launch_ex(conv_tc_kernel<NP, MODE, X3>, dim3(grid), dim3(kConvThreads), Cfg::SMEM, st, 1u, p);
}

template <int MODE>
void launch_conv(const ConvParams& p, int np, bool x3, int grid, cudaStream_t st) {
    if constexpr (MODE == CONV_WGRAD) {  // always 32 kernel columns (MN-major atom width)
        if (x3) launch_conv_inst<32, MODE, true>(p, grid, st);
        else launch_conv_inst<32, MODE, false>(p, grid, st);
        return;
    }
    if (np == 8) {
        if (x3) launch_conv_inst<8, MODE, true>(p, grid, st);
        else launch_conv_inst<8, MODE, false>(p, grid, st);
    } else if (np == 16) {
        if (x3) launch_conv_inst<16, MODE, true>(p, grid, st);
        else launch_conv_inst<16, MODE, false>(p, grid, st);
    } else {
        if (x3) launch_conv_inst<32, MODE, true>(p, grid, st);
        else launch_conv_inst<32, MODE, false>(p, grid, st);
    }
}
// each mode is instantiated in its own translation unit (conv_fwd.cu / conv_dgrad.cu / conv_wgrad.cu)
#ifndef B2N_CONV_INSTANTIATE
extern template void launch_conv<CONV_FWD>(const ConvParams&, int, bool, int, cudaStream_t);
extern template void launch_conv<CONV_DGRAD>(const ConvParams&, int, bool, int, cudaStream_t);
extern template void launch_conv<CONV_WGRAD>(const ConvParams&, int, bool, int, cudaStream_t);
#endif

inline void ConvFwdLaunch::run(cudaStream_t st) const { launch_conv<CONV_FWD>(p, np, x3, grid, st); }

inline void ConvBwdLaunch::run(cudaStream_t st, bool fused) const {
    const long long npool = (long long)pw.B * pw.g.k * pw.ph * pw.pw;
    launch_ex(conv_dz_kernel, dim3((unsigned)((npool + 255) / 256)), dim3(256), 0, st, 1u, pw, dz->as<float>());
    if (has_dgrad) launch_conv<CONV_DGRAD>(pd, np_d, x3, grid_d, st);
    launch_conv<CONV_WGRAD>(pw, 32, x3, grid_w, st);
    launch_ex(conv_wgrad_reduce_kernel, dim3(pw.ckk + 1), dim3(256), 0, st, 1u, (const float*)pw.ws, pw.chunks, pw.ckk,
              pw.g.k, pw.mtiles_w, kern, kvel, bias, bvel, gk, gb, fused ? 1 : 0, lr, mom, wd);
}

inline int conv_np(int n) {
    if (n <= 8) return 8;
    if (n <= 16) return 16;
    if (n <= 32) return 32;
    throw Error(B2N_ESHAPE, "b200nn conv: at most 32 kernels / channels per layer on the tensor-core path");
}

inline int sm_count() {
    static int n = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

inline ConvParams conv_base(const ConvGeom& g, int B, int act, bool pool) {
    ConvParams p;
    std::memset(&p, 0, sizeof(p));
    p.g = g;
    p.B = B;
    p.act = act;
    p.pool = pool ? 1 : 0;
    p.ph = pool ? g.oh / 2 : g.oh;
    p.pw = pool ? g.ow / 2 : g.ow;
    p.ckk = g.c * g.kh * g.kw;
    p.kkk = g.k * g.kh * g.kw;
    if (p.ckk > 320 || p.kkk > 320) throw Error(B2N_ESHAPE, "b200nn conv: c*kh*kw and k*kh*kw must be <= 320");
    return p;
}

inline ConvFwdLaunch plan_conv_fwd(const ConvGeom& g, int B, const float* x, long long ldx, const float* wk,
                                   const float* bias, int act, bool pool, float* y, long long ldy, uint8_t* arg,
                                   bool x3) {
    ConvFwdLaunch L;
    L.p = conv_base(g, B, act, pool);
    L.p.x = x;
    L.p.ldx = ldx;
    L.p.wk = wk;
    L.p.bias = bias;
    L.p.y = y;
    L.p.ldy = ldy;
    L.p.arg = arg;
    L.p.npix = (long long)B * g.oh * g.ow;
    L.p.items = (int)((L.p.npix + 127) / 128);
    L.p.kblocks = (L.p.ckk + 31) / 32;
    L.np = conv_np(g.k);
    L.x3 = x3;
    L.grid = std::min(L.p.items, sm_count());
    L.flops = 2.0 * L.p.npix * g.k * L.p.ckk;
    const double out = (double)B * g.k * L.p.ph * L.p.pw;
    L.bytes = (double)B * g.c * g.h * g.w * 4 + out * 4 + (pool ? out : 0) + (double)g.k * (L.p.ckk + 1) * 4;
    return L;
}

inline ConvBwdLaunch plan_conv_bwd(const ConvGeom& g, int B, const float* x, long long ldx, const float* wk,
                                   const float* bias, int act, bool pool, const float* y, long long ldy,
                                   const uint8_t* arg, const float* dy, long long lddy, float* dx, long long lddx,
                                   float* kern, float* kvel, float* biasp, float* bvel, float* gk, float* gb, float lr,
                                   float mom, float wd, bool x3) {
    (void)bias;
    ConvBwdLaunch L;
    ConvParams base = conv_base(g, B, act, pool);
    base.x = x;
    base.ldx = ldx;
    base.wk = wk;
    base.y = const_cast<float*>(y);
    base.ldy = ldy;
    base.arg = const_cast<uint8_t*>(arg);
    base.dy = dy;
    base.lddy = lddy;
    L.dz = std::make_shared<DevMem>();
    L.dz->alloc((size_t)B * g.k * g.oh * g.ow * 4);
    base.dz = L.dz->as<float>();
    L.x3 = x3;
    const double opix = (double)B * g.oh * g.ow, ipix = (double)B * g.h * g.w;
    const double pooled = (double)B * g.k * base.ph * base.pw;
    if (dx) {
        L.has_dgrad = true;
        L.pd = base;
        L.pd.dx = dx;
        L.pd.lddx = lddx;
        L.pd.npix = (long long)B * g.h * g.w;
        L.pd.items = (int)((L.pd.npix + 127) / 128);
        L.pd.kblocks = (base.kkk + 31) / 32;
        L.np_d = conv_np(g.c);
        L.grid_d = std::min(L.pd.items, sm_count());
        L.flops += 2.0 * ipix * g.c * base.kkk;
        L.bytes += pooled * 9 + ipix * g.c * 4;
    }
    L.pw = base;
    L.pw.npix = (long long)B * g.oh * g.ow;
    L.pw.mtiles_w = (base.ckk + 1 + 127) / 128;
    // pixel chunks: ~2 work items per SM, each a multiple of 32 pixels
    const long long want_items = 2LL * sm_count();
    long long chunks = std::max<long long>(1, want_items / L.pw.mtiles_w);
    long long chunk_px = (L.pw.npix + chunks - 1) / chunks;
    chunk_px = std::max<long long>(32, (chunk_px + 31) / 32 * 32);
    chunks = (L.pw.npix + chunk_px - 1) / chunk_px;
    L.pw.chunk_px = (int)chunk_px;
    L.pw.chunks = (int)chunks;
    L.pw.items = (int)(L.pw.mtiles_w * chunks);
    L.pw.kblocks = (int)(chunk_px / 32);
    L.grid_w = std::min(L.pw.items, sm_count());
    L.ws = std::make_shared<DevMem>();
    L.ws->alloc((size_t)L.pw.items * 128 * 32 * 4);
    L.pw.ws = L.ws->as<float>();
    L.kern = kern;
    L.kvel = kvel;
    L.bias = biasp;
    L.bvel = bvel;
    L.gk = gk;
    L.gb = gb;
    L.lr = lr;
    L.mom = mom;
    L.wd = wd;
    L.flops += 2.0 * opix * g.k * (base.ckk + 1);
    L.bytes += ipix * g.c * 4 + pooled * 9 + (double)g.k * (base.ckk + 1) * 16;
    return L;
}

}  // namespace b2n
