// conv.cuh -- convolution layers as implicit-GEMM tcgen05 kernels (conv_forward / conv_backward,
// layers.hpp:132-193, conv.hpp:180-345) with the layer's activation and 2x2 max-pool fused.
//
// One persistent, warp-specialised kernel template, three modes:
//   FWD   : M = output pixels (ordered so the 4 pixels of each pooling window are 4 consecutive
//           rows / TMEM lanes), N = kernels, K = c*kh*kw. Epilogue: bias + act, 2x2 max with the
//           reference's first-index tie rule (layers.hpp:228-232) via lane shuffles, writes only the
//           pooled activation and a 1-byte argmax code -- the full-resolution conv output never
//           reaches HBM.
//   DGRAD : M = input pixels, N = input channels, K = kernels*kh*kw; the A operand is dZ gathered on
//           the fly from the pooled gradient, argmax code and pooled activation (act'), i.e.
//           pool_backward + activation_gradient + the padded-valid full conv (conv.hpp:337-345) in
//           one pass. Skipped for the first layer (its dx is dead).
//   WGRAD : M = patch index (c,di,dj) plus a ones row (-> bias gradient), N = kernels, K = output
//           pixels split across CTAs; per-CTA partial tiles are reduced in fixed order by
//           conv_wgrad_reduce_kernel, which also applies the SGD-momentum step (deterministic).
// Roles (288 threads): warps 0-3 gather A (and per-block B) tiles into 128 B-swizzled smem with the
// 3xTF32 lo split, warp 4 allocates TMEM and issues tcgen05.mma, warps 5-8 drain a double-buffered
// TMEM accumulator through the epilogue.
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
    // work decomposition
    int items;       // total work items
    int kblocks;     // K blocks per item
    int ckk;         // c*kh*kw
    int kkk;         // k*kh*kw
    int mtiles_w;    // WGRAD: M' tiles
    int chunk_px;    // WGRAD: output pixels per item (multiple of 32)
    int chunks;      // WGRAD: pixel chunks
    long long npix;  // rows of the GEMM view (pixels)
};

constexpr int kConvThreads = 288;
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

__device__ __forceinline__ float act_grad(int act, float g, float y) {
    if (act == ACT_SIGMOID) return g * y * (1.0f - y);  // layers.hpp:294
    if (act == ACT_RELU) return y > 0.0f ? g : 0.0f;
    return g;
}

// dZ = gradient w.r.t. the conv's pre-activation output at (b, kk, oy, ox), from the pooled
// gradient: pool_backward (layers.hpp:240-271) then activation_gradient (layers.hpp:284-298)
__device__ __forceinline__ float conv_dz(const ConvParams& p, int b, int kk, int oy, int ox) {
    if (p.pool) {
        const int py = oy >> 1, px = ox >> 1;
        const long long pi = ((long long)kk * p.ph + py) * p.pw + px;
        const int code = p.arg[(long long)b * p.g.k * p.ph * p.pw + pi];
        if (code != ((oy & 1) << 1) + (ox & 1)) return 0.0f;
        return act_grad(p.act, p.dy[(long long)b * p.lddy + pi], p.y[(long long)b * p.ldy + pi]);
    }
    const long long pi = ((long long)kk * p.g.oh + oy) * p.g.ow + ox;
    return act_grad(p.act, p.dy[(long long)b * p.lddy + pi], p.y[(long long)b * p.ldy + pi]);
}

// decode a GEMM row of the FWD view into an output pixel; pool order puts a window on 4 rows
__device__ __forceinline__ bool fwd_pixel(const ConvParams& p, long long row, int& b, int& oy, int& ox) {
    if (row >= p.npix) return false;
    if (p.pool) {
        const long long win = row >> 2;
        const int w = (int)(row & 3);
        const long long per = (long long)p.ph * p.pw;
        b = (int)(win / per);
        const int rem = (int)(win % per);
        oy = 2 * (rem / p.pw) + (w >> 1);
        ox = 2 * (rem % p.pw) + (w & 1);
    } else {
        const long long per = (long long)p.g.oh * p.g.ow;
        b = (int)(row / per);
        const int rem = (int)(row % per);
        oy = rem / p.g.ow;
        ox = rem % p.g.ow;
    }
    return true;
}

template <int NP, int MODE, bool X3>
__global__ void __launch_bounds__(kConvThreads, 1) conv_tc_kernel(const ConvParams p) {
    using Cfg = ConvCfg<NP, MODE, X3>;
    constexpr int S = kConvStages;
    constexpr int NPAD = Cfg::NPAD;
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
    const int HW = g.h * g.w;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 128);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 128);
        }
        fence_barrier_init();
    }
    if (warp == 4) tmem_alloc(tslot, Cfg::TMEM_COLS);
    // per-k tables and the static weight operand (FWD: W[n][c,di,dj]; DGRAD: W[kk][n][di,dj] as [n][kk,di,dj])
    const int Kdim = MODE == CONV_DGRAD ? p.kkk : p.ckk;
    for (int k = threadIdx.x; k < Cfg::KMAX; k += blockDim.x) {
        int off = 0, didj = 0;
        if (k < Kdim) {
            const int khw = g.kh * g.kw;
            const int ch = k / khw, r = k % khw, di = r / g.kw, dj = r % g.kw;
            off = MODE == CONV_DGRAD ? ch * p.ph * p.pw : ch * HW;  // (unused for dgrad)
            didj = (di << 16) | dj;
            if (MODE == CONV_DGRAD) off = ch;
        }
        ktab[k] = make_int2(off, didj);
    }
    if (MODE != CONV_WGRAD) {
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
            const int kb = k >> 5;
            uint8_t* blk = wb + kb * (NP * 128);
            *reinterpret_cast<float*>(blk + kmaj_off(n, k & 31)) = v;
            if (X3) *reinterpret_cast<float*>(blk + Cfg::WB_BYTES / 2 + kmaj_off(n, k & 31)) = split_lo1(v);
        }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tslot;

    if (warp < 4) {
        // ===================== gather producers (128 threads)
        const int t = threadIdx.x;
        int it = 0;
        for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
            for (int kb = 0; kb < p.kblocks; ++kb, ++it) {
                const int s = it % S;
                mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
                uint8_t* a = stages + s * Cfg::STAGE_BYTES;
                uint8_t* alo = a + Cfg::A_BYTES + Cfg::B_BYTES;
                if (MODE == CONV_FWD) {
                    int b, oy, ox;
                    const bool ok = fwd_pixel(p, (long long)item * 128 + t, b, oy, ox);
                    const float* xb = p.x + (long long)b * p.ldx;
#pragma unroll 4
                    for (int kk = 0; kk < 32; ++kk) {
                        const int k = kb * 32 + kk;
                        float v = 0.0f;
                        if (ok && k < p.ckk) {
                            const int2 e = ktab[k];
                            const int iy = oy + (e.y >> 16) - g.pad, ix = ox + (e.y & 0xFFFF) - g.pad;
                            if (iy >= 0 && iy < g.h && ix >= 0 && ix < g.w) v = __ldg(xb + e.x + iy * g.w + ix);
                        }
                        *reinterpret_cast<float*>(a + kmaj_off(t, kk)) = v;
                        if (X3) *reinterpret_cast<float*>(alo + kmaj_off(t, kk)) = split_lo1(v);
                    }
                } else if (MODE == CONV_DGRAD) {
                    const long long row = (long long)item * 128 + t;
                    const bool ok = row < p.npix;
                    const int b = ok ? (int)(row / HW) : 0, rem = ok ? (int)(row % HW) : 0;
                    const int iy = rem / g.w, ix = rem % g.w;
#pragma unroll 4
                    for (int kk = 0; kk < 32; ++kk) {
                        const int k = kb * 32 + kk;
                        float v = 0.0f;
                        if (ok && k < p.kkk) {
                            const int2 e = ktab[k];
                            const int oy = iy + g.pad - (e.y >> 16), ox = ix + g.pad - (e.y & 0xFFFF);
                            if (oy >= 0 && oy < g.oh && ox >= 0 && ox < g.ow) v = conv_dz(p, b, e.x, oy, ox);
                        }
                        *reinterpret_cast<float*>(a + kmaj_off(t, kk)) = v;
                        if (X3) *reinterpret_cast<float*>(alo + kmaj_off(t, kk)) = split_lo1(v);
                    }
                } else {  // WGRAD: A'[K'=pixel][M'=patch] and B'[K'=pixel][N'=kernel], MN-major
                    const int mt = item / p.chunks, ch = item % p.chunks;
                    const int kp = t & 31, grp = t >> 5;
                    const long long px = (long long)ch * p.chunk_px + kb * 32 + kp;
                    const bool ok = px < p.npix && kb * 32 + kp < p.chunk_px;
                    const int per = g.oh * g.ow;
                    const int b = ok ? (int)(px / per) : 0, rem = ok ? (int)(px % per) : 0;
                    const int oy = rem / g.ow, ox = rem % g.ow;
                    const float* xb = p.x + (long long)b * p.ldx;
                    uint8_t* bb = a + Cfg::A_BYTES;
                    uint8_t* blo = alo + Cfg::A_BYTES;
#pragma unroll 4
                    for (int jj = 0; jj < 32; ++jj) {
                        const int j = mt * 128 + grp * 32 + jj;
                        float v = 0.0f;
                        if (ok) {
                            if (j < p.ckk) {
                                const int2 e = ktab[j];
                                const int iy = oy + (e.y >> 16) - g.pad, ix = ox + (e.y & 0xFFFF) - g.pad;
                                if (iy >= 0 && iy < g.h && ix >= 0 && ix < g.w) v = __ldg(xb + e.x + iy * g.w + ix);
                            } else if (j == p.ckk) {
                                v = 1.0f;  // ones row: its product with dZ is the bias gradient
                            }
                        }
                        const uint32_t o = mnmaj_off(grp * 32 + jj, kp);
                        *reinterpret_cast<float*>(a + o) = v;
                        if (X3) *reinterpret_cast<float*>(alo + o) = split_lo1(v);
                    }
#pragma unroll
                    for (int nn = 0; nn < 8; ++nn) {
                        const int n = grp * 8 + nn;
                        const float v = (ok && n < g.k) ? conv_dz(p, b, n, oy, ox) : 0.0f;
                        const uint32_t o = mnmaj_off(n, kp);
                        *reinterpret_cast<float*>(bb + o) = v;
                        if (X3) *reinterpret_cast<float*>(blo + o) = split_lo1(v);
                    }
                }
                fence_proxy_async_smem();
                mbar_arrive(&full[s]);
            }
        }
    } else if (warp == 4) {
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
        }
    } else {
        // ===================== epilogue (warps 5..8 -> TMEM quadrants 1,2,3,0)
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
                        p.y[(long long)b * p.ldy + ((long long)n * g.oh + oy) * g.ow + ox] = val;
                    }
                }
            } else if (MODE == CONV_DGRAD) {
                const long long row = (long long)item * 128 + r;
                if (row < p.npix) {
                    const int b = (int)(row / HW), rem = (int)(row % HW);
#pragma unroll
                    for (int n = 0; n < NPAD; ++n)
                        if (n < g.c) p.dx[(long long)b * p.lddx + (long long)n * HW + rem] = v[n];
                }
            } else {  // WGRAD partial tile: rows = patch index, cols = kernels
                float* dst = p.ws + (long long)item * 128 * 32 + r * 32;
#pragma unroll
                for (int n = 0; n < 32; n += 4) *reinterpret_cast<float4*>(dst + n) = make_float4(v[n], v[n + 1], v[n + 2], v[n + 3]);
            }
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
}

// fixed-order reduction of the WGRAD partials + the optimizer step on kernels and bias
// (sgd_momentum_step, optim.hpp:69-80) or a plain gradient store (data-parallel split mode)
__global__ void conv_wgrad_reduce_kernel(const float* __restrict__ ws, int chunks, int ckk, int kout, int mtiles,
                                         float* kern, float* kvel, float* bias, float* bvel, float* gk, float* gb,
                                         int fused, float lr, float mom, float wd) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // over kout * (ckk + 1)
    if (idx >= kout * (ckk + 1)) return;
    const int n = idx / (ckk + 1), j = idx % (ckk + 1);
    const int mt = j / 128, r = j % 128;
    float acc = 0.0f;
    for (int ch = 0; ch < chunks; ++ch) acc += ws[((long long)(mt * chunks + ch) * 128 + r) * 32 + n];
    float* pp = j < ckk ? kern + (long long)n * ckk + j : bias + n;
    float* vv = j < ckk ? kvel + (long long)n * ckk + j : bvel + n;
    float* gg = j < ckk ? gk + (long long)n * ckk + j : gb + n;
    if (fused) {
        const float gr = acc + wd * *pp;
        const float vel = mom * *vv - lr * gr;
        *vv = vel;
        *pp = *pp + vel;
    } else {
        *gg = acc;
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
    std::shared_ptr<DevMem> ws;
    float *kern, *kvel, *bias, *bvel, *gk, *gb;
    float lr, mom, wd;
    double flops = 0, bytes = 0;
    void run(cudaStream_t st, bool fused) const;
    int kernels() const { return has_dgrad ? 3 : 2; }
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
    conv_tc_kernel<NP, MODE, X3><<<grid, kConvThreads, Cfg::SMEM, st>>>(p);
    B2N_CUDA(cudaGetLastError());
}

template <int MODE>
inline void launch_conv(const ConvParams& p, int np, bool x3, int grid, cudaStream_t st) {
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

inline void ConvFwdLaunch::run(cudaStream_t st) const { launch_conv<CONV_FWD>(p, np, x3, grid, st); }

inline void ConvBwdLaunch::run(cudaStream_t st, bool fused) const {
    if (has_dgrad) launch_conv<CONV_DGRAD>(pd, np_d, x3, grid_d, st);
    launch_conv<CONV_WGRAD>(pw, 32, x3, grid_w, st);
    const int n = pw.g.k * (pw.ckk + 1);
    conv_wgrad_reduce_kernel<<<(n + 127) / 128, 128, 0, st>>>(pw.ws, pw.chunks, pw.ckk, pw.g.k, pw.mtiles_w, kern,
                                                              kvel, bias, bvel, gk, gb, fused ? 1 : 0, lr, mom, wd);
    B2N_CUDA(cudaGetLastError());
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
