// convx.cuh -- the conv-stack FORWARD (conv_forward + activation + 2x2 max-pool, layers.hpp:132-148,
// :205-238, :278-282) computed bit-for-bit as the reference computes it.
//
// Why not the tensor cores here: the forward makes DISCRETE decisions -- the first-index argmax of
// every pooling window and relu's "> 0" -- that route the whole backward pass. A 3xTF32 tensor-core
// value is within ~1e-6 of the reference's, yet over the ImageNet-shaped stack at batch 128 a dozen
// of the ~44 M windows are near-ties that it resolves differently, and each misrouted window moves
// the first layers' gradients by up to ~5e-3 of their norm (measured; tools/diag/imnet_layers.py).
// Recomputing only the doubtful windows exactly (convt.cuh's fix list) cannot help past the first
// layer: the NEXT layer's inputs are then tensor-core values, and near-ties flip on those. So the
// forward values themselves have to be the reference's: ONE fp32 fma chain per output over
// (c, di, dj) in that order from 0 (conv.hpp:62-119 add_corr_map / :215-273 im2col, both backends
// the same order), padding contributing exact zeros, then + bias (a separate rounding,
// layers.hpp:138-146), the activation, and the first-index 2x2 max. On 16-kernel filters this is
// also the faster path: the 3xTF32 tensor-core forward is bound by streaming its M=128 operand from
// shared memory at N = 16, while this kernel keeps 64 independent FFMA chains per thread.
//
// Layout: thread = one 2x2 output block (one pooling window) x KG = 4*KQ kernels (grid.y = kernel
// groups). Per tile (TR x TW outputs) the input halo is transposed from the row-blocked activations
// ([b][y][c/4][x][4], convt.cuh) into channel planes [C][HR][PWp] in shared memory and the kernel
// group's weights into [C][kh][kw][KG]; the channel loop streams two halo rows at a time (float2
// loads), every (c, di, dj) step is KQ broadcast float4 weight loads + 4*KG FFMAs.
#pragma once
#include "convt.cuh"

namespace b2n {

struct ConvXParams {
    int B, C, G, Hin, Win, kh, kw, pad, OH, OW, K;  // C real input channels (G quads in the blocked input)
    int TR, TW, HR, PW, PWp;                       // tile rows / cols (even), halo rows / cols, plane pitch
    int SR;                                        // output rows per pass of the threads (TR = passes * SR)
    int tiles_x, tiles_y;
    int act, pool;
    const float* x;  // row-blocked input [b][y][G][Win][4]
    long long x_bstride;
    const float* wk;    // [K][C][kh][kw]
    const float* bias;  // [K]
    TLayout out;        // pooled (or full) output, row-blocked or NCHW
    uint8_t* codes;     // pool argmax codes, row-blocked bytes [b][py][Kq][PWc][4]
    long long codes_bstride;
    int codes_pw;
};

// the reference's sigmoidf (layers.hpp:279): 1 / (1 + expf(-v)) with glibc's expf, bit for bit (ptx.cuh)
__device__ __forceinline__ float sigmoid_exact(float v) { return 1.0f / (1.0f + glibc_expf(-v)); }
__device__ __forceinline__ float act_exact(int act, float v) {
    if (act == ACT_SIGMOID) return sigmoid_exact(v);
    if (act == ACT_RELU) return v > 0.0f ? v : 0.0f;
    return v;
}

// 4-byte async copy global -> shared; src_bytes = 0 zero-fills (conv padding / map edges)
__device__ __forceinline__ void cp_async4(float* dst, const float* src, int src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes) : "memory");
}

template <int KH, int KW, int KQ, int ACT>
__global__ void __launch_bounds__(128, 4) convx_fwd_kernel(const ConvXParams p) {
    constexpr int KG = 4 * KQ;
    constexpr int NX = (KW + 2) / 2;  // float2 loads per halo row segment (KW + 1 values, rounded up)
    extern __shared__ float4 smx[];
    float4* ws = smx;                                                // [C][KH][KW][KQ] float4
    float* hs = reinterpret_cast<float*>(smx + p.C * KH * KW * KQ);  // planes [C][HR][PWp]
    const int tid = threadIdx.x, nt = blockDim.x;
    const int kg0 = blockIdx.y * KG;
    const int per = p.tiles_x * p.tiles_y;
    const int b = blockIdx.x / per, rem = blockIdx.x - b * per;
    const int ty = rem / p.tiles_x;
    const int y0 = ty * p.TR, x0 = (rem - ty * p.tiles_x) * p.TW;
    const int plane = p.HR * p.PWp;
    pdl_wait();  // weights and input are written by earlier kernels of the step
    {
        // halo rows [y0 - pad, + HR) x cols [x0 - pad, + PW) of the real channels, straight into channel
        // planes by 4-byte async copies (one round trip for the whole halo; consecutive threads read
        // consecutive floats of a [quad][col][4] row run), zero-filled outside the map (padding)
        const int ys = y0 - p.pad, xs = x0 - p.pad;
        // a thread keeps its (quad, col, j) positions of a halo row and walks the rows (no per-element
        // index division)
        const int rowlen = p.G * p.PW * 4;  // floats of one halo row: [quad][col][4]
        const float* xb = p.x + (long long)b * p.x_bstride;
        const long long ystride = (long long)p.G * p.Win * 4;
        for (int r2 = tid; r2 < rowlen; r2 += nt) {
            const int q = r2 / (p.PW * 4), r3 = r2 - q * (p.PW * 4);
            const int col = r3 >> 2, j = r3 & 3;
            const int c = 4 * q + j;
            if (c >= p.C) continue;
            const int ix = xs + col;
            const bool inx = (unsigned)ix < (unsigned)p.Win;
            float* dst = hs + c * plane + col;
            const float* src = xb + ((long long)q * p.Win + ix) * 4 + j;
            for (int row = 0; row < p.HR; ++row) {
                const int iy = ys + row;
                const bool in = inx && (unsigned)iy < (unsigned)p.Hin;
                cp_async4(dst + row * p.PWp, in ? src + iy * ystride : xb, in ? 4 : 0);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        float* wsf = reinterpret_cast<float*>(ws);
        const int n = p.C * KH * KW * KG;
        for (int i = tid; i < n; i += nt) {
            const int k = i % KG, r = i / KG;  // r = c * KH * KW + tap
            const int kk = kg0 + k;
            wsf[i] = kk < p.K ? __ldg(p.wk + (long long)kk * p.C * KH * KW + r) : 0.0f;
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
    pdl_trigger();
    const int wpr = p.TW / 2;    // windows per tile row
    const int wrows = p.SR / 2;  // window rows per pass of the CTA's threads
    const int wy0 = tid / wpr, wx = tid - wy0 * wpr;
    if (wy0 >= wrows) return;
    for (int wy = wy0; wy < p.TR / 2; wy += wrows) {  // the tile's passes reuse its halo
        const int oy = y0 + 2 * wy, ox = x0 + 2 * wx;
        if (oy >= p.OH || ox >= p.OW) break;
        float acc[4][KG];
#pragma unroll
        for (int o = 0; o < 4; ++o)
#pragma unroll
            for (int k = 0; k < KG; ++k) acc[o][k] = 0.0f;
        const float* hbase = hs + (2 * wy) * p.PWp + 2 * wx;
        for (int c = 0; c < p.C; ++c) {
            const float* hc = hbase + c * plane;
            float ra[2 * NX], rb[2 * NX];
#pragma unroll
            for (int j = 0; j < NX; ++j) {
                const float2 t2 = *reinterpret_cast<const float2*>(hc + 2 * j);
                ra[2 * j] = t2.x, ra[2 * j + 1] = t2.y;
            }
            const float4* wc = ws + c * KH * KW * KQ;
#pragma unroll
            for (int di = 0; di < KH; ++di) {
#pragma unroll
                for (int j = 0; j < NX; ++j) {
                    const float2 t2 = *reinterpret_cast<const float2*>(hc + (di + 1) * p.PWp + 2 * j);
                    rb[2 * j] = t2.x, rb[2 * j + 1] = t2.y;
                }
#pragma unroll
                for (int dj = 0; dj < KW; ++dj) {
                    float w[KG];
#pragma unroll
                    for (int q = 0; q < KQ; ++q) {
                        const float4 t4 = wc[(di * KW + dj) * KQ + q];
                        w[4 * q] = t4.x, w[4 * q + 1] = t4.y, w[4 * q + 2] = t4.z, w[4 * q + 3] = t4.w;
                    }
                    // acc = fma(ker, x, acc): the reference's chain order (c, di, dj), conv.hpp:62-89
#pragma unroll
                    for (int k = 0; k < KG; ++k) {
                        acc[0][k] = fmaf(w[k], ra[dj], acc[0][k]);
                        acc[1][k] = fmaf(w[k], ra[dj + 1], acc[1][k]);
                        acc[2][k] = fmaf(w[k], rb[dj], acc[2][k]);
                        acc[3][k] = fmaf(w[k], rb[dj + 1], acc[3][k]);
                    }
                }
#pragma unroll
                for (int j = 0; j < 2 * NX; ++j) ra[j] = rb[j];
            }
        }
        // + bias (its own rounding, layers.hpp:138-146), activation, then the pool or the plain store
        const int Kq = (p.out.C + 3) >> 2;
        float* ob = p.out.p + (long long)b * p.out.bstride;
        if (p.pool) {
            const int py = oy >> 1, px = ox >> 1;
    #pragma unroll
            for (int q = 0; q < KQ; ++q) {
                const int gq = (kg0 >> 2) + q;
                if (gq >= Kq) break;
                float o4[4];
                uint32_t cw = 0;
    #pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int k = 4 * q + jj, kk = kg0 + k;
                    float best = 0.0f;
                    uint32_t code = 0;
                    if (kk < p.K) {
                        const float bb = __ldg(p.bias + kk);
                        // window order (0,0) (0,1) (1,0) (1,1), the first maximum wins (layers.hpp:228-232)
                        best = act_exact(ACT, acc[0][k] + bb);
    #pragma unroll
                        for (int o = 1; o < 4; ++o) {
                            const float a = act_exact(ACT, acc[o][k] + bb);
                            if (a > best) best = a, code = (uint32_t)o;
                        }
                    }
                    o4[jj] = best;
                    cw |= code << (8 * jj);
                }
                if (p.out.blocked) {
                    *reinterpret_cast<float4*>(ob + (((long long)py * Kq + gq) * p.out.W + px) * 4) =
                        make_float4(o4[0], o4[1], o4[2], o4[3]);
                } else {
    #pragma unroll
                    for (int jj = 0; jj < 4; ++jj)
                        if (4 * gq + jj < p.out.C) ob[((long long)(4 * gq + jj) * p.out.H + py) * p.out.W + px] = o4[jj];
                }
                *reinterpret_cast<uint32_t*>(p.codes + (long long)b * p.codes_bstride +
                                             (((long long)py * Kq + gq) * p.codes_pw + px) * 4) = cw;
            }
        } else {
    #pragma unroll
            for (int o = 0; o < 4; ++o) {
                const int y = oy + (o >> 1), x = ox + (o & 1);
                if (y >= p.OH || x >= p.OW) continue;
    #pragma unroll
                for (int q = 0; q < KQ; ++q) {
                    const int gq = (kg0 >> 2) + q;
                    if (gq >= Kq) break;
                    float o4[4];
    #pragma unroll
                    for (int jj = 0; jj < 4; ++jj) {
                        const int kk = kg0 + 4 * q + jj;
                        o4[jj] = kk < p.K ? act_exact(ACT, acc[o][4 * q + jj] + __ldg(p.bias + kk)) : 0.0f;
                    }
                    if (p.out.blocked) {
                        *reinterpret_cast<float4*>(ob + (((long long)y * Kq + gq) * p.out.W + x) * 4) =
                            make_float4(o4[0], o4[1], o4[2], o4[3]);
                    } else {
    #pragma unroll
                        for (int jj = 0; jj < 4; ++jj)
                            if (4 * gq + jj < p.out.C) ob[((long long)(4 * gq + jj) * p.out.H + y) * p.out.W + x] = o4[jj];
                    }
                }
            }
        }
    }
}

struct ConvXLaunch {
    ConvXParams p;
    int kq = 4, groups = 1, threads = 128, smem = 0, grid = 1;
    double flops = 0, bytes = 0;
    void run(cudaStream_t st) const;
};

// the exact forward over a blocked input; output / codes / act / pool / weights filled by the caller
inline ConvXLaunch plan_convx_fwd(int B, int C, int Hin, int Win, int kh, int kw, int pad, int K) {
    if (!((kh == 3 && kw == 3) || (kh == 5 && kw == 5)))
        throw Error(B2N_ESHAPE, "b200nn conv: the exact forward covers 3x3 and 5x5 filters");
    ConvXLaunch L;
    ConvXParams& p = L.p;
    std::memset(&p, 0, sizeof(p));
    p.B = B;
    p.C = C;
    p.G = (C + 3) / 4;
    p.Hin = Hin;
    p.Win = Win;
    p.kh = kh;
    p.kw = kw;
    p.pad = pad;
    p.OH = Hin + 2 * pad - kh + 1;
    p.OW = Win + 2 * pad - kw + 1;
    p.K = K;
    L.kq = K <= 8 ? 2 : K <= 12 ? 3 : 4;
    L.groups = (K + 4 * L.kq - 1) / (4 * L.kq);
    auto even = [](int n) { return (n + 1) & ~1; };
    p.TW = std::min(32, even(p.OW));
    p.SR = std::min(16, even(p.OH));
    while ((p.SR / 2) * (p.TW / 2) > 128) p.SR -= 2;
    L.threads = std::max(32, ((p.SR / 2) * (p.TW / 2) + 31) / 32 * 32);
    // several passes per tile when the channel planes are small (few input channels): the CTA's fixed
    // costs (weights, the halo round trip, launch) are paid once per TR rows (<= ~40 KB of planes)
    p.PW = p.TW + kw - 1;
    p.PWp = (p.PW + 2) & ~1;  // float2 loads: even pitch, and room for the (KW + 1)-th column of the last window
    p.tiles_x = (p.OW + p.TW - 1) / p.TW;
    p.TR = p.SR;
    {  // taller tiles while the planes stay small and the grid keeps >= 8 CTAs per SM
        static const int maxpass = std::getenv("B2N_CONVX_PASSES") ? std::atoi(std::getenv("B2N_CONVX_PASSES")) : 4;
        auto planes = [&](int tr) { return (long long)C * (tr + kh - 1) * p.PWp * 4; };
        auto ctas = [&](int tr) { return (long long)B * p.tiles_x * ((p.OH + tr - 1) / tr); };
        while (p.TR + p.SR <= ((p.OH + 1) & ~1) && p.TR < maxpass * p.SR && planes(p.TR + p.SR) <= 40 * 1024 &&
               ctas(p.TR + p.SR) >= 8LL * sm_count())
            p.TR += p.SR;
    }
    p.HR = p.TR + kh - 1;
    p.tiles_y = (p.OH + p.TR - 1) / p.TR;
    L.smem = C * kh * kw * L.kq * 16 + C * p.HR * p.PWp * 4;  // weights (KQ float4 per tap) + planes
    if (L.smem > 226 * 1024) throw Error(B2N_ESHAPE, "b200nn conv: exact-forward tile does not fit shared memory");
    L.flops = 2.0 * B * p.OH * p.OW * K * (double)C * kh * kw;
    L.grid = B * p.tiles_x * p.tiles_y;
    return L;
}

void launch_convx_fwd(const ConvXLaunch& L, cudaStream_t st);
inline void ConvXLaunch::run(cudaStream_t st) const { launch_convx_fwd(*this, st); }

#ifdef B2N_CONVX_INSTANTIATE
template <int KH, int KW, int KQ, int ACT>
inline void launch_convx_inst(const ConvXLaunch& L, cudaStream_t st) {
    auto k = convx_fwd_kernel<KH, KW, KQ, ACT>;
    static int attr = 0;
    if (attr < L.smem) {
        B2N_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L.smem));
        // all of the unified L1 as shared memory: 4 CTAs of ~50 KB per SM (the default carveout fits 2)
        B2N_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        attr = L.smem;
    }
    launch_ex(k, dim3(L.grid, L.groups), dim3(L.threads), (size_t)L.smem, st, 1u, L.p);
}
template <int KH, int KW, int KQ>
inline void launch_convx_act(const ConvXLaunch& L, cudaStream_t st) {
    if (L.p.act == ACT_RELU) launch_convx_inst<KH, KW, KQ, ACT_RELU>(L, st);
    else if (L.p.act == ACT_SIGMOID) launch_convx_inst<KH, KW, KQ, ACT_SIGMOID>(L, st);
    else launch_convx_inst<KH, KW, KQ, ACT_NONE>(L, st);
}
void launch_convx_fwd(const ConvXLaunch& L, cudaStream_t st) {
    if (L.p.kh == 3) {
        if (L.kq == 2) launch_convx_act<3, 3, 2>(L, st);
        else if (L.kq == 3) launch_convx_act<3, 3, 3>(L, st);
        else launch_convx_act<3, 3, 4>(L, st);
    } else {
        if (L.kq == 2) launch_convx_act<5, 5, 2>(L, st);
        else if (L.kq == 3) launch_convx_act<5, 5, 3>(L, st);
        else launch_convx_act<5, 5, 4>(L, st);
    }
}
#endif

}  // namespace b2n
