// crbm_fused.cuh -- the whole convolutional-RBM CD-1 step (crbm_cd_update, energy.hpp:333-376) in
// ONE launch, one CTA per image, everything between v0 and the per-image statistics resident in
// shared memory.
//
// Why not the tensor cores here: a CRBM's visible side has few channels (MNIST: 1), so the
// v1 = conv_full(hs, K^T) product has N = c_in = 1 (padded to 8 on tcgen05: >= 87 % of every MMA
// wasted) and each of the four implicit-GEMM launches of the split path (crbm.cuh) is latency-
// bound at B = 100 (218 us / step measured). Per image the step is ~1 M FMA on ~100 KB of state,
// so the B200 mapping is: one CTA per image (100 CTAs on 148 SMs), FFMA with register strips
// (4 outputs per thread, a (4 + KW - 1)-wide input window slid along the row, taps broadcast from
// smem), and a deterministic cross-image reduction by the last CTA.
//
//   phase 0  v0 (global) and [K | bh | bv] -> smem; hs halo buffer zeroed
//   phase 1  h0 = sigmoid(conv_valid(v0, K) + bh), hs = (u < (double)h0) into the zero-padded halo
//   phase 2  v1 = sigmoid(conv over the padded hs with flipped, channel-transposed K + bv)
//   phase 3  h1 = sigmoid(conv_valid(v1, K) + bh)
//   phase 4  per-image partials: pos - neg per (f, c, di, dj), sum(h0 - h1) per f,
//            sum(v0 - v1) per c, sum((v0 - v1)^2) in double -> ws[img]
//   last CTA K / bh / bv += lr / B_global * sum_img partials (image order), recon = sum / B_global
//
// Accumulation orders of phases 1-3 are the oracle's (one fma chain over (c, di, dj) / (f, di, dj),
// oracle/fastnn_oracle.cpp conv_fwd / conv_bwd_data), so h0 / v1 / h1 differ from the reference only
// through expf; the statistics use per-lane chains + a fixed butterfly.
#pragma once
#include "runtime.cuh"

namespace b2n {

constexpr int kCfThreads = 512;

struct CrbmFusedParams {
    int C, H, W, K, KH, KW, OH, OW, HP;
    int VP, OP, HPP;     // smem row pitches (floats, multiples of 4) of v, h and the padded hs
    int B;               // images in this step
    int npart;           // floats per image partial row: K*CKK + K + C
    const float* v0;     // [B][C][H][W]
    const double* u;     // [B][K][OH][OW]
    float* P;            // [K (K,C,KH,KW) | bh (K) | bv (C)]
    float* ws;           // [B][npart] per-image partials
    double* rws;         // [B] per-image sum (v0 - v1)^2
    unsigned* ticket;    // CTAs finished (reset by the last one)
    double* recon;       // sum (v0 - v1)^2 / B_global
    float scale;         // lr / B_global
    long long stage_floats;  // smem floats after P available to stage the partials in the last CTA
    int ws_pitch;            // floats per partial row in ws (npart rounded up to 4)
    double inv_bg;
    // chain states of every image (for last_states / tests); null unless keep_states
    float *h0_out, *hs_out, *v1_out, *h1_out;
    unsigned long long* trace;  // bring-up timeline (B2N_TRACE=1, %globaltimer ns), null in production
    // data-parallel mode (non-null): the last CTA stores this shard's raw parameter sums and recon
    // sum here instead of updating P; crbm_dp_apply_kernel applies them after the allreduce
    float* G;
    double* Gd;
};
#define B2N_CF_TRACE(slot)                                                                \
    do {                                                                                  \
        if (p.trace && threadIdx.x == 0) p.trace[blockIdx.x * 64 + (slot)] = gtimer();    \
    } while (0)

// Row pitches: every 8-output strip reads its (8 + KW - 1)-wide input window as NV float4s (and
// the statistics pass 4-wide windows), so a row is padded until the last window fits; pads are zero
// (written once) and only feed outputs beyond the valid width, which are discarded.
constexpr int kCfStrip = 8;
struct CrbmPitches {
    int VP, OP, HPP;
};
inline CrbmPitches crbm_pitches(int W, int OW, int KW) {
    const int NV = (kCfStrip + KW - 1 + 3) / 4, NV4 = (4 + KW - 1 + 3) / 4;
    const int nsx1 = (OW + kCfStrip - 1) / kCfStrip, nsx2 = (W + kCfStrip - 1) / kCfStrip, WP = W + KW - 1;
    CrbmPitches q;
    q.VP = (int)round_up(std::max({W, kCfStrip * nsx1 - kCfStrip + 4 * NV, 4 * ((OW + 3) / 4) - 4 + 4 * NV4}), 4);
    q.OP = (int)round_up(OW, 4);
    q.HPP = (int)round_up(std::max(WP, kCfStrip * nsx2 - kCfStrip + 4 * NV), 4);
    return q;
}
inline long long crbm_stage_scratch(int C, int K, int KH, int KW) {
    return std::max<long long>(std::max<long long>(4096, 512LL * KW), (long long)K * C * KH * KW);
}
inline size_t crbm_fused_smem(int C, int H, int W, int K, int KH, int KW) {
    const int OH = H - KH + 1, OW = W - KW + 1, HP = OH + 2 * (KH - 1);
    const CrbmPitches q = crbm_pitches(W, OW, KW);
    const long long np = round_up((long long)K * C * KH * KW + K + C, 4);
    const long long fl = np + 2LL * K * C * KH * 8 + 2LL * C * H * q.VP + 2LL * K * OH * q.OP +
                         (long long)K * HP * q.HPP + crbm_stage_scratch(C, K, KH, KW);
    return (size_t)fl * 4 + 64 * 8;
}

__device__ __forceinline__ int rup4(int n) { return (n + 3) & ~3; }
__device__ __forceinline__ float sigmoid_f(float v) { return 1.0f / (1.0f + expf(-v)); }  // energy.hpp:36

// valid correlation of `in` (CI channels x IH rows, row pitch IP, smem) with taps into outputs
// (f, oy, ox) of F x OHh x OWw; each job owns a strip of 8 consecutive ox (adjacent lanes take
// adjacent strips: the float4 window loads are conflict-free). taps8 holds the taps of output f,
// input ci, row di at ((f*CI + ci)*KH + di)*8 (dj padded to 8; the phase-2 copy is already
// flipped and channel-transposed). With G > 1 the ci range is split over G jobs per strip
// (few-output phases): partial strips go to `part` and the caller runs conv_strips_finish after a
// barrier. `upre` (phase 1) prefetches the strip's Bernoulli uniforms before the product so their
// latency hides under it.
template <int KW, class Epi>
__device__ __forceinline__ void conv_strips(const float* __restrict__ in, int IP, int CI, int IH,
                                            const float* __restrict__ taps8, int F, int OHh, int OWw, int KH, int G,
                                            float* part, const double* upre, Epi epi) {
    constexpr int SW = kCfStrip;
    constexpr int NV = (SW + KW - 1 + 3) / 4;
    const int nsx = (OWw + SW - 1) / SW;
    const int total = F * OHh * nsx;
    for (int job = threadIdx.x; job < total * G; job += kCfThreads) {
        const int s = job % total, g = job / total;
        const int f = s / (OHh * nsx);
        const int rem = s - f * OHh * nsx;
        const int oy = rem / nsx;
        const int ox0 = (rem - oy * nsx) * SW;
        double uu[SW];
#pragma unroll
        for (int t = 0; t < SW; ++t) uu[t] = 0.0;
        if (upre) {
#pragma unroll
            for (int t = 0; t < SW; ++t)
                if (ox0 + t < OWw) uu[t] = upre[(f * OHh + oy) * OWw + ox0 + t];
        }
        float acc[SW];
#pragma unroll
        for (int t = 0; t < SW; ++t) acc[t] = 0.0f;
        const int ci0 = g * CI / G, ci1 = (g + 1) * CI / G;
        for (int ci = ci0; ci < ci1; ++ci) {
            const float* trow = taps8 + (f * CI + ci) * KH * 8;
            for (int di = 0; di < KH; ++di) {
                const float4* row = reinterpret_cast<const float4*>(in + (ci * IH + oy + di) * IP + ox0);
                float win[4 * NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const float4 q = row[v];
                    win[4 * v] = q.x;
                    win[4 * v + 1] = q.y;
                    win[4 * v + 2] = q.z;
                    win[4 * v + 3] = q.w;
                }
                const float4 k0 = *reinterpret_cast<const float4*>(trow + di * 8);
                const float4 k1 = *reinterpret_cast<const float4*>(trow + di * 8 + 4);
                const float kw[8] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
#pragma unroll
                for (int dj = 0; dj < KW; ++dj)
#pragma unroll
                    for (int t = 0; t < SW; ++t) acc[t] = fmaf(kw[dj], win[t + dj], acc[t]);
            }
        }
        if (G > 1) {
            float4* o = reinterpret_cast<float4*>(part + (g * total + s) * SW);
#pragma unroll
            for (int v = 0; v < SW / 4; ++v) o[v] = make_float4(acc[4 * v], acc[4 * v + 1], acc[4 * v + 2], acc[4 * v + 3]);
        } else {
            epi(f, oy, ox0, acc, uu, min(SW, OWw - ox0));
        }
    }
}
// the G partial strips summed in group order (one thread per strip), then the strip epilogue
template <class Epi>
__device__ __forceinline__ void conv_strips_finish(int F, int OHh, int OWw, int G, const float* part, Epi epi) {
    constexpr int SW = kCfStrip;
    const int nsx = (OWw + SW - 1) / SW;
    const int total = F * OHh * nsx;
    for (int s = threadIdx.x; s < total; s += kCfThreads) {
        const int f = s / (OHh * nsx), rem = s - f * OHh * nsx, oy = rem / nsx, ox0 = (rem - oy * nsx) * SW;
        float a[SW];
        const double uu[SW] = {};
#pragma unroll
        for (int t = 0; t < SW; ++t) a[t] = part[s * SW + t];
        for (int g = 1; g < G; ++g)
#pragma unroll
            for (int t = 0; t < SW; ++t) a[t] += part[(g * total + s) * SW + t];
        epi(f, oy, ox0, a, uu, min(SW, OWw - ox0));
    }
}

// n consecutive floats of a strip: two 16-byte stores when the strip is whole and aligned (the
// scalar form is an 8-way bank conflict: adjacent lanes own strips 8 floats apart)
__device__ __forceinline__ void store_strip(float* dst, const float* v, int n) {
    if (n == kCfStrip && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
    } else {
        for (int t = 0; t < n; ++t) dst[t] = v[t];
    }
}

template <int KW>
__global__ void __launch_bounds__(kCfThreads, 1) crbm_cd1_fused_kernel(const CrbmFusedParams p) {
    extern __shared__ __align__(16) float sm[];
    constexpr int NV = (KW + 3 + 3) / 4;
    const int C = p.C, H = p.H, W = p.W, K = p.K, KH = p.KH, OH = p.OH, OW = p.OW, HP = p.HP;
    const int VP = p.VP, OP = p.OP, HPP = p.HPP;
    const int CKK = C * KH * KW;
    const int HW = H * W, OHW = OH * OW;
    float* sP = sm;
    float* sK8 = sP + rup4(p.npart);       // taps K[f][c][di][0..8) (phases 1, 3)
    float* sKT8 = sK8 + K * C * KH * 8;    // taps K[k][c][KH-1-di][KW-1-dj] as [c][k][di][0..8) (phase 2)
    float* sv0 = sKT8 + K * C * KH * 8;
    float* sv1 = sv0 + C * H * VP;
    float* sh0 = sv1 + C * H * VP;
    float* sh1 = sh0 + K * OH * OP;
    float* shp = sh1 + K * OH * OP;
    double* sred = reinterpret_cast<double*>(shp + K * HP * HPP);
    float* sst = reinterpret_cast<float*>(sred + 64);  // phase-2 / phase-4a partials
    __shared__ unsigned s_last;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int NW = kCfThreads / 32;

    B2N_CF_TRACE(0);
    {  // zero the image buffers once: row pads and the hs halo border are never written again
        float4* z = reinterpret_cast<float4*>(sv0);
        const int n4 = (2 * C * H * VP + 2 * K * OH * OP + K * HP * HPP) / 4;
        for (int i = tid; i < n4; i += kCfThreads) z[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    }
    pdl_wait();  // P is updated by the previous step's last CTA
    for (int i = tid; i < p.npart; i += kCfThreads) sP[i] = p.P[i];
    __syncthreads();
    for (int i = tid; i < K * C * KH * 8; i += kCfThreads) {
        const int dj = i & 7, r = i >> 3, di = r % KH, fc = r / KH;  // fc = f*C + c
        sK8[i] = dj < KW ? sP[r * KW + dj] : 0.0f;
        const int c2 = fc / K, k2 = fc % K;  // sKT8 row (c2, k2, di) <- K[k2][c2][KH-1-di][KW-1-dj]
        sKT8[i] = dj < KW ? sP[((k2 * C + c2) * KH + (KH - 1 - di)) * KW + (KW - 1 - dj)] : 0.0f;
    }
    B2N_CF_TRACE(1);
    const float* sbh = sP + K * CKK;
    const float* sbv = sbh + K;

    for (int img = blockIdx.x; img < p.B; img += gridDim.x) {
        const float* gv0 = p.v0 + (long long)img * C * HW;
        const double* gu = p.u + (long long)img * K * OHW;
        for (int i = tid; i < C * HW; i += kCfThreads) {
            const int r = i / W;
            sv0[r * VP + (i - r * W)] = gv0[i];
        }
        __syncthreads();
        B2N_CF_TRACE(2);
        // phase 1: hidden means + samples (crbm_hidden_preact + unit_mean / unit_sample)
        conv_strips<KW>(sv0, VP, C, H, sK8, K, OH, OW, KH, 1, sst, gu,
                        [&](int f, int oy, int ox0, const float* a, const double* uv, int n) {
            float pr[kCfStrip], hs[kCfStrip];
#pragma unroll
            for (int t = 0; t < kCfStrip; ++t) {
                pr[t] = sigmoid_f(a[t] + sbh[f]);
                hs[t] = uv[t] < (double)pr[t] ? 1.0f : 0.0f;
            }
            store_strip(sh0 + (f * OH + oy) * OP + ox0, pr, n);
            store_strip(shp + (f * HP + oy + KH - 1) * HPP + ox0 + KW - 1, hs, n);
        });
        __syncthreads();
        B2N_CF_TRACE(3);
        // phase 2: visible means from the sample (crbm_visible_preact: full conv, K^T); few
        // outputs, so the hidden-map sum is split over G jobs per strip
        {
            auto epi2 = [&](int c, int y, int ox0, const float* a, const double*, int n) {
                float v[kCfStrip];
#pragma unroll
                for (int t = 0; t < kCfStrip; ++t) v[t] = sigmoid_f(a[t] + sbv[c]);
                store_strip(sv1 + (c * H + y) * VP + ox0, v, n);
            };
            const int strips2 = C * H * ((W + kCfStrip - 1) / kCfStrip);
            const int G2 = max(1, min(K, kCfThreads / strips2));
            conv_strips<KW>(shp, HPP, K, HP, sKT8, C, H, W, KH, G2, sst, nullptr, epi2);
            if (G2 > 1) {
                __syncthreads();
                conv_strips_finish(C, H, W, G2, sst, epi2);
            }
        }
        __syncthreads();
        B2N_CF_TRACE(4);
        // phase 3: hidden means of the reconstruction
        conv_strips<KW>(sv1, VP, C, H, sK8, K, OH, OW, KH, 1, sst, nullptr,
                        [&](int f, int oy, int ox0, const float* a, const double*, int n) {
            float v[kCfStrip];
#pragma unroll
            for (int t = 0; t < kCfStrip; ++t) v[t] = sigmoid_f(a[t] + sbh[f]);
            store_strip(sh1 + (f * OH + oy) * OP + ox0, v, n);
        });
        __syncthreads();
        B2N_CF_TRACE(5);
        // phase 4a: correlation statistics pos - neg (crbm_corr_stats). Thread = (f, c, di) x a
        // segment of the output rows; KW pos / neg accumulators, the v windows slid along the row
        // (4 outputs per step, zero pads past OW), segments summed in order below.
        float* wrow = p.ws + (long long)img * p.ws_pitch;
        {
            const int T = K * C * KH;
            const int S = max(1, min(OH, kCfThreads / T));
            for (int job = tid; job < T * S; job += kCfThreads) {
                const int tup = job / S, seg = job - tup * S;
                const int f = tup / (C * KH), r = tup - f * C * KH, c = r / KH, di = r - c * KH;
                float pos[KW], neg[KW];
#pragma unroll
                for (int dj = 0; dj < KW; ++dj) pos[dj] = neg[dj] = 0.0f;
                for (int oy = seg; oy < OH; oy += S) {
                    const float* r0 = sv0 + (c * H + oy + di) * VP;
                    const float* r1 = sv1 + (c * H + oy + di) * VP;
                    const float* g0 = sh0 + (f * OH + oy) * OP;
                    const float* g1 = sh1 + (f * OH + oy) * OP;
                    for (int ox0 = 0; ox0 < OW; ox0 += 4) {
                        const float4 a0 = *reinterpret_cast<const float4*>(g0 + ox0);
                        const float4 a1 = *reinterpret_cast<const float4*>(g1 + ox0);
                        const float av0[4] = {a0.x, a0.y, a0.z, a0.w}, av1[4] = {a1.x, a1.y, a1.z, a1.w};
                        float w0[4 * NV], w1[4 * NV];
#pragma unroll
                        for (int v = 0; v < NV; ++v) {
                            const float4 q0 = *reinterpret_cast<const float4*>(r0 + ox0 + 4 * v);
                            const float4 q1 = *reinterpret_cast<const float4*>(r1 + ox0 + 4 * v);
                            w0[4 * v] = q0.x;
                            w0[4 * v + 1] = q0.y;
                            w0[4 * v + 2] = q0.z;
                            w0[4 * v + 3] = q0.w;
                            w1[4 * v] = q1.x;
                            w1[4 * v + 1] = q1.y;
                            w1[4 * v + 2] = q1.z;
                            w1[4 * v + 3] = q1.w;
                        }
#pragma unroll
                        for (int dj = 0; dj < KW; ++dj)
#pragma unroll
                            for (int t = 0; t < 4; ++t) {
                                pos[dj] = fmaf(w0[t + dj], av0[t], pos[dj]);
                                neg[dj] = fmaf(w1[t + dj], av1[t], neg[dj]);
                            }
                    }
                }
#pragma unroll
                for (int dj = 0; dj < KW; ++dj) sst[(tup * S + seg) * KW + dj] = pos[dj] - neg[dj];
            }
            __syncthreads();
            for (int o = tid; o < T * KW; o += kCfThreads) {  // o = ((f*C + c)*KH + di)*KW + dj
                const int tup = o / KW, dj = o - tup * KW;
                float a = 0.0f;
                for (int seg = 0; seg < S; ++seg) a += sst[(tup * S + seg) * KW + dj];
                wrow[o] = a;
            }
        }
        // phase 4b: bias sums and the reconstruction error, one warp per hidden map / channel
        // (whole pitched planes: the pads are zero on both sides)
        for (int t = warp; t < K + C; t += NW) {
            if (t < K) {
                const float* a = sh0 + t * OH * OP;
                const float* b = sh1 + t * OH * OP;
                float s = 0.0f;
                for (int q = lane; q < OH * OP; q += 32) s += a[q] - b[q];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0) wrow[K * CKK + t] = s;
            } else {
                const int c = t - K;
                const float* a = sv0 + c * H * VP;
                const float* b = sv1 + c * H * VP;
                float s = 0.0f;
                double d2 = 0.0;
                for (int q = lane; q < H * VP; q += 32) {
                    const float x0 = a[q], x1 = b[q];
                    s += x0 - x1;
                    const double e = (double)x0 - (double)x1;
                    d2 += e * e;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    s += __shfl_xor_sync(0xffffffffu, s, o);
                    d2 += __shfl_xor_sync(0xffffffffu, d2, o);
                }
                if (lane == 0) {
                    wrow[K * CKK + t] = s;
                    sred[c] = d2;
                }
            }
        }
        B2N_CF_TRACE(6);
        if (p.h0_out) {  // chain states for last_states (tests / debugging)
            for (int i = tid; i < K * OHW; i += kCfThreads) {
                const int f = i / OHW, q = i - f * OHW, oy = q / OW, ox = q - oy * OW;
                const long long g = (long long)img * K * OHW + i;
                p.h0_out[g] = sh0[(f * OH + oy) * OP + ox];
                p.h1_out[g] = -sh1[(f * OH + oy) * OP + ox];  // the split path's layout (stored negated)
                p.hs_out[g] = shp[(f * HP + oy + KH - 1) * HPP + ox + KW - 1];
            }
            for (int i = tid; i < C * HW; i += kCfThreads) {
                const int r = i / W;
                p.v1_out[(long long)img * C * HW + i] = sv1[r * VP + (i - r * W)];
            }
        }
        __syncthreads();
        if (tid == 0) {
            double r = 0.0;
            for (int c = 0; c < C; ++c) r += sred[c];
            p.rws[img] = r;
        }
        __syncthreads();
    }
    // the last CTA to finish reduces the per-image partials in image order and updates P
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        s_last = atomicAdd(p.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    B2N_CF_TRACE(7);
    if (!s_last) return;
    __threadfence();
    const long long nws = (long long)p.B * p.ws_pitch;
    if (nws <= p.stage_floats) {
        // stage every image's partial row in shared memory with independent coalesced loads
        // (the image buffers are dead now), then sum each parameter's column in image order
        float* st = sm + rup4(p.npart);
        const int n4 = (int)(nws / 4);  // rows padded to ws_pitch (a multiple of 4)
        const float4* src = reinterpret_cast<const float4*>(p.ws);
        float4* dst = reinterpret_cast<float4*>(st);
        for (int i0 = tid; i0 < n4; i0 += 8 * kCfThreads) {  // 8 independent 16-byte loads in flight
            float4 t8[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int i = i0 + q * kCfThreads;
                t8[q] = i < n4 ? __ldcg(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int i = i0 + q * kCfThreads;
                if (i < n4) dst[i] = t8[q];
            }
        }
        __syncthreads();
        B2N_CF_TRACE(8);
        for (int i = tid; i < p.npart; i += kCfThreads) {
            float s = 0.0f;
            for (int img = 0; img < p.B; ++img) s += st[(long long)img * p.ws_pitch + i];
            if (p.G) p.G[i] = s;
            else p.P[i] = sP[i] + p.scale * s;
        }
    } else {
        for (int i = tid; i < p.npart; i += kCfThreads) {
            float s = 0.0f;
            for (int img = 0; img < p.B; ++img) s += __ldcg(p.ws + (long long)img * p.ws_pitch + i);
            if (p.G) p.G[i] = s;
            else p.P[i] = sP[i] + p.scale * s;
        }
    }
    if (tid < 32) {  // recon: lane-strided image sums + a fixed butterfly
        double r = 0.0;
        for (int img = tid; img < p.B; img += 32) r += __ldcg(p.rws + img);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
        if (tid == 0) {
            if (p.Gd) *p.Gd = r;
            else *p.recon = r * p.inv_bg;
            *p.ticket = 0u;
        }
    }
    __syncthreads();
    B2N_CF_TRACE(9);
}

// data-parallel CRBM step: P += lr / B_global * (allreduced parameter sums), recon = sum / B_global
static __global__ void crbm_dp_apply_kernel(float* __restrict__ P, const float* __restrict__ G, int n, float scale,
                                            const double* __restrict__ Gd, double* recon, double inv_bg) {
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) P[i] += scale * G[i];
    if (i == 0) *recon = *Gd * inv_bg;
}

}  // namespace b2n
