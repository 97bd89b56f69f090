// gemm_tc.cuh -- the tcgen05 tensor-core GEMM with fused training-step epilogues.
//
// D[M x N] = op(A)[M x K] . op(B)[K x N], fp32 in HBM, computed as 3xTF32 (a = a_hi + a_lo split in
// shared memory; D += a_lo.b_hi + a_hi.b_lo + a_hi.b_hi) so results track the reference's fp32
// arithmetic (gemm.hpp:30-125) to ~1e-6; a 1xTF32 instantiation exists for the fast mode.
//
// Structure (one 128 x BN output tile per CTA, 6 warps):
//   warp 0      : TMA producer  (cp.async.bulk.tensor, SWIZZLE_128B boxes, mbarrier expect_tx)
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer (commit -> smem slot release)
//   warps 2..5  : 3xTF32 hi/lo splitters for each landed stage, then the epilogue
//                 (tcgen05.ld TMEM -> registers -> fused bias / activation / softmax-xent /
//                  SGD-momentum / RBM sampling -> global)
// Operands may be K-major (row-major [rows][K], "NT" side) or MN-major (row-major [K][rows], the
// transposed side of the reference's NN / TN calls); both are legal UMMA layouts for kind::tf32,
// so no transpose pass is ever run. TMA zero-fills out-of-bounds boxes, which pads M, N and K.
#pragma once
#include "ptx.cuh"

namespace b2n {

enum EpiKind : int {
    EPI_STORE = 0,         // C = alpha * acc
    EPI_BIAS_ACT = 1,      // C = act(acc + bias[n])                          dense_forward + activation_apply
    EPI_DACT = 2,          // C = acc * act'(aux[m,n])                        dense_backward dx + activation_gradient
    EPI_SOFTMAX_XENT = 3,  // logits=acc+bias; probs, dlogits=(p-y)/B, loss, argmax   softmax + softmax_cross_entropy
    EPI_SGD = 4,           // grad=acc; v = mom*v - lr*(g + wd*p); p += v     dense_backward gw + sgd_momentum_step
    EPI_RBM_HID = 5,       // p = sigmoid(acc+bias); C = p; C2 = (u < p)      rbm_hidden_given_visible (+sample)
    EPI_RBM_VIS = 6,       // p = sigmoid(acc+bias); C = p; row partial sum (aux - p)^2   + sq_diff_per_row
    EPI_RBM_NEGHID = 7,    // C = -sigmoid(acc + bias)                        negative-phase hidden means
    EPI_AXPY = 8,          // C += alpha * acc                                 W += lr/B (pos - neg)
};
enum ActKind : int { ACT_NONE = 0, ACT_SIGMOID = 1, ACT_RELU = 2 };

struct EpiParams {
    float* C;
    long long ldc;
    const float* bias;
    long long bias_stride;
    int act;
    const float* aux;
    long long ld_aux;
    float alpha;
    // softmax / xent
    const int* labels;
    float batch_div;  // dlogits divisor (float)B_global, network.hpp:430
    double* row_loss;
    int* argmax;
    float* probs;
    long long ld_probs;
    // sgd
    float* V;
    long long ldv;
    float lr, mom, wd;
    // rbm
    const double* u;
    long long ldu;
    float* C2;
    long long ldc2;
    double* row_part;
    long long ld_part;
};

struct GemmParams {
    int M, N, K;
    int a_mn, b_mn;  // 1 = MN-major operand (row-major [K][rows])
    int epi;
    EpiParams ep;
};

constexpr int kBM = 128;
constexpr int kBK = 32;  // 32 fp32 = one 128-byte swizzle row
constexpr int kThreads = 192;

template <int BN, bool X3>
struct GemmCfg {
    static constexpr int A_BYTES = kBM * kBK * 4;
    static constexpr int B_BYTES = BN * kBK * 4;
    static constexpr int STAGE_BYTES = (A_BYTES + B_BYTES) * (X3 ? 2 : 1);
    static constexpr int STAGES_FIT = (200 * 1024) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_FIT > 4 ? 4 : STAGES_FIT;
    static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
    static_assert(STAGES >= 2, "tile too large");
};

__device__ __forceinline__ float sigmoid_ref(float v) { return 1.0f / (1.0f + expf(-v)); }  // layers.hpp:279

__device__ __forceinline__ float apply_act(int act, float v) {
    if (act == ACT_SIGMOID) return sigmoid_ref(v);
    if (act == ACT_RELU) return v > 0.0f ? v : 0.0f;
    return v;
}

// 3xTF32 split of one landed tile: hi (truncated to tf32) in place, lo = x - hi to the lo slot.
__device__ __forceinline__ void split_tile(uint8_t* hi, uint8_t* lo, int bytes, int tid, int nthreads) {
    float4* h = reinterpret_cast<float4*>(hi);
    float4* l = reinterpret_cast<float4*>(lo);
    for (int i = tid; i < bytes / 16; i += nthreads) {
        float4 x = h[i];
        float4 a, b;
        a.x = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
        a.y = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
        a.z = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
        a.w = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
        b.x = x.x - a.x;
        b.y = x.y - a.y;
        b.z = x.z - a.z;
        b.w = x.w - a.w;
        h[i] = a;
        l[i] = b;
    }
}

template <int BN>
__device__ __forceinline__ void gemm_epilogue(const GemmParams& p, uint32_t tmem_row, int m, int n0) {
    const EpiParams& e = p.ep;
    const bool mok = m < p.M;
    if (p.epi == EPI_SOFTMAX_XENT) {
        // whole row lives in this thread (host guarantees N <= BN, one N tile). softmax
        // (layers.hpp:301-320) then softmax_cross_entropy (network.hpp:410-437), sequential in j.
        float mx = -INFINITY;
        for (int c = 0; c < BN; c += 16) {
            float v[16];
            tmem_ld16(tmem_row + c, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int n = c + i;
                if (n < p.N) mx = fmaxf(mx, v[i] + e.bias[(long long)n * e.bias_stride]);
            }
        }
        float sum = 0.0f;
        for (int c = 0; c < BN; c += 16) {
            float v[16];
            tmem_ld16(tmem_row + c, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int n = c + i;
                if (n < p.N) sum += expf((v[i] + e.bias[(long long)n * e.bias_stride]) - mx);
            }
        }
        const int label = mok ? e.labels[m] : 0;
        int best = 0;
        float bestp = -1.0f;
        float ptrue = 0.0f;
        for (int c = 0; c < BN; c += 16) {
            float v[16];
            tmem_ld16(tmem_row + c, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int n = c + i;
                if (n < p.N && mok) {
                    const float q = expf((v[i] + e.bias[(long long)n * e.bias_stride]) - mx) / sum;
                    if (q > bestp) {  // strict >: first maximum wins (network.hpp:69-70)
                        bestp = q;
                        best = n;
                    }
                    if (n == label) ptrue = q;
                    const float y = n == label ? 1.0f : 0.0f;
                    e.C[(long long)m * e.ldc + n] = (q - y) / e.batch_div;
                    if (e.probs) e.probs[(long long)m * e.ld_probs + n] = q;
                }
            }
        }
        if (mok) {
            e.row_loss[m] = -log(fmax((double)ptrue, 1e-300));
            if (e.argmax) e.argmax[m] = best;
        }
        return;
    }
    double part = 0.0;
    for (int c = 0; c < BN; c += 16) {
        float v[16];
        tmem_ld16(tmem_row + c, v);
        if (!mok) continue;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int n = n0 + c + i;
            if (n >= p.N) break;
            const float a = v[i];
            const long long mn = (long long)m * e.ldc + n;
            switch (p.epi) {
                case EPI_STORE: e.C[mn] = e.alpha * a; break;
                case EPI_BIAS_ACT: e.C[mn] = apply_act(e.act, a + e.bias[(long long)n * e.bias_stride]); break;
                case EPI_DACT: {
                    const float y = e.aux[(long long)m * e.ld_aux + n];
                    e.C[mn] = e.act == ACT_SIGMOID ? a * y * (1.0f - y) : (y > 0.0f ? a : 0.0f);
                    break;
                }
                case EPI_SGD: {  // optim.hpp:75-78
                    float* pp = e.C + mn;
                    float* vv = e.V + (long long)m * e.ldv + n;
                    const float g = a + e.wd * *pp;
                    const float vel = e.mom * *vv - e.lr * g;
                    *vv = vel;
                    *pp = *pp + vel;
                    break;
                }
                case EPI_RBM_HID: {  // energy.hpp:101-110 + unit_sample_inplace :59-61
                    const float pr = sigmoid_ref(a + e.bias[(long long)n * e.bias_stride]);
                    e.C[mn] = pr;
                    e.C2[(long long)m * e.ldc2 + n] = (e.u[(long long)m * e.ldu + n] < (double)pr) ? 1.0f : 0.0f;
                    break;
                }
                case EPI_RBM_VIS: {
                    const float pr = sigmoid_ref(a + e.bias[(long long)n * e.bias_stride]);
                    e.C[mn] = pr;
                    const double d = (double)e.aux[(long long)m * e.ld_aux + n] - (double)pr;
                    part += d * d;
                    break;
                }
                case EPI_RBM_NEGHID: e.C[mn] = -sigmoid_ref(a + e.bias[(long long)n * e.bias_stride]); break;
                case EPI_AXPY: e.C[mn] = e.C[mn] + e.alpha * a; break;
                default: break;
            }
        }
    }
    if (p.epi == EPI_RBM_VIS && mok) e.row_part[(long long)blockIdx.x * e.ld_part + m] = part;
}

template <int BN, bool X3>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const GemmParams p) {
    using Cfg = GemmCfg<BN, X3>;
    constexpr int S = Cfg::STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::STAGE_BYTES);
    uint64_t* ready = full + S;
    uint64_t* empty = ready + S;
    uint64_t* tmem_full = empty + S;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * BN;
    const int num_kb = (p.K + kBK - 1) / kBK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&ready[s], 128);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        fence_barrier_init();
        tma_prefetch(&mapA);
        tma_prefetch(&mapB);
    }
    if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % S;
                const uint32_t ph = (kb / S) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t* a = smem + s * Cfg::STAGE_BYTES;
                uint8_t* b = a + Cfg::A_BYTES;
                mbar_arrive_expect_tx(&full[s], Cfg::A_BYTES + Cfg::B_BYTES);
                const int k0 = kb * kBK;
                if (!p.a_mn) {
                    tma_load_2d(a, &mapA, &full[s], k0, m0);
                } else {
#pragma unroll
                    for (int j = 0; j < kBM / 32; ++j) tma_load_2d(a + j * 4096, &mapA, &full[s], m0 + 32 * j, k0);
                }
                if (!p.b_mn) {
                    tma_load_2d(b, &mapB, &full[s], k0, n0);
                } else {
#pragma unroll
                    for (int j = 0; j < BN / 32; ++j) tma_load_2d(b + j * 4096, &mapB, &full[s], n0 + 32 * j, k0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            const uint32_t idesc = umma_idesc_tf32(kBM, BN, p.a_mn, p.b_mn);
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % S;
                const uint32_t ph = (kb / S) & 1;
                mbar_wait(X3 ? &ready[s] : &full[s], ph);
                tc_fence_after();
                const uint32_t a_hi = smem_u32(smem + s * Cfg::STAGE_BYTES);
                const uint32_t b_hi = a_hi + Cfg::A_BYTES;
                const uint32_t a_lo = b_hi + Cfg::B_BYTES;
                const uint32_t b_lo = a_lo + Cfg::A_BYTES;
#pragma unroll
                for (int kk = 0; kk < kBK / 8; ++kk) {
                    const uint64_t dah = p.a_mn ? desc_mnmajor(a_hi, kk) : desc_kmajor(a_hi, kk);
                    const uint64_t dbh = p.b_mn ? desc_mnmajor(b_hi, kk) : desc_kmajor(b_hi, kk);
                    const uint32_t acc = (kb | kk) != 0;
                    if (X3) {
                        const uint64_t dal = p.a_mn ? desc_mnmajor(a_lo, kk) : desc_kmajor(a_lo, kk);
                        const uint64_t dbl = p.b_mn ? desc_mnmajor(b_lo, kk) : desc_kmajor(b_lo, kk);
                        mma_tf32(tmem_base, dal, dbh, idesc, acc);
                        mma_tf32(tmem_base, dah, dbl, idesc, 1);
                        mma_tf32(tmem_base, dah, dbh, idesc, 1);
                    } else {
                        mma_tf32(tmem_base, dah, dbh, idesc, acc);
                    }
                }
                mma_commit(&empty[s]);
            }
            mma_commit(tmem_full);
        }
    } else {  // ---------------- splitters + epilogue (warps 2..5)
        const int ct = threadIdx.x - 64;
        if (X3) {
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % S;
                const uint32_t ph = (kb / S) & 1;
                mbar_wait(&full[s], ph);
                uint8_t* a = smem + s * Cfg::STAGE_BYTES;
                split_tile(a, a + Cfg::A_BYTES + Cfg::B_BYTES, Cfg::A_BYTES, ct, 128);
                split_tile(a + Cfg::A_BYTES, a + 2 * Cfg::A_BYTES + Cfg::B_BYTES, Cfg::B_BYTES, ct, 128);
                fence_proxy_async_smem();
                mbar_arrive(&ready[s]);
            }
        }
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const int q = warp & 3;  // TMEM lane quadrant this warp may access
        const int row = 32 * q + lane;
        gemm_epilogue<BN>(p, tmem_base + ((uint32_t)(32 * q) << 16), m0 + row, n0);
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
}

}  // namespace b2n
