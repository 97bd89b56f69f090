// gemm_tc.cuh -- the tcgen05 tensor-core GEMM with fused training-step epilogues.
//
// D[M x N] = op(A)[M x K] . op(B)[K x N], fp32 in HBM, computed as 3xTF32 so results track the
// reference's fp32 arithmetic (gemm.hpp:30-125) to ~1e-6: kind::tf32 truncates each fp32 operand
// to tf32 (measured on B200), so the TMA-landed raw tile IS the hi part; splitter warps write only
// lo = x - trunc(x), and D += a_lo.b + a.b_lo + a.b. A 1xTF32 instantiation is the fast mode.
//
// One 128 x BN output tile per CTA (or per cluster of `splits` CTAs, split-K), 10 warps:
//   warp 0      : TMA producer (cp.async.bulk.tensor into 128 B-swizzled smem, mbarrier expect_tx)
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer (tcgen05.commit frees a stage)
//   warps 2..9  : lo splitters for each landed stage, then TMEM -> smem tile (tcgen05.ld)
//   all warps   : split-K reduction (partials through an L2 workspace, cluster barrier, each CTA of
//                 the cluster reduces a row slice in fixed split order -> deterministic) and the fused
//                 epilogue on coalesced float4 rows: bias / activation / act' / SGD-momentum /
//                 RBM sampling / W += lr/B (pos - neg); softmax-xent row-wise.
// Operands may be K-major (row-major [rows][K]) or MN-major (row-major [K][rows], the transposed
// side of the reference's NN / TN calls), both legal UMMA layouts for kind::tf32, so no transpose
// pass ever runs. TMA zero-fills out-of-bounds boxes, which pads M, N and K.
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
    int splits;      // split-K factor == cluster size along z
    int kb_per_split;
    int pre_a, pre_b;  // operand not written by the preceding kernel: TMA it before griddepcontrol.wait
    float* ws;       // split-K partial tiles [tile][split][128][BN]
    EpiParams ep;
    unsigned long long* trace;  // bring-up timeline (%globaltimer ns), null in production
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// slots per CTA: 0 start, 1 setup done, 2+kb TMA issue (kb<16), 18+kb stage landed (kb<16),
// 34+kb mma issued (kb<16), 50 last commit, 51 epilogue start, 52 end, 53 tile in smem, 54 partial
// written, 55 cluster barrier passed, 56 reduced, 57 epilogue done
#define B2N_TRACE(slot)                                                                                          \
    do {                                                                                                         \
        if (p.trace && (slot) < 64)                                                                              \
            p.trace[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 64 + (slot)] = gtimer(); \
    } while (0)

constexpr int kBM = 128;
constexpr int kBK = 32;  // 32 fp32 = one 128-byte swizzle row
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;  // 320

template <int BN, bool X3>
struct GemmCfg {
    static constexpr int A_BYTES = kBM * kBK * 4;
    static constexpr int B_BYTES = BN * kBK * 4;
    static constexpr int STAGE_BYTES = (A_BYTES + B_BYTES) * (X3 ? 2 : 1);
    static constexpr int STAGES_FIT = (200 * 1024) / STAGE_BYTES;
    static constexpr int STAGES = STAGES_FIT > 6 ? 6 : STAGES_FIT;
    // 3xTF32 with BN <= 128 stacks B hi | B lo along N: one MMA (N = 2 BN) gives a_hi.b_hi in columns
    // [0, BN) and a_hi.b_lo in [BN, 2 BN), a second adds a_lo.b_hi to [0, BN): 2 MMAs per K step, not 3
    static constexpr bool STACK = X3 && BN <= 128;
    static constexpr int ACC_COLS = STACK ? 2 * BN : BN;
    static constexpr int TMEM_COLS = ACC_COLS <= 32 ? 32 : ACC_COLS <= 64 ? 64 : ACC_COLS <= 128 ? 128 : 256;
    static constexpr int TP = BN + 4;  // padded smem tile pitch (floats): conflict-free row writes
    static constexpr int TILE_BYTES = kBM * TP * 4;
    static constexpr int MAIN_BYTES = STAGES * STAGE_BYTES > TILE_BYTES ? STAGES * STAGE_BYTES : TILE_BYTES;
    static constexpr int SMEM = MAIN_BYTES + 1024 + 256;
    static_assert(STAGES >= 2, "tile too large");
};

// layers.hpp:279. The tensor-core products feeding it differ from the reference's fp32 sums at ~1e-6,
// so CUDA's expf (<= 2 ulp) costs nothing in accuracy here; the bit-exact paths (convx.cuh forward,
// ops.cu) use glibc_expf
__device__ __forceinline__ float sigmoid_ref(float v) { return 1.0f / (1.0f + expf(-v)); }

__device__ __forceinline__ float apply_act(int act, float v) {
    if (act == ACT_SIGMOID) return sigmoid_ref(v);
    if (act == ACT_RELU) return v > 0.0f ? v : 0.0f;
    return v;
}

// lo = x - trunc_tf32(x) of one landed tile (the raw tile doubles as the hi operand)
__device__ __forceinline__ void split_lo(const uint8_t* raw, uint8_t* lo, int bytes, int tid, int nthreads) {
    const uint32_t r = smem_u32(raw), l = smem_u32(lo);
#pragma unroll 4
    for (int i = tid * 16; i < bytes; i += nthreads * 16) {
        float x0, x1, x2, x3;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x0), "=f"(x1), "=f"(x2), "=f"(x3) : "r"(r + i));
        const float y0 = x0 - __uint_as_float(__float_as_uint(x0) & 0xFFFFE000u);
        const float y1 = x1 - __uint_as_float(__float_as_uint(x1) & 0xFFFFE000u);
        const float y2 = x2 - __uint_as_float(__float_as_uint(x2) & 0xFFFFE000u);
        const float y3 = x3 - __uint_as_float(__float_as_uint(x3) & 0xFFFFE000u);
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(l + i), "f"(y0), "f"(y1), "f"(y2), "f"(y3)
                     : "memory");
    }
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// 4 consecutive columns of one row: vector access when the row pitch and column allow it
__device__ __forceinline__ bool vec_ok(const void* base, long long ld, int n, int N) {
    return n + 3 < N && (ld & 3) == 0 && ((reinterpret_cast<uintptr_t>(base) & 15) == 0);
}

// Epilogue inputs of 4 columns [n, n+4) of row m that do not depend on the product.
struct EpiIn {
    float4 a, b;  // aux / C / V rows
    double u[4];  // RBM sampling uniforms
};
constexpr int kEpiPrefetch = 4;  // iterations whose inputs are loaded before the split-K exchange

__device__ __forceinline__ float4 ld4(const float* base, long long ld, int m, int n, int N) {
    const long long o = (long long)m * ld + n;
    if (vec_ok(base, ld, n, N)) return *reinterpret_cast<const float4*>(base + o);
    float t[4] = {0.f, 0.f, 0.f, 0.f};
    for (int i = 0; i < 4 && n + i < N; ++i) t[i] = base[o + i];
    return make_float4(t[0], t[1], t[2], t[3]);
}

// bias of the thread's 4 columns (constant over its tile rows)
template <int EPI>
__device__ __forceinline__ void epi_bias(const GemmParams& p, int n, float (&b)[4]) {
    const EpiParams& e = p.ep;
    if (EPI == EPI_BIAS_ACT || EPI == EPI_RBM_HID || EPI == EPI_RBM_VIS || EPI == EPI_RBM_NEGHID)
        for (int i = 0; i < 4; ++i) b[i] = n + i < p.N ? e.bias[(long long)(n + i) * e.bias_stride] : 0.0f;
}

template <int EPI>
__device__ __forceinline__ void epi_load(const GemmParams& p, int m, int n, EpiIn& in) {
    const EpiParams& e = p.ep;
    switch (EPI) {
        case EPI_DACT: in.a = ld4(e.aux, e.ld_aux, m, n, p.N); break;
        case EPI_SGD: in.a = ld4(e.C, e.ldc, m, n, p.N); in.b = ld4(e.V, e.ldv, m, n, p.N); break;
        case EPI_AXPY: in.a = ld4(e.C, e.ldc, m, n, p.N); break;
        case EPI_RBM_VIS: in.a = ld4(e.aux, e.ld_aux, m, n, p.N); break;
        case EPI_RBM_HID:
            for (int i = 0; i < 4; ++i) in.u[i] = n + i < p.N ? e.u[(long long)m * e.ldu + n + i] : 2.0;
            break;
        default: break;
    }
}

// elementwise epilogue on 4 columns [n, n+4) of row m (values v); returns the row partial for RBM_VIS
template <int EPI>
__device__ __forceinline__ double epi_apply(const GemmParams& p, int m, int n, const float (&v)[4],
                                            const float (&bias)[4], const EpiIn& in) {
    const EpiParams& e = p.ep;
    const int cnt = p.N - n < 4 ? p.N - n : 4;
    const long long row = (long long)m * e.ldc;
    double part = 0.0;
    auto st4 = [&](float* base, long long ld, const float (&o)[4]) {
        if (vec_ok(base, ld, n, p.N))
            *reinterpret_cast<float4*>(base + (long long)m * ld + n) = make_float4(o[0], o[1], o[2], o[3]);
        else
            for (int i = 0; i < cnt; ++i) base[(long long)m * ld + n + i] = o[i];
    };
    const float a[4] = {in.a.x, in.a.y, in.a.z, in.a.w}, b[4] = {in.b.x, in.b.y, in.b.z, in.b.w};
    switch (EPI) {
        case EPI_STORE: {
            const float o[4] = {e.alpha * v[0], e.alpha * v[1], e.alpha * v[2], e.alpha * v[3]};
            st4(e.C, e.ldc, o);
            break;
        }
        case EPI_BIAS_ACT: {  // dense_forward + activation_apply
            float o[4];
            for (int i = 0; i < 4; ++i) o[i] = apply_act(e.act, v[i] + bias[i]);
            st4(e.C, e.ldc, o);
            break;
        }
        case EPI_DACT: {  // layers.hpp:294 order: dy * y * (1 - y)
            float o[4];
            for (int i = 0; i < 4; ++i)
                o[i] = e.act == ACT_SIGMOID ? v[i] * a[i] * (1.0f - a[i]) : (a[i] > 0.0f ? v[i] : 0.0f);
            st4(e.C, e.ldc, o);
            break;
        }
        case EPI_SGD: {  // optim.hpp:75-78 on (w | b) tiles
            float pp[4], vv[4];
            for (int i = 0; i < 4; ++i) {
                const float g = v[i] + e.wd * a[i];
                vv[i] = e.mom * b[i] - e.lr * g;
                pp[i] = a[i] + vv[i];
            }
            st4(e.C, e.ldc, pp);
            st4(e.V, e.ldv, vv);
            break;
        }
        case EPI_RBM_HID: {  // energy.hpp:101-110 + unit_sample_inplace :59-61
            float pr[4], hs[4];
            for (int i = 0; i < 4; ++i) {
                pr[i] = sigmoid_ref(v[i] + bias[i]);
                hs[i] = (in.u[i] < (double)pr[i]) ? 1.0f : 0.0f;
            }
            st4(e.C, e.ldc, pr);
            st4(e.C2, e.ldc2, hs);
            break;
        }
        case EPI_RBM_VIS: {
            float pr[4];
            for (int i = 0; i < 4; ++i) pr[i] = sigmoid_ref(v[i] + bias[i]);
            for (int i = 0; i < cnt; ++i) {
                const double d = (double)a[i] - (double)pr[i];
                part += d * d;
            }
            st4(e.C, e.ldc, pr);
            break;
        }
        case EPI_RBM_NEGHID: {
            float o[4];
            for (int i = 0; i < 4; ++i) o[i] = -sigmoid_ref(v[i] + bias[i]);
            st4(e.C, e.ldc, o);
            break;
        }
        case EPI_AXPY: {
            float o[4];
            for (int i = 0; i < 4; ++i) o[i] = a[i] + e.alpha * v[i];
            st4(e.C, e.ldc, o);
            break;
        }
        default: break;
    }
    (void)row;
    return part;
}

// smem tile row store of a reduced float4
__device__ __forceinline__ void red_buf_store(float* tile, int r, int c, int TP, const float4& v) {
    *reinterpret_cast<float4*>(tile + r * TP + c) = v;
}
// distributed shared memory: address of the same smem offset in cluster CTA `rank`, and a 16 B load
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ float4 ld_dsmem4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
                 : "memory");
    return v;
}

// softmax (layers.hpp:301-320) + softmax_cross_entropy (network.hpp:410-437) of one full row held
// in the smem tile; sequential in j like the reference.
__device__ __forceinline__ void softmax_row(const GemmParams& p, const float* trow, int m, const float* sbias) {
    const EpiParams& e = p.ep;
    float mx = -INFINITY;
    auto bias = [&](int n) { return sbias ? sbias[n] : e.bias[(long long)n * e.bias_stride]; };
    for (int n = 0; n < p.N; ++n) mx = fmaxf(mx, trow[n] + bias(n));
    float sum = 0.0f;
    for (int n = 0; n < p.N; ++n) sum += expf((trow[n] + bias(n)) - mx);
    const int label = e.labels[m];
    int best = 0;
    float bestp = -1.0f, ptrue = 0.0f;
    for (int n = 0; n < p.N; ++n) {
        const float q = expf((trow[n] + bias(n)) - mx) / sum;
        if (q > bestp) {  // strict >: first maximum wins (network.hpp:69-70)
            bestp = q;
            best = n;
        }
        if (n == label) ptrue = q;
        e.C[(long long)m * e.ldc + n] = (q - (n == label ? 1.0f : 0.0f)) / e.batch_div;
        if (e.probs) e.probs[(long long)m * e.ld_probs + n] = q;
    }
    e.row_loss[m] = -log(fmax((double)ptrue, 1e-300));
    if (e.argmax) e.argmax[m] = best;
}

// L2 prefetch of the epilogue's input rows for this tile, issued while the main loop runs
template <int BN, int EPI>
__device__ __forceinline__ void epilogue_prefetch(const GemmParams& p, int m0, int n0, int ct) {
    const EpiParams& e = p.ep;
    const int rows = min(kBM, p.M - m0);
    auto rowpf = [&](const void* base, long long ld, int es) {
        if (!base) return;
        const int lines = (BN * es + 127) / 128;
        for (int idx = ct; idx < rows * lines; idx += 32 * kEpiWarps) {
            const int r = idx / lines, l = idx % lines;
            prefetch_l2(static_cast<const char*>(base) + ((long long)(m0 + r) * ld + n0) * es + l * 128);
        }
    };
    switch (EPI) {
        case EPI_DACT: rowpf(e.aux, e.ld_aux, 4); rowpf(e.C, e.ldc, 4); break;
        case EPI_SGD: rowpf(e.C, e.ldc, 4); rowpf(e.V, e.ldv, 4); break;
        case EPI_AXPY: rowpf(e.C, e.ldc, 4); break;
        case EPI_RBM_HID: rowpf(e.u, e.ldu, 8); rowpf(e.C, e.ldc, 4); rowpf(e.C2, e.ldc2, 4); break;
        case EPI_RBM_VIS: rowpf(e.aux, e.ld_aux, 4); rowpf(e.C, e.ldc, 4); break;
        default: rowpf(e.C, e.ldc, 4); break;
    }
    if (e.bias && ct < BN && n0 + ct < p.N) prefetch_l2(e.bias + (long long)(n0 + ct) * e.bias_stride);
}

template <int BN, bool X3, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const GemmParams p) {
    using Cfg = GemmCfg<BN, X3>;
    constexpr int S = Cfg::STAGES;
    constexpr int TP = Cfg::TP;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::MAIN_BYTES);
    uint64_t* ready = full + S;
    uint64_t* empty = ready + S;
    uint64_t* tmem_full = empty + S;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
    float* tile = reinterpret_cast<float*>(smem);  // epilogue staging, reuses the drained stages

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * BN;
    const int num_kb_total = (p.K + kBK - 1) / kBK;
    const int split = blockIdx.z;
    const int kb0 = split * p.kb_per_split;
    const int kb1 = min(num_kb_total, kb0 + p.kb_per_split);
    const int num_kb = kb1 > kb0 ? kb1 - kb0 : 0;

    if (threadIdx.x == 0) {
        B2N_TRACE(0);
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&ready[s], 32 * kEpiWarps);
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
    if (threadIdx.x == 0) B2N_TRACE(1);

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            auto load_a = [&](int i) {
                uint8_t* a = smem + (i % S) * Cfg::STAGE_BYTES;
                const int k0 = (kb0 + i) * kBK;
                if (!p.a_mn) {
                    tma_load_2d(a, &mapA, &full[i % S], k0, m0);
                } else {
#pragma unroll
                    for (int j = 0; j < kBM / 32; ++j) tma_load_2d(a + j * 4096, &mapA, &full[i % S], m0 + 32 * j, k0);
                }
            };
            auto load_b = [&](int i) {
                uint8_t* b = smem + (i % S) * Cfg::STAGE_BYTES + Cfg::A_BYTES;
                const int k0 = (kb0 + i) * kBK;
                if (!p.b_mn) {
                    tma_load_2d(b, &mapB, &full[i % S], k0, n0);
                } else {
#pragma unroll
                    for (int j = 0; j < BN / 32; ++j) tma_load_2d(b + j * 4096, &mapB, &full[i % S], n0 + 32 * j, k0);
                }
            };
            // pull every K block past the resident stages toward L2 now: after the step's L2 flush
            // the loads would otherwise pay HBM latency one pipeline round at a time
            for (int i = S; i < num_kb; ++i) {
                const int k0 = (kb0 + i) * kBK;
                if (!p.a_mn) tma_prefetch_2d(&mapA, k0, m0);
                else for (int j = 0; j < kBM / 32; ++j) tma_prefetch_2d(&mapA, m0 + 32 * j, k0);
                if (!p.b_mn) tma_prefetch_2d(&mapB, k0, n0);
                else for (int j = 0; j < BN / 32; ++j) tma_prefetch_2d(&mapB, n0 + 32 * j, k0);
            }
            // operands independent of the preceding kernel stream in while it drains (PDL)
            const int pre = min(num_kb, S);
            for (int i = 0; i < pre; ++i) {
                mbar_arrive_expect_tx(&full[i], Cfg::A_BYTES + Cfg::B_BYTES);
                if (i < 16) B2N_TRACE(2 + i);
                if (p.pre_a) load_a(i);
                if (p.pre_b) load_b(i);
            }
            pdl_wait();
            for (int i = 0; i < pre; ++i) {
                if (!p.pre_a) load_a(i);
                if (!p.pre_b) load_b(i);
            }
            for (int i = pre; i < num_kb; ++i) {
                const int s = i % S;
                const uint32_t ph = (i / S) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&full[s], Cfg::A_BYTES + Cfg::B_BYTES);
                if (i < 16) B2N_TRACE(2 + i);
                load_a(i);
                load_b(i);
            }
        }
    } else if (warp == 1) {  // ---------------- MMA issue: whole warp, one elected lane per MMA
        // descriptors advance by running adds on the 14-bit start-address field: a K-major kk step is
        // 32 B (SW128 rows), an MN-major one 1024 B (8 K-rows of 128 B); stages STAGE_BYTES apart
        const uint32_t idesc = umma_idesc_tf32(kBM, BN, p.a_mn, p.b_mn);
        const uint32_t idesc2 = umma_idesc_tf32(kBM, Cfg::STACK ? 2 * BN : BN, p.a_mn, p.b_mn);
        const uint32_t a0 = smem_u32(smem), b0 = a0 + Cfg::A_BYTES;
        const uint64_t da0 = p.a_mn ? desc_mnmajor(a0, 0) : desc_kmajor(a0, 0);
        const uint64_t db0 = p.b_mn ? desc_mnmajor(b0, 0) : desc_kmajor(b0, 0);
        const uint64_t a_kk = p.a_mn ? 64 : 2, b_kk = p.b_mn ? 64 : 2;
        constexpr uint64_t lo_add = (uint64_t)((Cfg::A_BYTES + Cfg::B_BYTES) >> 4);
        for (int i = 0; i < num_kb; ++i) {
            const int s = i % S;
            const uint32_t ph = (i / S) & 1;
            mbar_wait(X3 ? &ready[s] : &full[s], ph);
            tc_fence_after();
            if (i < 16 && lane == 0) B2N_TRACE(34 + i);
            const uint64_t st = (uint64_t)((s * Cfg::STAGE_BYTES) >> 4);
            uint64_t dah = da0 + st, dbh = db0 + st;
#pragma unroll
            for (int kk = 0; kk < kBK / 8; ++kk, dah += a_kk, dbh += b_kk) {
                if (Cfg::STACK) {  // stage: A hi | B hi | B lo | A lo
                    mma_tf32_warp(tmem_base, dah, dbh, idesc2, (i | kk) != 0);
                    mma_tf32_warp(tmem_base, dah + (uint64_t)((Cfg::A_BYTES + 2 * Cfg::B_BYTES) >> 4), dbh, idesc, 1);
                } else if (X3) {
                    mma_tf32_warp(tmem_base, dah + lo_add, dbh, idesc, (i | kk) != 0);
                    mma_tf32_warp(tmem_base, dah, dbh + lo_add, idesc, 1);
                    mma_tf32_warp(tmem_base, dah, dbh, idesc, 1);
                } else {
                    mma_tf32_warp(tmem_base, dah, dbh, idesc, (i | kk) != 0);
                }
            }
            mma_commit_warp(&empty[s]);
        }
        mma_commit_warp(tmem_full);
        if (lane == 0) B2N_TRACE(50);
    } else {  // ---------------- splitters, then TMEM -> smem tile (warps 2..9)
        const int ct = threadIdx.x - 64;
        epilogue_prefetch<BN, EPI>(p, m0, n0, ct);
        if (X3) {
            for (int i = 0; i < num_kb; ++i) {
                const int s = i % S;
                const uint32_t ph = (i / S) & 1;
                mbar_wait(&full[s], ph);
                if (ct == 0 && i < 16) B2N_TRACE(18 + i);
                uint8_t* a = smem + s * Cfg::STAGE_BYTES;
                if (Cfg::STACK) {
                    split_lo(a + Cfg::A_BYTES, a + Cfg::A_BYTES + Cfg::B_BYTES, Cfg::B_BYTES, ct, 32 * kEpiWarps);
                    split_lo(a, a + Cfg::A_BYTES + 2 * Cfg::B_BYTES, Cfg::A_BYTES, ct, 32 * kEpiWarps);
                } else {
                    split_lo(a, a + Cfg::A_BYTES + Cfg::B_BYTES, Cfg::A_BYTES + Cfg::B_BYTES, ct, 32 * kEpiWarps);
                }
                fence_proxy_async_smem();
                mbar_arrive(&ready[s]);
            }
        }
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        if (ct == 0) {
            B2N_TRACE(51);
            pdl_trigger();  // main loop done: let the next kernel launch and run its prologue
        }
        const int q = warp & 3;            // TMEM lane quadrant this warp may access
        const int half = (warp - 2) >> 2;  // two warps per quadrant split the columns
        const int row = 32 * q + lane;
        const uint32_t trow = tmem_base + ((uint32_t)(32 * q) << 16);
        float* dst = tile + row * TP;
        if (num_kb == 0) {
            for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); ++c) dst[c] = 0.0f;
        } else if (BN >= 32) {
            for (int c = half * (BN / 2); c < (half + 1) * (BN / 2); c += 16) {
                float v[16];
                tmem_ld16(trow + c, v);
                if (Cfg::STACK) {  // fold the a_hi.b_lo half
                    float w[16];
                    tmem_ld16(trow + c + BN, w);
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[i] += w[i];
                }
#pragma unroll
                for (int i = 0; i < 16; i += 4)
                    *reinterpret_cast<float4*>(dst + c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            }
        } else {
            float v[8];
            tmem_ld8(trow + half * 8, v);
            if (Cfg::STACK) {
                float w[8];
                tmem_ld8(trow + half * 8 + BN, w);
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] += w[i];
            }
#pragma unroll
            for (int i = 0; i < 8; i += 4)
                *reinterpret_cast<float4*>(dst + half * 8 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        }
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    pdl_wait();  // global writes (and epilogue reads) only after the preceding kernel completed
    if (threadIdx.x == 0) B2N_TRACE(53);

    // rows of the tile this CTA finishes: all of them, or (split-K) one slice per cluster rank
    int r_lo = 0, r_hi = kBM;
    const int rank = p.splits > 1 ? (int)cluster_rank() : 0;
    if (p.splits > 1) {
        const int rows = (kBM + p.splits - 1) / p.splits;
        r_lo = min(kBM, rank * rows);
        r_hi = min(kBM, r_lo + rows);
    }
    // epilogue inputs that do not depend on the product (bias, u, aux, C, V) are loaded now, so their
    // latency overlaps the split-K exchange instead of following it
    constexpr int G = BN / 4;  // threads per tile row (kThreads % G == 0: a thread keeps its columns)
    const int total = (r_hi - r_lo) * G;
    const int iters = (total + kThreads - 1) / kThreads;
    const int ccol = (threadIdx.x % G) * 4;
    float bias4[4] = {0.f, 0.f, 0.f, 0.f};
    EpiIn pre[kEpiPrefetch];
    // softmax: the bias row (one strided column of W_aug) staged in the drained operand stages
    // behind the tile with independent loads now, instead of a serial global load per class later
    constexpr bool kStageBias = Cfg::MAIN_BYTES >= Cfg::TILE_BYTES + 256 * 4;
    float* sbias = kStageBias ? tile + kBM * TP : nullptr;
    if constexpr (EPI == EPI_SOFTMAX_XENT && kStageBias) {
        for (int i = threadIdx.x; i < p.N; i += kThreads) sbias[i] = p.ep.bias[(long long)i * p.ep.bias_stride];
        if (p.splits <= 1) __syncthreads();  // (split-K: the cluster barriers below order it)
    }
    if constexpr (EPI != EPI_SOFTMAX_XENT) {
        epi_bias<EPI>(p, n0 + ccol, bias4);
#pragma unroll
        for (int it = 0; it < kEpiPrefetch; ++it) {
            const int idx = it * kThreads + threadIdx.x;
            const int m = m0 + r_lo + idx / G, n = n0 + ccol;
            if (it < iters && idx < total && m < p.M && n < p.N) epi_load<EPI>(p, m, n, pre[it]);
        }
    }

    // ---------------- split-K reduction across the cluster through distributed shared memory: every
    // CTA's partial tile stays in its own smem; rank z sums its row slice over the peers in fixed split
    // order (deterministic), then a second cluster barrier keeps the peers' smem alive until all read
    if (p.splits > 1) {
        if (threadIdx.x == 0) B2N_TRACE(54);
        cluster_sync_all();  // release our partial / acquire everyone's
        if (threadIdx.x == 0) B2N_TRACE(55);
        const uint32_t tl = smem_u32(tile);
        for (int idx = threadIdx.x; idx < (r_hi - r_lo) * (BN / 4); idx += kThreads) {
            const int r = r_lo + idx / (BN / 4), c = (idx % (BN / 4)) * 4;
            const uint32_t off = (uint32_t)((r * TP + c) * 4);
            float4 acc = ld_dsmem4(mapa_u32(tl + off, 0));
            for (int z = 1; z < p.splits; ++z) {
                const float4 t = ld_dsmem4(mapa_u32(tl + off, (uint32_t)z));
                acc.x += t.x;
                acc.y += t.y;
                acc.z += t.z;
                acc.w += t.w;
            }
            red_buf_store(tile, r, c, TP, acc);
        }
        if (threadIdx.x == 0) B2N_TRACE(58);
        cluster_sync_all();  // every peer has read our partial: slices may now be overwritten
        if (threadIdx.x == 0) B2N_TRACE(56);
    }

    // ---------------- fused epilogue on rows [r_lo, r_hi) of the tile
    if (threadIdx.x == 0) B2N_TRACE(59);
    if constexpr (EPI == EPI_SOFTMAX_XENT) {
        for (int r = r_lo + threadIdx.x; r < r_hi; r += kThreads)
            if (m0 + r < p.M) softmax_row(p, tile + r * TP, m0 + r, sbias);
    } else {
        auto body = [&](int it, const EpiIn& in) {
            const int idx = it * kThreads + threadIdx.x;
            const int r = r_lo + idx / G, c = ccol;
            const int m = m0 + r, n = n0 + c;
            double part = 0.0;
            if (idx < total && m < p.M && n < p.N) {
                const float4 t = *reinterpret_cast<const float4*>(tile + r * TP + c);
                const float v[4] = {t.x, t.y, t.z, t.w};
                part = epi_apply<EPI>(p, m, n, v, bias4, in);
            }
            if constexpr (G <= 32 && EPI == EPI_RBM_VIS) {  // row partial over this CTA's BN columns
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                if (idx < total && (idx % G) == 0 && m < p.M)
                    p.ep.row_part[(long long)blockIdx.x * p.ep.ld_part + m] = part;
            }
        };
#pragma unroll
        for (int it = 0; it < kEpiPrefetch; ++it)
            if (it < iters) body(it, pre[it]);
        for (int it = kEpiPrefetch; it < iters; ++it) {
            EpiIn in;
            const int idx = it * kThreads + threadIdx.x;
            const int m = m0 + r_lo + idx / G, n = n0 + ccol;
            if (idx < total && m < p.M && n < p.N) epi_load<EPI>(p, m, n, in);
            body(it, in);
        }
    }

    if (threadIdx.x == 0) B2N_TRACE(60);
    __syncthreads();
    if (threadIdx.x == 0) B2N_TRACE(57);
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
    if (threadIdx.x == 0) B2N_TRACE(52);
}

}  // namespace b2n
