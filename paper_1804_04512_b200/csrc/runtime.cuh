// runtime.cuh -- host-side plumbing shared by every op: typed errors (mirroring fastnn's
// config.hpp:11-57 hierarchy as status codes), TMA descriptor encoding, GEMM planning / launch,
// and the bandwidth-bound kernels that are not GEMM epilogues (SGD over packed buffers,
// standalone softmax-xent for classes > 256, fills).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <random>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <chrono>
#include <string>
#include <memory>
#include <vector>

#include "../../include/b200nn.h"
#include "gemm_tc.cuh"

namespace b2n {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define B2N_CUDA(x)                                                                                        \
    do {                                                                                                   \
        cudaError_t e_ = (x);                                                                              \
        if (e_ != cudaSuccess)                                                                             \
            throw ::b2n::Error(B2N_ECUDA, std::string(#x) + " failed: " + cudaGetErrorString(e_) + " (" + \
                                              __FILE__ + ":" + std::to_string(__LINE__) + ")");            \
    } while (0)

inline long long round_up(long long n, long long m) { return (n + m - 1) / m * m; }

// std::uniform_real_distribution<float>(a, b) as libstdc++ evaluates it (random.h:1907-1909:
// generate_canonical<float, 24>(urng) * (b - a) + a) with the multiply-add fused, which is what the
// reference's -march=native build emits (-ffp-contract=fast); spelled out so the init is
// bit-identical to fastnn::glorot_fill (layers.hpp:40-48) whatever flags compile this file.
struct UniformF32 {
    float a, b;
    UniformF32(float lo, float hi) : a(lo), b(hi) {}
    template <class R>
    float operator()(R& rng) {
        const float u = std::generate_canonical<float, std::numeric_limits<float>::digits>(rng);
        return std::fma(u, b - a, a);
    }
};

// ------------------------------------------------------------------ TMA descriptors
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        B2N_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw Error(B2N_ECUDA, "cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// cuStreamWriteValue32: a stream-ordered 32-bit store, fenced after the stream's earlier work
// (copies included), for device-side readiness flags
inline void stream_write_u32(cudaStream_t st, unsigned* addr, unsigned v) {
    typedef CUresult (*WriteFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
    static WriteFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        B2N_CUDA(cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw Error(B2N_ECUDA, "cuStreamWriteValue32 unavailable");
        return reinterpret_cast<WriteFn>(p);
    }();
    const CUresult r = fn(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(addr), v, 0);
    if (r != CUDA_SUCCESS) throw Error(B2N_ECUDA, "cuStreamWriteValue32 failed (" + std::to_string((int)r) + ")");
}

// 2-D fp32 map over a row-major matrix of `outer` rows x `inner` logical columns with row pitch
// `ld` elements; 128 B-swizzled boxes of box_inner (32) x box_outer (16 B atoms for K-major operands,
// 32 B atoms for MN-major ones); out-of-bounds reads fill zero.
inline CUtensorMap make_map_2d(const float* base, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                               uint32_t box_outer, bool mn_major = false) {
    if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * 4) & 15))
        throw Error(B2N_ESHAPE, "tensor-core operand needs a 16-byte aligned base and a row pitch that is a "
                                "multiple of 4 floats (fastnn pads rows to 8, tensor.hpp:142)");
    CUtensorMap m;
    cuuint64_t dims[2] = {inner, std::max<uint64_t>(outer, 1)};
    cuuint64_t strides[1] = {ld * 4};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE,
                             mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(B2N_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

// Low-latency host wait for the step result: record an event behind the work and busy-poll it (a
// blocking cudaStreamSynchronize may sleep and wake the host thread several microseconds late; the
// step itself is tens of microseconds). One event per thread, reused.
// While a host thread waits, the live NCCL communicators are polled (failure detection):
// an asynchronous NCCL error or a wait beyond the communicator's timeout aborts it and throws
// B2N_ENCCL instead of hanging the process behind a dead peer (nccl_dyn.cuh, DpComm::poll).
struct WaitWatch {
    virtual void poll(double waited_s) = 0;
    virtual ~WaitWatch() = default;
};
inline std::vector<WaitWatch*>& wait_watches() {
    static std::vector<WaitWatch*> v;
    return v;
}

inline void spin_sync(cudaStream_t st) {
    thread_local cudaEvent_t ev = [] {
        cudaEvent_t e = nullptr;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) e = nullptr;
        return e;
    }();
    if (!ev) {
        B2N_CUDA(cudaStreamSynchronize(st));
        return;
    }
    B2N_CUDA(cudaEventRecord(ev, st));
    cudaError_t e;
    unsigned long long spins = 0;
    std::chrono::steady_clock::time_point t0;
    while ((e = cudaEventQuery(ev)) == cudaErrorNotReady) {
        if (!wait_watches().empty() && (++spins & 0x3FFF) == 0) {  // every few ms of waiting
            if (spins == 0x4000) t0 = std::chrono::steady_clock::now();
            const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            for (WaitWatch* w : wait_watches()) w->poll(waited);
        }
    }
    B2N_CUDA(e);
}

struct DevMem {
    void* p = nullptr;
    size_t bytes = 0;
    DevMem() = default;
    DevMem(const DevMem&) = delete;  // owns p
    DevMem& operator=(const DevMem&) = delete;
    void alloc(size_t n) {
        release();
        if (n == 0) return;
        cudaError_t e = cudaMalloc(&p, n);
        if (e != cudaSuccess) {
            p = nullptr;
            throw Error(e == cudaErrorMemoryAllocation ? B2N_EOOM : B2N_ECUDA,
                        std::string("cudaMalloc(") + std::to_string(n) + "): " + cudaGetErrorString(e));
        }
        bytes = n;
        // zero-fill, then wait for it: the objects' streams are non-blocking and do not order
        // against the legacy stream cudaMemset runs on
        B2N_CUDA(cudaMemset(p, 0, n));
        B2N_CUDA(cudaDeviceSynchronize());
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    ~DevMem() { release(); }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct HostPinned {
    void* p = nullptr;
    size_t bytes = 0;
    void alloc(size_t n) {
        release();
        B2N_CUDA(cudaMallocHost(&p, std::max<size_t>(n, 64)));
        bytes = n;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
    }
    ~HostPinned() { release(); }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// ------------------------------------------------------------------ launches
// Every step kernel is launched with programmatic stream serialization (PDL): inside a captured
// graph the edge becomes programmatic, so a kernel's launch + prologue overlap its predecessor's
// tail; kernels call pdl_wait() before touching dependent data. B2N_PDL=0 disables it.
inline bool pdl_enabled() {
    static bool on = [] {
        const char* e = std::getenv("B2N_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename... KArgs, typename... Args>
inline void launch_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                      unsigned cluster_z, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int n = 0;
    if (pdl_enabled()) {
        at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    if (cluster_z > 1) {
        at[n].id = cudaLaunchAttributeClusterDimension;
        at[n].val.clusterDim.x = 1;
        at[n].val.clusterDim.y = 1;
        at[n].val.clusterDim.z = cluster_z;
        ++n;
    }
    cfg.attrs = at;
    cfg.numAttrs = n;
    B2N_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// ------------------------------------------------------------------ GEMM plan
// One operand of D = op(A) . op(B). K-major: row-major [rows][K] (fastnn NT side);
// MN-major: row-major [K][rows] (the transposed side).
struct Operand {
    const float* ptr;
    long long ld;
    bool mn_major;
};

struct GemmLaunch {
    CUtensorMap ma, mb;
    GemmParams p;
    int bn = 64;
    bool x3 = true;
    dim3 grid;
    std::shared_ptr<DevMem> ws;  // split-K partial tiles
    double flops = 0, bytes = 0;  // algorithmic work of one launch (roofline numerators)
    // address ranges for the PDL prefetch analysis: operands read, epilogue outputs written
    std::pair<uintptr_t, uintptr_t> a_rng{0, 0}, b_rng{0, 0};
    std::vector<std::pair<uintptr_t, uintptr_t>> writes;
    void run(cudaStream_t st) const;
};

inline std::pair<uintptr_t, uintptr_t> rng_of(const void* p, long long rows, long long ld, int elem = 4) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    return {a, a + (uintptr_t)std::max<long long>(rows, 0) * ld * elem};
}
inline bool overlaps(std::pair<uintptr_t, uintptr_t> x, std::pair<uintptr_t, uintptr_t> y) {
    return x.first < y.second && y.first < x.second;
}

// Algorithmic HBM bytes of one GEMM launch: each operand read once, each epilogue stream once.
inline double gemm_bytes(int M, int N, int K, int epi) {
    const double mn = (double)M * N, a = (double)M * K * 4, b = (double)N * K * 4;
    double e = 0;
    switch (epi) {
        case EPI_STORE: e = mn * 4; break;
        case EPI_BIAS_ACT: e = mn * 4 + N * 4.0; break;
        case EPI_DACT: e = mn * 8; break;
        case EPI_SOFTMAX_XENT: e = mn * 8 + M * 16.0 + N * 4.0; break;
        case EPI_SGD: e = mn * 16; break;
        case EPI_RBM_HID: e = mn * 16 + N * 4.0; break;
        case EPI_RBM_VIS: e = mn * 8 + M * 8.0 + N * 4.0; break;
        case EPI_RBM_NEGHID: e = mn * 4 + N * 4.0; break;
        case EPI_AXPY: e = mn * 8; break;
        default: e = mn * 4;
    }
    return a + b + e;
}

template <int BN, bool X3, int EPI>
void launch_gemm_inst(const GemmLaunch& g, cudaStream_t st) {
    using Cfg = GemmCfg<BN, X3>;
    static bool attr = [] {
        B2N_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, X3, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      Cfg::SMEM));
        return true;
    }();
    (void)attr;
    // split-K CTAs of one tile form a cluster along z
    launch_ex(gemm_tc_kernel<BN, X3, EPI>, g.grid, dim3(kThreads, 1, 1), Cfg::SMEM, st, (unsigned)g.p.splits, g.ma,
              g.mb, g.p);
}

// per-epilogue launchers, each instantiated in its own translation unit (gemm_e<N>.cu): one
// kernel per (BN, precision, epilogue) keeps each kernel's code small -- after the per-step L2
// flush every first-executed instruction line comes from HBM
// tile widths the planner can choose per epilogue: 16 only with a K-major B (N <= 16), 256 only for
// a fused softmax over up to 256 classes
constexpr bool bn_allowed(int epi, int bn) {
    return bn == 16 ? (epi == EPI_STORE || epi == EPI_BIAS_ACT || epi == EPI_SOFTMAX_XENT)
                    : bn == 256 ? epi == EPI_SOFTMAX_XENT : true;
}

template <int BN, int EPI>
inline void launch_gemm_bn(const GemmLaunch& g, cudaStream_t st) {
    if constexpr (bn_allowed(EPI, BN)) {
        if (g.x3)
            launch_gemm_inst<BN, true, EPI>(g, st);
        else
            launch_gemm_inst<BN, false, EPI>(g, st);
    } else {
        throw Error(B2N_EINTERNAL, "tile width not instantiated for this epilogue");
    }
}

template <int EPI>
void gemm_launch_epi(const GemmLaunch& g, cudaStream_t st) {
    switch (g.bn) {
        case 16: launch_gemm_bn<16, EPI>(g, st); break;
        case 32: launch_gemm_bn<32, EPI>(g, st); break;
        case 64: launch_gemm_bn<64, EPI>(g, st); break;
        case 128: launch_gemm_bn<128, EPI>(g, st); break;
        case 256: launch_gemm_bn<256, EPI>(g, st); break;
        default: throw Error(B2N_ESHAPE, "bad BN");
    }
}
#ifndef B2N_GEMM_INSTANTIATE
extern template void gemm_launch_epi<EPI_STORE>(const GemmLaunch&, cudaStream_t);
extern template void gemm_launch_epi<EPI_BIAS_ACT>(const GemmLaunch&, cudaStream_t);
extern template void gemm_launch_epi<EPI_DACT>(const GemmLaunch&, cudaStream_t);
extern template void gemm_launch_epi<EPI_SOFTMAX_XENT>(const GemmLaunch&, cudaStream_t);
extern template void gemm_launch_epi<EPI_SGD>(const GemmLaunch&, cudaStream_t);
extern template void gemm_launch_epi<EPI_RBM_HID>(const GemmLaunch&, cudaStream_t);
extern template void gemm_launch_epi<EPI_RBM_VIS>(const GemmLaunch&, cudaStream_t);
extern template void gemm_launch_epi<EPI_RBM_NEGHID>(const GemmLaunch&, cudaStream_t);
extern template void gemm_launch_epi<EPI_AXPY>(const GemmLaunch&, cudaStream_t);
#endif

inline void GemmLaunch::run(cudaStream_t st) const {
    switch (p.epi) {
        case EPI_STORE: gemm_launch_epi<EPI_STORE>(*this, st); break;
        case EPI_BIAS_ACT: gemm_launch_epi<EPI_BIAS_ACT>(*this, st); break;
        case EPI_DACT: gemm_launch_epi<EPI_DACT>(*this, st); break;
        case EPI_SOFTMAX_XENT: gemm_launch_epi<EPI_SOFTMAX_XENT>(*this, st); break;
        case EPI_SGD: gemm_launch_epi<EPI_SGD>(*this, st); break;
        case EPI_RBM_HID: gemm_launch_epi<EPI_RBM_HID>(*this, st); break;
        case EPI_RBM_VIS: gemm_launch_epi<EPI_RBM_VIS>(*this, st); break;
        case EPI_RBM_NEGHID: gemm_launch_epi<EPI_RBM_NEGHID>(*this, st); break;
        case EPI_AXPY: gemm_launch_epi<EPI_AXPY>(*this, st); break;
        default: throw Error(B2N_EINTERNAL, "bad epilogue");
    }
}

// Tile width and split-K factor: enough CTAs to put most SMs to work on these latency-bound shapes
// (<= 128 CTAs in clusters of <= 8, the co-residency limit), the widest tile that still gets there.
struct Tiling {
    int bn, splits, kb_per_split;
};
inline Tiling pick_tiling(int M, int N, int K, bool b_mn, int epi) {
    const int mt = (M + kBM - 1) / kBM, nkb = (K + kBK - 1) / kBK;
    int bn;
    if (epi == EPI_SOFTMAX_XENT) {
        bn = N <= 16 ? 16 : N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
        if (b_mn && bn < 32) bn = 32;
    } else if (N <= 16 && !b_mn && bn_allowed(epi, 16)) {
        bn = 16;
    } else if (epi == EPI_SGD && mt * ((N + 31) / 32) <= 148) {
        // the SGD epilogue reads and writes W and V (16 B per output) -- far more traffic than the
        // K = batch product: the narrowest tile spreads it over the most SMs (while one wave)
        bn = 32;
    } else {
        bn = 32;
        for (int c : {128, 64})
            if ((long long)mt * ((N + c - 1) / c) * std::min(8, nkb) >= 96) {
                bn = c;
                break;
            }
    }
    const int tiles = mt * ((N + bn - 1) / bn);
    // split-K only where it pays: ~0.35 us per 3xTF32 K block vs ~1.3 us for the cluster reduction
    // (measured, tests/_graph_trace.py); power-of-two clusters, <= 112 CTAs for clusters of 8
    int splits = 1;
    double best = nkb * 0.35;
    for (int sp = 2; sp <= 8 && sp <= nkb; sp *= 2) {
        if (tiles * sp > (sp == 8 ? 112 : 148)) break;
        const double t = ((nkb + sp - 1) / sp) * 0.35 + 1.3;
        if (t < best - 1e-9) {
            best = t;
            splits = sp;
        }
    }
    const int kbps = (nkb + splits - 1) / splits;
    return {bn, splits, kbps};
}

// Bring-up tracing (B2N_TRACE=1): every planned GEMM gets a region of a global device buffer in
// which each CTA records %globaltimer stamps (gemm_tc.cuh B2N_TRACE slots); b2n_debug_trace_read
// copies it out. Off by default (null trace pointer, no cost).
struct TraceRegistry {
    static constexpr int kRegionCtas = 512;
    static constexpr int kMaxRegions = 64;
    DevMem buf;
    int used = 0;
    bool on = false;
    static TraceRegistry& get() {
        static TraceRegistry r;
        static const bool init = [] {
            const char* e = std::getenv("B2N_TRACE");
            r.on = e && e[0] == '1';
            return true;
        }();
        (void)init;
        return r;
    }
    unsigned long long* next() {
        if (!on) return nullptr;
        if (!buf.p) buf.alloc((size_t)kMaxRegions * kRegionCtas * 64 * 8);
        if (used >= kMaxRegions) return nullptr;
        return buf.as<unsigned long long>() + (size_t)(used++) * kRegionCtas * 64;
    }
};

inline GemmLaunch plan_gemm(int M, int N, int K, Operand A, Operand B, int epi, const EpiParams& ep, bool x3,
                            int bn = 0) {
    if (M <= 0 || N <= 0 || K <= 0) throw Error(B2N_ESHAPE, "gemm extents must be positive");
    GemmLaunch g;
    Tiling t = pick_tiling(M, N, K, B.mn_major, epi);
    if (bn) t.bn = bn;
    g.bn = t.bn;
    if (epi == EPI_SOFTMAX_XENT && N > g.bn) throw Error(B2N_ESHAPE, "fused softmax needs classes <= 256");
    if (B.mn_major && g.bn < 32) g.bn = 32;
    g.x3 = x3;
    g.ma = A.mn_major ? make_map_2d(A.ptr, M, K, A.ld, 32, 32, true) : make_map_2d(A.ptr, K, M, A.ld, 32, kBM);
    g.mb = B.mn_major ? make_map_2d(B.ptr, N, K, B.ld, 32, 32, true) : make_map_2d(B.ptr, K, N, B.ld, 32, g.bn);
    g.p.M = M;
    g.p.N = N;
    g.p.K = K;
    g.p.a_mn = A.mn_major;
    g.p.b_mn = B.mn_major;
    g.p.epi = epi;
    g.p.ep = ep;
    g.p.trace = nullptr;
    if ((long long)((N + 31) / 32) * ((M + kBM - 1) / kBM) * 8 <= TraceRegistry::kRegionCtas)
        g.p.trace = TraceRegistry::get().next();
    g.p.splits = t.splits;
    g.p.kb_per_split = t.kb_per_split;
    g.p.pre_a = 0;
    g.p.pre_b = 0;
    g.p.ws = nullptr;
    g.grid = dim3((N + g.bn - 1) / g.bn, (M + kBM - 1) / kBM, t.splits);
    if (t.splits > 1) {
        g.ws = std::make_shared<DevMem>();
        g.ws->alloc((size_t)g.grid.x * g.grid.y * t.splits * kBM * g.bn * 4);
        g.p.ws = g.ws->as<float>();
    }
    g.flops = 2.0 * M * N * K;
    g.bytes = gemm_bytes(M, N, K, epi);
    g.a_rng = rng_of(A.ptr, A.mn_major ? K : M, A.ld);
    g.b_rng = rng_of(B.ptr, B.mn_major ? K : N, B.ld);
    if (ep.C) g.writes.push_back(rng_of(ep.C, M, ep.ldc));
    if (epi == EPI_SGD && ep.V) g.writes.push_back(rng_of(ep.V, M, ep.ldv));
    if (epi == EPI_RBM_HID && ep.C2) g.writes.push_back(rng_of(ep.C2, M, ep.ldc2));
    if (epi == EPI_RBM_VIS && ep.row_part) g.writes.push_back(rng_of(ep.row_part, 64, ep.ld_part, 8));
    if (epi == EPI_SOFTMAX_XENT) {
        if (ep.probs) g.writes.push_back(rng_of(ep.probs, M, ep.ld_probs));
        if (ep.row_loss) g.writes.push_back(rng_of(ep.row_loss, M, 1, 8));
        if (ep.argmax) g.writes.push_back(rng_of(ep.argmax, M, 1, 4));
    }
    return g;
}

inline EpiParams epi_default() {
    EpiParams e;
    std::memset(&e, 0, sizeof(e));
    e.alpha = 1.0f;
    e.batch_div = 1.0f;
    return e;
}

// ------------------------------------------------------------------ bandwidth kernels
// sgd_momentum_step (optim.hpp:69-80) over one packed parameter / velocity / gradient buffer:
// float4-vectorised, grid-stride, 16 B per thread per access.
static __global__ void sgd_packed_kernel(float4* __restrict__ p, float4* __restrict__ v, const float4* __restrict__ g,
                                  long long n4, float lr, float mom, float wd) {
    pdl_wait();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        float4 pp = p[i], vv = v[i];
        const float4 gg = g[i];
        float gx = gg.x + wd * pp.x, gy = gg.y + wd * pp.y, gz = gg.z + wd * pp.z, gw = gg.w + wd * pp.w;
        vv.x = mom * vv.x - lr * gx;
        vv.y = mom * vv.y - lr * gy;
        vv.z = mom * vv.z - lr * gz;
        vv.w = mom * vv.w - lr * gw;
        pp.x += vv.x;
        pp.y += vv.y;
        pp.z += vv.z;
        pp.w += vv.w;
        p[i] = pp;
        v[i] = vv;
    }
}

// adagrad / adadelta / adam steps (optim.hpp:83-127) over the packed buffers. s1 = acc (adagrad,
// adadelta) or m (adam); s2 = acc_update (adadelta) or v (adam). Adam's bias corrections come from
// a host-computed table c[t] = {1 - powf(b1, t), 1 - powf(b2, t)} (the reference's std::pow on
// floats) indexed by the device step counter, which the last block to finish advances -- so a
// replayed graph steps t without the host.
struct OptCounter {
    long long t;            // completed adam steps
    unsigned int done;      // blocks finished in the current launch
};
constexpr int OPT_ADAGRAD = 1, OPT_ADADELTA = 2, OPT_ADAM = 3;

template <int KIND>
__device__ __forceinline__ void opt_elem(float& p, float& a, float& b, float g, float lr, float eps, float rho,
                                         float b1, float b2, float c1, float c2) {
    if constexpr (KIND == OPT_ADAGRAD) {
        a += g * g;
        p -= lr * g / (sqrtf(a) + eps);
    } else if constexpr (KIND == OPT_ADADELTA) {
        a = rho * a + (1.0f - rho) * g * g;
        const float delta = -sqrtf(b + eps) / sqrtf(a + eps) * g;
        b = rho * b + (1.0f - rho) * delta * delta;
        p += delta;
    } else {
        a = b1 * a + (1.0f - b1) * g;
        b = b2 * b + (1.0f - b2) * g * g;
        p -= lr * (a / c1) / (sqrtf(b / c2) + eps);
    }
}

template <int KIND>
static __global__ void opt_packed_kernel(float4* __restrict__ p, float4* __restrict__ s1, float4* __restrict__ s2,
                                         const float4* __restrict__ g, long long n4, float lr, float eps, float rho,
                                         float b1, float b2, const float2* __restrict__ ctab, OptCounter* cnt) {
    pdl_wait();
    float c1 = 1.0f, c2 = 1.0f;
    if (KIND == OPT_ADAM) {
        const float2 c = ctab[cnt->t + 1];
        c1 = c.x;
        c2 = c.y;
    }
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        float4 pp = p[i], aa = s1[i], bb = KIND == OPT_ADAGRAD ? make_float4(0, 0, 0, 0) : s2[i];
        const float4 gg = g[i];
        opt_elem<KIND>(pp.x, aa.x, bb.x, gg.x, lr, eps, rho, b1, b2, c1, c2);
        opt_elem<KIND>(pp.y, aa.y, bb.y, gg.y, lr, eps, rho, b1, b2, c1, c2);
        opt_elem<KIND>(pp.z, aa.z, bb.z, gg.z, lr, eps, rho, b1, b2, c1, c2);
        opt_elem<KIND>(pp.w, aa.w, bb.w, gg.w, lr, eps, rho, b1, b2, c1, c2);
        p[i] = pp;
        s1[i] = aa;
        if (KIND != OPT_ADAGRAD) s2[i] = bb;
    }
    if (KIND == OPT_ADAM) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(&cnt->done, 1u) == gridDim.x - 1) {  // every block has read t
                cnt->t += 1;
                cnt->done = 0;
            }
        }
    }
}

static __global__ void fill_kernel(float* __restrict__ p, long long n, float v) {
    pdl_wait();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}

// ones column of an augmented activation matrix (the bias trick: [X | 1] . [W | b]^T)
static __global__ void set_column_kernel(float* __restrict__ p, long long rows, long long ld, long long col, float v) {
    pdl_wait();
    long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r < rows) p[r * ld + col] = v;
}

// W += alpha * D over a packed buffer (data-parallel RBM update after the allreduce)
static __global__ void axpy_kernel(float4* __restrict__ w, const float4* __restrict__ d, long long n4, float alpha) {
    pdl_wait();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        float4 a = w[i];
        const float4 b = d[i];
        a.x += alpha * b.x;
        a.y += alpha * b.y;
        a.z += alpha * b.z;
        a.w += alpha * b.w;
        w[i] = a;
    }
}

// softmax + softmax_cross_entropy for class counts beyond one tensor-core tile: one warp per row,
// the max / exp-sum / normalise passes run in the reference's sequential order by lane 0 after a
// warp-parallel max (max is order-independent), so dlogits and loss follow network.hpp:410-437.
// softmax + cross-entropy over rows of > 256 classes (layers.hpp:301-320, network.hpp:423-437): one CTA
// of kSxThreads per row, the row staged once in shared memory (float4 loads, all in flight). The exp
// terms are computed in parallel; ONE thread sums them in the reference's sequential order (the fp32
// add chain, 4 clk per class, is the floor of the row); then every thread finishes its share of the
// row: probs, loss, gradient (q - onehot) / batch written once, and the first-max argmax of q (fixed
// tree: lowest index on equal q).
constexpr int kSxThreads = 128;
static __global__ void __launch_bounds__(kSxThreads) softmax_xent_rows_kernel(
    const float* __restrict__ logits, long long ld, int rows, int cols, const int* __restrict__ labels, float batch_div,
    float* __restrict__ dlogits, long long ldd, double* __restrict__ row_loss, int* __restrict__ argmax,
    float* __restrict__ probs, long long ldp) {
    extern __shared__ __align__(16) float e[];  // [cols rounded up to 4]
    __shared__ float s_red[kSxThreads / 32];
    __shared__ int s_idx[kSxThreads / 32];
    __shared__ float s_sum;
    pdl_wait();
    const int row = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (row >= rows) return;
    const float* z = logits + (long long)row * ld;
    float* dl = dlogits + (long long)row * ldd;
    float mx = -INFINITY;
    const int c4 = (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(logits) & 15) == 0 ? cols >> 2 : 0;
#pragma unroll 4
    for (int i = tid; i < c4; i += kSxThreads) {
        const float4 v = *reinterpret_cast<const float4*>(z + 4 * i);
        *reinterpret_cast<float4*>(e + 4 * i) = v;
        mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
    }
    for (int j = 4 * c4 + tid; j < cols; j += kSxThreads) {
        const float v = z[j];
        e[j] = v;
        mx = fmaxf(mx, v);
    }
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) s_red[w] = mx;
    __syncthreads();
    mx = s_red[0];
#pragma unroll
    for (int i = 1; i < kSxThreads / 32; ++i) mx = fmaxf(mx, s_red[i]);
#pragma unroll 4
    for (int j = tid; j < cols; j += kSxThreads) e[j] = expf(e[j] - mx);
    __syncthreads();
    if (tid == 0) {  // sequential, layers.hpp:312-315 order
        float sum = 0.0f;
        int j = 0;
#pragma unroll 8
        for (; j + 4 <= cols; j += 4) {
            const float4 v = *reinterpret_cast<const float4*>(e + j);
            sum += v.x;
            sum += v.y;
            sum += v.z;
            sum += v.w;
        }
        for (; j < cols; ++j) sum += e[j];
        s_sum = sum;
    }
    __syncthreads();
    const float sum = s_sum;
    const int label = labels[row];
    float bestp = -1.0f;
    int best = 0;
#pragma unroll 4
    for (int j = tid; j < cols; j += kSxThreads) {
        const float q = e[j] / sum;
        if (q > bestp) {
            bestp = q;
            best = j;
        }
        if (probs) probs[(long long)row * ldp + j] = q;
        if (j == label) row_loss[row] = -log(fmax((double)q, 1e-300));
        dl[j] = (q - (j == label ? 1.0f : 0.0f)) / batch_div;
    }
    for (int o = 16; o; o >>= 1) {  // first-max argmax: lanes, then warps
        const float bp = __shfl_xor_sync(0xffffffffu, bestp, o);
        const int bi = __shfl_xor_sync(0xffffffffu, best, o);
        if (bp > bestp || (bp == bestp && bi < best)) {
            bestp = bp;
            best = bi;
        }
    }
    __syncthreads();  // s_red reused
    if (lane == 0) {
        s_red[w] = bestp;
        s_idx[w] = best;
    }
    __syncthreads();
    if (tid == 0) {
        for (int i = 1; i < kSxThreads / 32; ++i)
            if (s_red[i] > bestp || (s_red[i] == bestp && s_idx[i] < best)) {
                bestp = s_red[i];
                best = s_idx[i];
            }
        dl[cols] = 0.0f;  // the ones column of the next dW product
        if (argmax) argmax[row] = best;
    }
}

inline int grid_for(long long n, int block = 256) {
    long long g = (n + block - 1) / block;
    return (int)std::min<long long>(std::max<long long>(g, 1), 148 * 8);
}

}  // namespace b2n
