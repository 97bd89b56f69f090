// rbm.cuh -- device-resident replacement of fastnn::Rbm + cd_k_update (energy.hpp:16-32, :131-171)
// for binary units. One CD-k step is k*2 + 2 tcgen05 GEMM launches (4 for CD-1):
//
//   h0/hs : Vcat[0:B] . W^T, epilogue sigmoid(+bh) -> h0 (into Hcat[0:B]) and hs = (u < h0)
//   v1    : hs . W,          epilogue sigmoid(+bv) -> Vcat[B:2B], row partials of (v0 - v1)^2
//   h1    : Vcat[B:2B] . W^T, epilogue -sigmoid(+bh) -> Hcat[B:2B]
//   dW    : Hcat^T . Vcat over K = 2B  ->  W_aug += lr/B * acc
//
// W_aug is (H+1) x ldw: W in [0:H, 0:V], bh in column V, bv in row H. Hcat carries a +1 / -1
// column and Vcat a ones column, so the single concatenated-K GEMM yields
//   [0:H, 0:V] = pos - neg,  [0:H, V] = sum(h0 - h1),  [H, 0:V] = sum(v0 - v1)
// i.e. the reference's weight update and both bias updates (energy.hpp:148-169) in one pass.
#pragma once
#include <cstdio>
#include <random>

#include "mt19937.cuh"
#include "nccl_dyn.cuh"
#include "network.cuh"
#include "rbm_fused.cuh"

namespace b2n {

// The one summation order of a step's (tile, row) reconstruction partials, shared by the host
// (Rbm::recon), dbn_pretrain's device accumulator and the fused kernel's in-kernel sum: 32 lanes
// take rows lane, lane + 32, ... (tiles inner, in order), then the xor butterfly of a warp
// shuffle reduction (lane 0's result), simulated lane by lane here.
__host__ __device__ inline double recon_tree_sum(const double* part, int tiles, long long cap, long long B) {
    double lane[32];
    for (int l = 0; l < 32; ++l) {
        double a = 0.0;
        for (long long r = l; r < B; r += 32)
            for (int t = 0; t < tiles; ++t) a += part[t * cap + r];
        lane[l] = a;
    }
    for (int o = 16; o > 0; o >>= 1) {
        double nx[32];
        for (int l = 0; l < 32; ++l) nx[l] = lane[l] + lane[l ^ o];
        for (int l = 0; l < 32; ++l) lane[l] = nx[l];
    }
    return lane[0];
}

// dbn_pretrain's per-step reconstruction error (recon_tree_sum / batch) added to the epoch sum
// (energy.hpp:232)
static __global__ void recon_accum_kernel(const double* __restrict__ part, int tiles, long long cap, long long B,
                                          double* acc) {
    if (threadIdx.x != 0) return;
    *acc += recon_tree_sum(part, tiles, cap, B) / (double)B;
}

// lo = x - trunc_tf32(x), the 3xTF32 correction operand of W kept next to W for the fused step
static __global__ void tf32_lo_kernel(const float4* __restrict__ x, float4* __restrict__ lo, long long n4) {
    pdl_wait();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
        const float4 v = x[i];
        lo[i] = make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
    }
}

// v0 rows into a visible staging buffer (pitch ldd) plus their tf32 lo parts (copy == 0: already there),
// and flags[s] = 1 iff 128-column slice s holds a value that is not exact in tf32 (0 otherwise, every
// one of the 16 flags written -- no memset before). CTA s owns slice s over all B rows: lanes take
// float4 columns, the warps take rows.
static __global__ void stage_rows_kernel(const float* __restrict__ src, long long lds, float* __restrict__ dst,
                                         float* __restrict__ dlo, long long ldd, int B, int V, int copy,
                                         unsigned* flags) {
    pdl_wait();
    const int s = blockIdx.x, c0 = 128 * s, c1 = min(V, c0 + 128);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const bool vec = (V & 3) == 0 && ((lds | ldd) & 3) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(dlo) & 15) == 0 && (!copy || (reinterpret_cast<uintptr_t>(dst) & 15) == 0);
    int inexact = 0;
#pragma unroll 4
    for (int r = w; r < B; r += nw) {
        const float* sr = src + (long long)r * lds;
        float* dr = dst + (long long)r * ldd;
        float* lr = dlo + (long long)r * ldd;
        if (vec) {
            const int c = c0 + 4 * lane;
            if (c < c1) {
                const float4 x = *reinterpret_cast<const float4*>(sr + c);
                if (copy) *reinterpret_cast<float4*>(dr + c) = x;
                const float4 lo = make_float4(tf32_lo(x.x), tf32_lo(x.y), tf32_lo(x.z), tf32_lo(x.w));
                *reinterpret_cast<float4*>(lr + c) = lo;
                inexact |= lo.x != 0.0f || lo.y != 0.0f || lo.z != 0.0f || lo.w != 0.0f;
            }
        } else {
            for (int c = c0 + lane; c < c1; c += 32) {
                const float x = sr[c];
                if (copy) dr[c] = x;
                const float lo = tf32_lo(x);
                lr[c] = lo;
                inexact |= lo != 0.0f;
            }
        }
    }
    inexact = __syncthreads_or(inexact);
    if (threadIdx.x == 0 && s < 16) flags[s] = inexact ? 1u : 0u;  // (only the fused step's slices are read)
    if (s == 0)
        for (int t = gridDim.x + threadIdx.x; t < 16; t += blockDim.x) flags[t] = 0u;
}

class Rbm {
  public:
    static constexpr int kStage = 8;  // visible-side buffers: train_stream stages up to 8 steps ahead
    Rbm(long long H, long long V, int device, int precision)
        : H_(H), V_(V), device_(device), x3_(precision == B2N_TF32X3) {
        if (H < 1 || V < 1) throw Error(B2N_ESHAPE, "rbm extents must be positive");
        B2N_CUDA(cudaSetDevice(device));
        B2N_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
        ldw_ = round_up(V + 1, 8);
        nW_ = round_up((H + 1) * ldw_, 32);
        W_.alloc(nW_ * 4);
        Wlo_.alloc(nW_ * 4);
        G_.alloc(nW_ * 4);
        h_recon_.alloc(8 * 1024);
    }
    ~Rbm() {
        plans_.clear();
        for (cudaEvent_t e : uev_)
            if (e) cudaEventDestroy(e);
        for (int j = 0; j < kStage; ++j) {
            if (ev_used_[j]) cudaEventDestroy(ev_used_[j]);
            if (ev_rng_[j]) cudaEventDestroy(ev_rng_[j]);
        }
        if (copy_stream_) cudaStreamDestroy(copy_stream_);
        if (recon_host_) cudaFreeHost(recon_host_);
        if (stream_) cudaStreamDestroy(stream_);
    }

    void init(unsigned seed) {  // energy.hpp:31 -> glorot_fill(w, visible, hidden)
        std::mt19937 rng(seed);
        const float limit = std::sqrt(6.0f / static_cast<float>(V_ + H_));
        UniformF32 dist(-limit, limit);
        std::vector<float> w((size_t)(H_ * V_));
        for (float& v : w) v = dist(rng);
        std::vector<float> zh((size_t)H_, 0.0f), zv((size_t)V_, 0.0f);
        set(w.data(), zv.data(), zh.data());
    }
    void set(const float* w, const float* bv, const float* bh) {
        wlo_valid_ = false;
        float* W = W_.as<float>();
        B2N_CUDA(cudaMemsetAsync(W, 0, nW_ * 4, stream_));
        B2N_CUDA(cudaMemcpy2DAsync(W, ldw_ * 4, w, V_ * 4, V_ * 4, H_, cudaMemcpyHostToDevice, stream_));
        B2N_CUDA(cudaMemcpy2DAsync(W + V_, ldw_ * 4, bh, 4, 4, H_, cudaMemcpyHostToDevice, stream_));
        B2N_CUDA(cudaMemcpyAsync(W + H_ * ldw_, bv, V_ * 4, cudaMemcpyHostToDevice, stream_));
        B2N_CUDA(cudaStreamSynchronize(stream_));
    }
    void get(float* w, float* bv, float* bh) {
        const float* W = W_.as<float>();
        if (w) B2N_CUDA(cudaMemcpy2DAsync(w, V_ * 4, W, ldw_ * 4, V_ * 4, H_, cudaMemcpyDeviceToHost, stream_));
        if (bh) B2N_CUDA(cudaMemcpy2DAsync(bh, 4, W + V_, ldw_ * 4, 4, H_, cudaMemcpyDeviceToHost, stream_));
        if (bv) B2N_CUDA(cudaMemcpyAsync(bv, W + H_ * ldw_, V_ * 4, cudaMemcpyDeviceToHost, stream_));
        B2N_CUDA(cudaStreamSynchronize(stream_));
    }

    double cd_k(const float* v0, long long B, int k, float lr, const double* u, long long Bg) {
        if (k < 1) throw Error(B2N_EPARAM, "cd_k_update: k must be >= 1, got " + std::to_string(k));
        if (B < 1 || Bg < B) throw Error(B2N_ESHAPE, "cd_k_update: need 1 <= batch <= batch_global");
        ensure_capacity(B, k);
        Plan& pl = plan_for(B, k, lr, Bg);
        const float* v0d = device_alias(v0);
        const double* ud = u ? device_alias(u) : nullptr;
        if (pl.fused && v0d && (ud || !u) && V_ % 4 == 0) {
            if (!u) {  // the Bernoulli draws from the device generator (set_rng)
                ud = U_.as<double>();
                rng_.draw(U_.as<double>(), B * H_, stream_);
            }
            // pinned caller buffers: the fused kernel reads v0 and the uniforms itself (zero-copy),
            // launched directly with this call's pointers instead of staging copies + the graph
            staged_B_ = B;
            staged_k_ = k;
            prepare(pl);
            RbmFusedParams rp = pl.rp;
            rp.v0_src = v0d;
            rp.ld_src = V_;
            rp.v0_inexact = nullptr;  // staged in-kernel: exactness unknown, full 3xTF32
            rp.u_src = ud;
            rp.recon_out = recon_host_dev_;
            recon_mapped_ = true;
            launch_ex(rbm_cd1_fused_kernel, dim3(kRfSlices, rp.jt), dim3(kRfThreads), (size_t)kRfSmem, stream_, 1u,
                      pl.maps[0], rp);
            vb_ = 0;
        } else {
            stage(v0, u, B, k);
            launch(pl);
        }
        if (dp_) throw Error(B2N_EPARAM, "data-parallel RBM steps through run_staged");
        last_B_ = B;
        last_Bg_ = Bg;
        return recon();
    }
    void stage(const float* v0, const double* u, long long B, int k = 1) {
        ensure_capacity(B, k);
        float* Vc = Vcat_[0].as<float>();
        B2N_CUDA(cudaMemcpy2DAsync(Vc, ldv_ * 4, v0, V_ * 4, V_ * 4, B, cudaMemcpyHostToDevice, stream_));
        stage_lo(0, B, stream_);
        vb_ = 0;
        if (u)
            B2N_CUDA(cudaMemcpyAsync(U_.p, u, (size_t)k * B * H_ * 8, cudaMemcpyHostToDevice, stream_));
        else  // u == null: draw the k * B * H uniforms from the device generator (set_rng)
            rng_.draw(U_.as<double>(), (long long)k * B * H_, stream_);
        staged_B_ = B;
        staged_k_ = k;
    }
    void run_staged(int steps, float lr, long long Bg) {
        if (!staged_B_) throw Error(B2N_EPARAM, "run_staged before stage");
        Plan& pl = plan_for(staged_B_, staged_k_, lr, Bg ? Bg : staged_B_);
        for (int s = 0; s < steps; ++s) launch(pl);
        last_B_ = staged_B_;
        last_Bg_ = pl.Bg;
    }
    double recon() {  // sum of the per-(tile,row) partials / batch_global
        if (recon_mapped_) {  // the fused step already wrote it to host-mapped memory
            spin_sync(stream_);
            return *reinterpret_cast<volatile double*>(recon_host_);
        }
        const long long nt = recon_tiles_;
        // partials are [tile][cap_]: copy through the last tile's rows
        B2N_CUDA(cudaMemcpyAsync(h_recon_.p, recon_.p, ((nt - 1) * cap_ + last_B_) * 8, cudaMemcpyDeviceToHost, stream_));
        spin_sync(stream_);
        return recon_tree_sum(h_recon_.as<double>(), (int)nt, cap_, last_B_) / (double)last_Bg_;
    }
    void last_states(float* h0, float* hs, float* v1, float* h1) {
        const long long B = last_B_;
        const float* Hc = Hcat_.as<float>();
        const float* Vc = Vcat_[vb_].as<float>();
        const auto D2H = cudaMemcpyDeviceToHost;
        if (h0) B2N_CUDA(cudaMemcpy2DAsync(h0, H_ * 4, Hc, ldh_ * 4, H_ * 4, B, D2H, stream_));
        if (hs) B2N_CUDA(cudaMemcpy2DAsync(hs, H_ * 4, HS_.p, ldhs_ * 4, H_ * 4, B, D2H, stream_));
        if (v1) B2N_CUDA(cudaMemcpy2DAsync(v1, V_ * 4, Vc + B * ldv_, ldv_ * 4, V_ * 4, B, D2H, stream_));
        if (h1) B2N_CUDA(cudaMemcpy2DAsync(h1, H_ * 4, Hc + B * ldh_, ldh_ * 4, H_ * 4, B, D2H, stream_));
        B2N_CUDA(cudaStreamSynchronize(stream_));
        if (h1) {
            for (long long i = 0; i < B * H_; ++i) h1[i] = -h1[i];  // stored negated for the dW GEMM
        }
    }
    void dp_init(const char id[128], int rank, int world) {
        dp_ = std::make_unique<DpComm>();
        dp_->init(id, rank, world);
        plans_.clear();
    }
    // gradient-only steps (the caller reduces the shards): cd_k_update leaves W alone and keeps this
    // shard's raw sums dW_aug = (Hcat^T Vcat)^T in G; apply_update then adds lr / batch_global * G
    void set_grad_only(bool on) {
        if (on != grad_only_) plans_.clear();
        grad_only_ = on;
    }
    void get_grad(float* w, float* bv, float* bh) {
        const float* G = G_.as<float>();
        if (w) B2N_CUDA(cudaMemcpy2DAsync(w, V_ * 4, G, ldw_ * 4, V_ * 4, H_, cudaMemcpyDeviceToHost, stream_));
        if (bh) B2N_CUDA(cudaMemcpy2DAsync(bh, 4, G + V_, ldw_ * 4, 4, H_, cudaMemcpyDeviceToHost, stream_));
        if (bv) B2N_CUDA(cudaMemcpyAsync(bv, G + H_ * ldw_, V_ * 4, cudaMemcpyDeviceToHost, stream_));
        B2N_CUDA(cudaStreamSynchronize(stream_));
    }
    void set_grad(const float* w, const float* bv, const float* bh) {
        float* G = G_.as<float>();
        B2N_CUDA(cudaMemsetAsync(G, 0, nW_ * 4, stream_));
        B2N_CUDA(cudaMemcpy2DAsync(G, ldw_ * 4, w, V_ * 4, V_ * 4, H_, cudaMemcpyHostToDevice, stream_));
        B2N_CUDA(cudaMemcpy2DAsync(G + V_, ldw_ * 4, bh, 4, 4, H_, cudaMemcpyHostToDevice, stream_));
        B2N_CUDA(cudaMemcpyAsync(G + H_ * ldw_, bv, V_ * 4, cudaMemcpyHostToDevice, stream_));
        B2N_CUDA(cudaStreamSynchronize(stream_));
    }
    void apply_update(float lr, long long Bg) {  // energy.hpp:148-169 with the shards' summed G
        if (Bg < 1) throw Error(B2N_EPARAM, "apply_update: batch_global must be >= 1");
        const long long n = nW_;
        launch_ex(axpy_kernel, dim3(grid_for(n / 4)), dim3(256), 0, stream_, 1u, reinterpret_cast<float4*>(W_.as<float>()),
                  reinterpret_cast<const float4*>(G_.as<float>()), n / 4, lr / static_cast<float>(Bg));
        wlo_valid_ = false;
        B2N_CUDA(cudaStreamSynchronize(stream_));
    }
    // the caller's std::mt19937 (625 words: state, position) for the steps that take no uniforms
    void set_rng(const uint32_t* st) { rng_.load(st, stream_); }
    void get_rng(uint32_t* st) { rng_.store(st, stream_); }
    long long hidden() const { return H_; }
    long long visible() const { return V_; }
    long long ld_visible() const { return round_up(V_ + 1, 8); }  // row pitch of a visible-side data matrix

    // One epoch of dbn_pretrain's inner loop (energy.hpp:226-233): CD-1 over rows [0, n) of a
    // device-resident data matrix (pitch ld_visible()) in file order, `batch` rows per step (the
    // last step takes the remainder). The Bernoulli uniforms come from `fill` (the caller's
    // mt19937 stream, B x H per step, in step order) through two pinned buffers so the host
    // draws step i+1 while the GPU runs step i. The per-step reconstruction errors are summed on
    // the device in the reference's order; one host synchronisation per epoch.
    double train_epoch(const float* data, long long n, long long batch, float lr, b2n_uniform_fn fill, void* ctx) {
        if (dp_) throw Error(B2N_EPARAM, "dbn_pretrain: data-parallel RBMs step through run_staged");
        ensure_capacity(std::min(batch, n), 1);
        const long long per = std::min(batch, n) * H_;
        for (int j = 0; fill && j < 2; ++j) {
            if (ubuf_[j].bytes < (size_t)per * 8) ubuf_[j].alloc((size_t)per * 8);
            if (!uev_[j]) B2N_CUDA(cudaEventCreateWithFlags(&uev_[j], cudaEventDisableTiming));
        }
        if (!racc_.p) racc_.alloc(16);
        B2N_CUDA(cudaMemsetAsync(racc_.p, 0, 8, stream_));
        const long long ldd = ld_visible();
        long long batches = 0;
        bool pending[2] = {false, false};
        for (long long lo = 0; lo < n; lo += batch, ++batches) {
            const long long B = std::min(batch, n - lo);
            const int j = (int)(batches & 1);
            if (fill) {
                if (pending[j]) B2N_CUDA(cudaEventSynchronize(uev_[j]));  // its previous H2D has drained
                fill(ctx, ubuf_[j].as<double>(), B * H_);
                B2N_CUDA(cudaMemcpyAsync(U_.p, ubuf_[j].p, (size_t)(B * H_ * 8), cudaMemcpyHostToDevice, stream_));
                B2N_CUDA(cudaEventRecord(uev_[j], stream_));
                pending[j] = true;
            } else {  // the device generator (set_rng): no host draws, no copies
                rng_.draw(U_.as<double>(), B * H_, stream_);
            }
            B2N_CUDA(cudaMemcpy2DAsync(Vcat_[0].p, ldv_ * 4, data + lo * ldd, ldd * 4, V_ * 4, B,
                                       cudaMemcpyDeviceToDevice, stream_));
            stage_lo(0, B, stream_);
            vb_ = 0;
            Plan& pl = plan_for(B, 1, lr, B);
            launch(pl);
            recon_accum_kernel<<<1, 32, 0, stream_>>>(recon_.as<double>(), recon_tiles_, cap_, B, racc_.as<double>());
            B2N_CUDA(cudaGetLastError());
        }
        double acc = 0.0;
        B2N_CUDA(cudaMemcpyAsync(&acc, racc_.p, 8, cudaMemcpyDeviceToHost, stream_));
        B2N_CUDA(cudaStreamSynchronize(stream_));
        last_B_ = 0;
        return acc / (double)batches;
    }

    // A stream of CD-1 steps over host batches (the reference's training loop of cd_k_update calls,
    // energy.hpp:131): step i takes rows [i B, (i + 1) B) of v0 (pitch V) and of the uniforms
    // (pitch H, or null: drawn on the device). Up to kStage steps ahead of the compute stream, a copy
    // stream lands step i's v0 in visible buffer i % kStage (+ its tf32 lo parts) and the device
    // generator draws its uniforms on a third stream; the step kernel polls a readiness flag instead
    // of a cross-stream event. Each step's reconstruction error lands in a device array read back
    // once. recon_out[i] = step i's cd_k_update return value.
    void train_stream(const float* v0, const double* u, long long steps, long long B, float lr, double* recon_out) {
        if (dp_) throw Error(B2N_EPARAM, "train_stream: data-parallel RBMs step through run_staged");
        if (steps < 1 || B < 1) throw Error(B2N_ESHAPE, "train_stream: need steps >= 1 and batch >= 1");
        ensure_capacity(B, 1);
        Plan& pl = plan_for(B, 1, lr, B);
        if (!pl.fused || V_ % 4 != 0) {  // the split path: staged copies + the step graph, in order
            for (long long i = 0; i < steps; ++i) {
                stage(v0 + i * B * V_, u ? u + i * B * H_ : nullptr, B, 1);
                launch(pl);
                last_B_ = B;
                last_Bg_ = B;
                recon_out[i] = recon();
            }
            return;
        }
        prepare(pl);
        for (int j = 0; j < kStage; ++j) {
            if (su_[j].bytes < (size_t)(B * H_ * 8)) su_[j].alloc((size_t)(B * H_ * 8));
            if (!ev_used_[j]) B2N_CUDA(cudaEventCreateWithFlags(&ev_used_[j], cudaEventDisableTiming));
            if (!ev_rng_[j]) B2N_CUDA(cudaEventCreateWithFlags(&ev_rng_[j], cudaEventDisableTiming));
        }
        if (!copy_stream_) B2N_CUDA(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));
        // per-step recon slots, grown geometrically (no allocation inside a later, longer stream)
        if (rstream_.bytes < (size_t)steps * 8) rstream_.alloc(std::max<size_t>((size_t)steps * 8 * 2, 8192));
        // readiness flags: the copy stream stamps step i + 1 into flag j after step i's copies (a
        // stream memory write, fenced after them); the step kernel polls it, so the compute stream
        // carries no cross-stream event and consecutive steps keep their programmatic overlap
        if (!sready_.p) sready_.alloc(64);
        B2N_CUDA(cudaMemsetAsync(sready_.p, 0, 64, stream_));
        for (int j = 0; j < kStage; ++j)
            B2N_CUDA(cudaEventRecord(ev_used_[j], stream_));  // staging buffers free after prior work
        if (!u) rng_.stream_begin(B * H_, stream_, 4);
        for (long long i = 0; i < steps; ++i) {
            const int j = (int)(i % kStage);
            B2N_CUDA(cudaStreamWaitEvent(copy_stream_, ev_used_[j], 0));  // step i - kStage done with buffer j
            B2N_CUDA(cudaMemcpy2DAsync(Vcat_[j].p, ldv_ * 4, v0 + i * B * V_, V_ * 4, V_ * 4, B, cudaMemcpyDefault,
                                       copy_stream_));  // host (pinned or not) or device-resident batches
            stage_lo(j, B, copy_stream_);
            if (u)
                B2N_CUDA(cudaMemcpyAsync(su_[j].p, u + i * B * H_, (size_t)(B * H_ * 8), cudaMemcpyDefault,
                                         copy_stream_));
            else {  // step i's draws from the device generator (jump-ahead pipelined), up to kStage steps ahead
                rng_.stream_step((int)i, (int)steps, su_[j].as<double>(), ev_used_[j], ev_rng_[j]);
                B2N_CUDA(cudaStreamWaitEvent(copy_stream_, ev_rng_[j], 0));
            }
            unsigned* flag = sready_.as<unsigned>() + j;
            stream_write_u32(copy_stream_, flag, (unsigned)(i + 1));
            RbmFusedParams rp = pl.rp;
            rp.Vcat = Vcat_[j].as<float>();
            rp.Vlo = Vlo_[j].as<float>();
            rp.v0_inexact = vflags_.as<unsigned>() + 16 * j;
            rp.u_src = su_[j].as<double>();
            rp.ready = flag;
            rp.ready_val = (unsigned)(i + 1);
            rp.recon_out = rstream_.as<double>() + i;
            if (rp.trace) rp.trace += 256 * (i & 1);  // bring-up: consecutive steps in separate halves
            launch_ex(rbm_cd1_fused_kernel, dim3(kRfSlices, rp.jt), dim3(kRfThreads), (size_t)kRfSmem, stream_, 1u,
                      pl.maps[j], rp);
            B2N_CUDA(cudaEventRecord(ev_used_[j], stream_));
            vb_ = j;
        }
        B2N_CUDA(cudaEventRecord(ev_used_[0], copy_stream_));  // after the last draw (copy stream waited on it)
        B2N_CUDA(cudaStreamWaitEvent(stream_, ev_used_[0], 0));
        if (!u) rng_.stream_end((int)steps, stream_);
        B2N_CUDA(cudaMemcpyAsync(recon_out, rstream_.p, (size_t)steps * 8, cudaMemcpyDeviceToHost, stream_));
        spin_sync(stream_);
        staged_B_ = B;
        staged_k_ = 1;
        last_B_ = B;
        last_Bg_ = B;
        recon_mapped_ = false;
    }

    // rbm_transform_up (energy.hpp:122-126): out = sigmoid(data . W^T + bh) for n rows, data pitch
    // ld_visible(), out pitch round_up(H + 1, 8) (the next layer's ld_visible())
    void transform_up(const float* data, long long n, float* out) {
        EpiParams e = epi_default();
        e.C = out;
        e.ldc = round_up(H_ + 1, 8);
        e.bias = W_.as<float>() + V_;
        e.bias_stride = ldw_;
        e.act = ACT_SIGMOID;
        GemmLaunch g = plan_gemm((int)n, (int)H_, (int)V_, {data, ld_visible(), false}, {W_.as<float>(), ldw_, false},
                                 EPI_BIAS_ACT, e, x3_);
        g.run(stream_);
        B2N_CUDA(cudaGetLastError());
    }
    cudaStream_t stream() const { return stream_; }
    int kernels_per_step() const { return last_kernels_; }
    std::vector<OpStats> profile(int steps, float lr, long long Bg) {
        if (!staged_B_) throw Error(B2N_EPARAM, "profile before stage");
        Plan& pl = plan_for(staged_B_, staged_k_, lr, Bg ? Bg : staged_B_);
        prepare(pl);  // the +1/-1 column, W's lo companion
        if (hcol_B_ != pl.B) launch(pl);
        return profile_ops(pl.ops, steps, stream_);
    }

  private:
    struct Plan {
        long long B, Bg;
        int k;
        float lr;
        std::vector<Op> ops;
        int nk = 0;
        int recon_tiles = 1;
        bool fused = false;         // rp / maps describe the single fused launch
        RbmFusedParams rp;
        RbmMaps maps[kStage];
        cudaGraphExec_t graph = nullptr;
        ~Plan() {
            if (graph) cudaGraphExecDestroy(graph);
        }
    };


    void ensure_capacity(long long B, int k) {
        if (B <= cap_ && k <= kcap_) return;
        cap_ = std::max(cap_, B);
        kcap_ = std::max(kcap_, k);
        plans_.clear();
        hcol_B_ = -1;
        ldv_ = round_up(V_ + 1, 8);
        ldh_ = round_up(H_ + 1, 8);
        ldhs_ = round_up(H_, 8);
        for (int k = 0; k < kStage; ++k) {
            Vcat_[k].alloc(2 * cap_ * ldv_ * 4);
            Vlo_[k].alloc(2 * cap_ * ldv_ * 4);
        }
        Hcat_.alloc(2 * cap_ * ldh_ * 4);
        Hlo_.alloc(2 * cap_ * ldh_ * 4);
        vflags_.alloc((size_t)kStage * 64);
        HS_.alloc(cap_ * ldhs_ * 4);
        U_.alloc((size_t)kcap_ * cap_ * H_ * 8);
        recon_.alloc((size_t)cap_ * 64 * 8);
        if (h_recon_.bytes < (size_t)cap_ * 64 * 8) h_recon_.alloc((size_t)cap_ * 64 * 8);
        for (int k = 0; k < kStage; ++k)
            set_column_kernel<<<grid_for(2 * cap_), 256, 0, stream_>>>(Vcat_[k].as<float>(), 2 * cap_, ldv_, V_, 1.0f);
        B2N_CUDA(cudaGetLastError());
        B2N_CUDA(cudaStreamSynchronize(stream_));
    }

    Plan& plan_for(long long B, int k, float lr, long long Bg) {
        for (auto& p : plans_)
            if (p->B == B && p->k == k && p->lr == lr && p->Bg == Bg) return *p;
        auto pl = std::make_unique<Plan>();
        pl->B = B;
        pl->k = k;
        pl->lr = lr;
        pl->Bg = Bg;
        build(*pl);
        plans_.push_back(std::move(pl));
        return *plans_.back();
    }

    // the fused single-kernel CD-1 step (rbm_fused.cuh) covers k = 1, 3xTF32, single GPU, B <= 128,
    // H < 512, V < 1024, when all its clusters can be co-resident (grid barrier); B2N_RBM_FUSED=0 opts out
    bool fused_ok(const Plan& pl) const {
        const char* e = std::getenv("B2N_RBM_FUSED");
        if (e && e[0] == '0') return false;
        const int jt = (int)((H_ + 1 + kRfTileH - 1) / kRfTileH);
        if (pl.k != 1 || !x3_ || pl.B > 128 || pl.B > 16LL * jt || jt > 8 || V_ + 1 > kRfSlices * kRfSliceW)
            return false;
        static int clusters = [] {
            B2N_CUDA(cudaFuncSetAttribute(rbm_cd1_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kRfSmem));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(kRfSlices, 8);
            cfg.blockDim = dim3(kRfThreads);
            cfg.dynamicSmemBytes = kRfSmem;
            cudaLaunchAttribute at;
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = kRfSlices;
            at.val.clusterDim.y = 1;
            at.val.clusterDim.z = 1;
            cfg.attrs = &at;
            cfg.numAttrs = 1;
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, rbm_cd1_fused_kernel, &cfg) != cudaSuccess) {
                cudaGetLastError();
                cfg.numAttrs = 0;  // compile-time cluster dims only
                if (cudaOccupancyMaxActiveClusters(&n, rbm_cd1_fused_kernel, &cfg) != cudaSuccess) n = 0;
            }
            cudaGetLastError();
            return n;
        }();
        if (std::getenv("B2N_RBM_FUSED_VERBOSE"))
            std::fprintf(stderr, "b2n: fused CD-1 needs %d co-resident clusters of %d, device reports %d\n", jt, kRfSlices,
                         clusters);
        return clusters >= jt;
    }

    void build_fused(Plan& pl) {
        const int B = (int)pl.B, H = (int)H_, V = (int)V_;
        const int jt = (H + 1 + kRfTileH - 1) / kRfTileH;
        float* W = W_.as<float>();
        float* Vc = Vcat_[0].as<float>();
        float* Hc = Hcat_.as<float>();
        if (!fused_ws_.p) {
            fused_ws_.alloc((size_t)8 * 128 * kRfSlices * kRfSliceW * 4 + (size_t)8 * kRfSlices * 128 * kRfTileH * 4);
            gbar_.alloc(8 * 128 + 256);  // 8 slice counters, 128 B apart
        }
        RbmFusedParams rp;
        std::memset(&rp, 0, sizeof(rp));
        rp.B = B;
        rp.H = H;
        rp.V = V;
        rp.ldw = ldw_;
        rp.ldv = ldv_;
        rp.ldh = ldh_;
        rp.ldhs = ldhs_;
        rp.W = W;
        rp.Vcat = Vc;
        rp.Hcat = Hc;
        rp.Wlo = Wlo_.as<float>();
        rp.Vlo = Vlo_[0].as<float>();
        rp.v0_inexact = vflags_.as<unsigned>();
        rp.Hlo = Hlo_.as<float>();
        rp.HS = HS_.as<float>();
        rp.u = U_.as<double>();
        rp.row_part = recon_.as<double>();
        rp.cap = cap_;
        rp.ws2 = fused_ws_.as<float>();
        rp.ws1 = rp.ws2 + (size_t)8 * 128 * kRfSlices * kRfSliceW;
        rp.gbar = gbar_.as<unsigned>();
        rp.alpha = pl.lr / static_cast<float>(pl.Bg);
        rp.jt = jt;
        if (!recon_host_) {
            B2N_CUDA(cudaHostAlloc((void**)&recon_host_, 64, cudaHostAllocMapped));
            B2N_CUDA(cudaHostGetDevicePointer((void**)&recon_host_dev_, recon_host_, 0));
            done_.alloc(64);
        }
        rp.recon_out = nullptr;  // set per direct (zero-copy) launch: a host-mapped store costs the
        rp.done = done_.as<unsigned>();  // device-resident step ~3 us at its end
        rp.bg = (double)pl.Bg;
        rp.G = G_.as<float>();
        rp.grad_only = (dp_ || grad_only_) ? 1 : 0;
        if (std::getenv("B2N_RBM_TRACE")) {
            if (!trace_.p) trace_.alloc(512 * 8);  // two steps (train_stream alternates)
            rp.trace = trace_.as<unsigned long long>();
        }
        // TMA maps: K-major operands of phases 1-3, MN-major ones of phases 2 and 4 (see rbm_fused.cuh),
        // each with its tf32 lo companion
        RbmMaps mp;
        const float* Wl = Wlo_.as<float>();
        const float* Vl = Vlo_[0].as<float>();
        const float* Hl = Hlo_.as<float>();
        mp.vk = make_map_2d(Vc, V, 2 * B, ldv_, 32, 128);
        mp.wk = make_map_2d(W, V, H, ldw_, 32, kRfTileH);
        mp.hsk = make_map_2d(HS_.as<float>(), H, B, ldhs_, 32, 128);
        mp.wmn = make_map_2d(W, V, H, ldw_, 32, 32, true);
        mp.vmn = make_map_2d(Vc, V + 1, 2 * B, ldv_, 32, 32, true);
        mp.hmn = make_map_2d(Hc, H + 1, 2 * B, ldh_, 32, 32, true);
        mp.vk_lo = make_map_2d(Vl, V, 2 * B, ldv_, 32, 128);
        mp.wk_lo = make_map_2d(Wl, V, H, ldw_, 32, kRfTileH);
        mp.wmn_lo = make_map_2d(Wl, V, H, ldw_, 32, 32, true);
        mp.vmn_lo = make_map_2d(Vl, V + 1, 2 * B, ldv_, 32, 32, true);
        mp.hmn_lo = make_map_2d(Hl, H + 1, 2 * B, ldh_, 32, 32, true);
        const double flops = 2.0 * B * H * V * 4, bytes = 4.0 * ((double)H * V * 4 + (double)B * (V + H) * 6);
        pl.ops.push_back(Op([=](cudaStream_t st) {
            launch_ex(rbm_cd1_fused_kernel, dim3(kRfSlices, jt), dim3(kRfThreads), (size_t)kRfSmem, st, 1u, mp, rp);
        }, dp_ || grad_only_ ? "rbm.cd1_fused(grad)" : "rbm.cd1_fused", flops, bytes));
        if (dp_) {  // sum the shards' raw dW / dbh / dbv, then the same update on every replica
            DpComm* dp = dp_.get();
            float* G = G_.as<float>();
            const long long n = nW_;
            const float scale = pl.lr / static_cast<float>(pl.Bg);
            float* Wl2 = Wlo_.as<float>();
            pl.ops.push_back(Op([=](cudaStream_t s) {
                dp->allreduce_f32(G, (size_t)n, s);
                launch_ex(axpy_kernel, dim3(grid_for(n / 4)), dim3(256), 0, s, 1u, reinterpret_cast<float4*>(W),
                          reinterpret_cast<const float4*>(G), n / 4, scale);
                launch_ex(tf32_lo_kernel, dim3(grid_for(n / 4)), dim3(256), 0, s, 1u, reinterpret_cast<const float4*>(W),
                          reinterpret_cast<float4*>(Wl2), n / 4);
            }, "allreduce+update", 0.0, (double)n * 12));
        }
        pl.fused = true;
        pl.rp = rp;
        for (int k = 0; k < kStage; ++k) {  // one map set per visible staging buffer
            pl.maps[k] = mp;
            pl.maps[k].vk = make_map_2d(Vcat_[k].as<float>(), V, 2 * B, ldv_, 32, 128);
            pl.maps[k].vmn = make_map_2d(Vcat_[k].as<float>(), V + 1, 2 * B, ldv_, 32, 32, true);
            pl.maps[k].vk_lo = make_map_2d(Vlo_[k].as<float>(), V, 2 * B, ldv_, 32, 128);
            pl.maps[k].vmn_lo = make_map_2d(Vlo_[k].as<float>(), V + 1, 2 * B, ldv_, 32, 32, true);
        }
        pl.recon_tiles = kRfSlices;
        pl.nk = dp_ ? 2 : 1;
        last_kernels_ = pl.nk;
    }

    void build(Plan& pl) {
        if (fused_ok(pl)) {
            build_fused(pl);
            return;
        }
        const int B = (int)pl.B;
        float* W = W_.as<float>();
        float* G = G_.as<float>();
        float* Vc = Vcat_[0].as<float>();
        float* Hc = Hcat_.as<float>();
        float* HSp = HS_.as<float>();
        double* U = U_.as<double>();
        const int H = (int)H_, V = (int)V_;
        auto hidden = [&](const float* vin, int epi, float* out, long long ldo, const double* u) {
            EpiParams e = epi_default();
            e.C = out;
            e.ldc = ldo;
            e.bias = W + V;
            e.bias_stride = ldw_;
            e.u = u;
            e.ldu = H;
            e.C2 = HSp;
            e.ldc2 = ldhs_;
            GemmLaunch g = plan_gemm(B, H, V, {vin, ldv_, false}, {W, ldw_, false}, epi, e, x3_);
            pl.ops.push_back(gemm_op(g, epi == EPI_RBM_HID ? "rbm.hidden+sample" : "rbm.neg_hidden"));
            ++pl.nk;
        };
        auto visible = [&](double* recon_rows) {
            EpiParams e = epi_default();
            e.C = Vc + (long long)B * ldv_;
            e.ldc = ldv_;
            e.bias = W + (long long)H * ldw_;
            e.bias_stride = 1;
            e.aux = Vc;
            e.ld_aux = ldv_;
            e.row_part = recon_rows;
            e.ld_part = cap_;
            GemmLaunch g = plan_gemm(B, V, H, {HSp, ldhs_, false}, {W, ldw_, true}, EPI_RBM_VIS, e, x3_);
            pl.recon_tiles = (int)g.grid.x;
            pl.ops.push_back(gemm_op(g, "rbm.visible+recon"));
            ++pl.nk;
        };
        // CD-k chain (energy.hpp:137-146): h0 mean + first sample share one GEMM
        hidden(Vc, EPI_RBM_HID, Hc, ldh_, U);
        for (int step = 1; step <= pl.k; ++step) {
            visible(step == 1 ? recon_.as<double>() : recon_.as<double>() + (size_t)cap_ * 32);
            if (step < pl.k) {
                // resample hidden from v_step into HS (h mean scratch: Hcat[B:2B], overwritten below)
                hidden(Vc + (long long)B * ldv_, EPI_RBM_HID, Hc + (long long)B * ldh_, ldh_,
                       U + (size_t)step * B * H);
            }
        }
        hidden(Vc + (long long)B * ldv_, EPI_RBM_NEGHID, Hc + (long long)B * ldh_, ldh_, nullptr);
        // dW / dbh / dbv in one GEMM over K = 2B
        const float scale = pl.lr / static_cast<float>(pl.Bg);
        EpiParams e = epi_default();
        if (dp_ || grad_only_) {
            e.C = G;
            e.ldc = ldw_;
            e.alpha = 1.0f;
        } else {
            e.C = W;
            e.ldc = ldw_;
            e.alpha = scale;
        }
        const bool go = dp_ || grad_only_;
        GemmLaunch g = plan_gemm(H + 1, V + 1, 2 * B, {Hc, ldh_, true}, {Vc, ldv_, true}, go ? EPI_STORE : EPI_AXPY, e,
                                 x3_);
        pl.ops.push_back(gemm_op(g, go ? "rbm.dW" : "rbm.dW+update"));
        ++pl.nk;
        if (dp_) {
            DpComm* dp = dp_.get();
            long long n = nW_;
            pl.ops.push_back(Op([=](cudaStream_t s) {
                dp->allreduce_f32(G, (size_t)n, s);
                launch_ex(axpy_kernel, dim3(grid_for(n / 4)), dim3(256), 0, s, 1u, reinterpret_cast<float4*>(W),
                          reinterpret_cast<const float4*>(G), n / 4, scale);
            }, "allreduce+update", 0.0, (double)n * 12));
            ++pl.nk;
        }
        assign_prefetch(pl.ops);
        last_kernels_ = pl.nk;
    }

    // device alias of a host pointer the GPU can read directly (pinned + mapped under UVA), else null
    static const void* device_alias_v(const void* h) {
        cudaPointerAttributes a;
        if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
    }
    template <class T>
    static const T* device_alias(const T* h) {
        return static_cast<const T*>(device_alias_v(h));
    }

    void prepare(Plan& pl) {
        if (hcol_B_ != pl.B) {  // the +1 / -1 column of Hcat for this batch split
            float* Hc = Hcat_.as<float>();
            const long long B = pl.B;
            set_column_kernel<<<grid_for(B), 256, 0, stream_>>>(Hc, B, ldh_, H_, 1.0f);
            set_column_kernel<<<grid_for(B), 256, 0, stream_>>>(Hc + B * ldh_, B, ldh_, H_, -1.0f);
            B2N_CUDA(cudaGetLastError());
            hcol_B_ = pl.B;
        }
        recon_tiles_ = pl.recon_tiles;
        recon_mapped_ = false;
        if (!pl.fused) {
            wlo_valid_ = false;  // the split path updates W without its lo companion
        } else if (!wlo_valid_) {
            const long long n = nW_;
            launch_ex(tf32_lo_kernel, dim3(grid_for(n / 4)), dim3(256), 0, stream_, 1u,
                      reinterpret_cast<const float4*>(W_.as<float>()), reinterpret_cast<float4*>(Wlo_.as<float>()), n / 4);
            wlo_valid_ = true;
        }
    }

    // the tf32 lo parts of v0 rows [0, B) of visible buffer k (after their copy into Vcat_[k])
    void stage_lo(int k, long long B, cudaStream_t st) {
        const float* Vc = Vcat_[k].as<float>();
        unsigned* fl = vflags_.as<unsigned>() + 16 * k;
        launch_ex(stage_rows_kernel, dim3((unsigned)((V_ + 127) / 128)), dim3(1024), 0, st, 1u, Vc, ldv_, (float*)nullptr,
                  Vlo_[k].as<float>(), ldv_, (int)B, (int)V_, 0, fl);
    }

    void launch(Plan& pl) {
        prepare(pl);
        if (!pl.graph) {
            cudaGraph_t graph;
            B2N_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
            try {
                for (auto& op : pl.ops) op(stream_);
            } catch (...) {
                cudaStreamEndCapture(stream_, &graph);
                throw;
            }
            B2N_CUDA(cudaStreamEndCapture(stream_, &graph));
            B2N_CUDA(cudaGraphInstantiate(&pl.graph, graph, 0));
            cudaGraphDestroy(graph);
        }
        B2N_CUDA(cudaGraphLaunch(pl.graph, stream_));
    }

    long long H_, V_;
    int device_;
    bool x3_;
    cudaStream_t stream_ = nullptr;
    long long ldw_ = 0, nW_ = 0, ldv_ = 0, ldh_ = 0, ldhs_ = 0;
    long long cap_ = 0;
    int kcap_ = 0;
    DevMem W_, G_, Hcat_, HS_, U_, recon_;
    DevMem Vcat_[kStage];      // [v0; v1] (+ ones column): buffer 0 for every path, 0..3 in rotation for train_stream
    DevMem Wlo_, Vlo_[kStage], Hlo_;  // tf32 lo parts of W_aug / Vcat / Hcat (the fused step's 3xTF32 operands)
    int vb_ = 0;               // the Vcat buffer of the last step
    DevMem vflags_;            // per visible buffer: 16 slice flags "v0 not exact in tf32" (stage_rows_kernel)
    bool wlo_valid_ = false;   // Wlo_ matches W_ (kept by the fused step; anything else that writes W clears it)
    DevMem fused_ws_, gbar_, trace_;
    HostPinned ubuf_[2];       // train_epoch: double-buffered uniforms
    cudaEvent_t uev_[2] = {nullptr, nullptr};
    DevMem racc_;              // train_epoch: device sum of per-step reconstruction errors
    DevMem su_[kStage];        // train_stream: device staging of the uniforms, kStage deep
    DevMem rstream_;           // train_stream: per-step reconstruction errors
    DevMem sready_;            // train_stream: staging readiness flags (step index + 1 per buffer)
    cudaEvent_t ev_used_[kStage] = {};
    cudaEvent_t ev_rng_[kStage] = {};
    cudaStream_t copy_stream_ = nullptr;
    DevRng rng_;               // the device copy of the caller's std::mt19937 (u == null steps)
  public:
    void read_trace(unsigned long long* h) {
        B2N_CUDA(cudaDeviceSynchronize());
        if (trace_.p) B2N_CUDA(cudaMemcpy(h, trace_.p, 512 * 8, cudaMemcpyDeviceToHost));
    }
  private:  // fused CD-1 kernel: phase-2 partials, grid-barrier counters
    HostPinned h_recon_;
    long long staged_B_ = 0, last_B_ = 0, last_Bg_ = 0;
    int staged_k_ = 1;
    int last_kernels_ = 0;
    int recon_tiles_ = 1;
    bool recon_mapped_ = false;
    double* recon_host_ = nullptr;      // cudaHostAllocMapped: the fused step's recon
    double* recon_host_dev_ = nullptr;  // its device alias
    DevMem done_;
    long long hcol_B_ = -1;
    std::vector<std::unique_ptr<Plan>> plans_;
    std::unique_ptr<DpComm> dp_;
    bool grad_only_ = false;
};

}  // namespace b2n
