// crbm.cuh -- device-resident replacement of fastnn::Crbm + crbm_cd_update (energy.hpp:245-376),
// binary units, non-pooled formulation. One CD-1 step is five launches of the implicit-GEMM
// tcgen05 conv kernels (conv.cuh) and one reduction, captured as a CUDA graph:
//
//   h0/hs : FWD   Vc[0:B]  (*) K, epilogue h0 = sigmoid(acc + bh) -> Hc[0:B], hs = (u < h0) -> HS
//   v1    : DGRAD HS (full conv) K^T, epilogue v1 = sigmoid(acc + bv) -> Vc[B:2B], per-warp
//           partials of sum(v0 - v1) and sum((v0 - v1)^2) (bv update, sq_diff_per_row)
//   h1    : FWD   Vc[B:2B] (*) K, epilogue -sigmoid(acc + bh) -> Hc[B:2B]
//   stats : WGRAD over the 2B concatenated images: sum corr(v, h) = pos - neg (crbm_corr_stats,
//           energy.hpp:316-329) and, through the ones row, sum(h0 - h1) per kernel
//   update: fixed-order reduction of the WGRAD partials and the visible partials, then
//           K += lr/B (pos - neg), bh += lr/B sum(h0 - h1), bv += lr/B sum(v0 - v1), recon / B
//
// Parameters live in one buffer P = [K (k,c,kh,kw) | bh (k) | bv (c)]. Envelope of the conv
// kernels: k, c <= 32, c*kh*kw <= 320, k*kh*kw <= 320 (ShapeError outside it -- no fallback).
//
// When an image's whole chain fits in shared memory (kw <= 8, <= 200 KB), the step is instead ONE
// launch of crbm_cd1_fused_kernel (crbm_fused.cuh: a CTA per image, FFMA register strips, last-CTA
// fixed-order reduction) -- the product path for the few-channel CRBM shapes, where N = c_in makes
// the tensor-core dgrad mostly padding. B2N_CRBM_FUSED=0 forces the split path.
#pragma once
#include "mt19937.cuh"
#include <random>

#include "conv.cuh"
#include "crbm_fused.cuh"
#include "nccl_dyn.cuh"
#include "network.cuh"

namespace b2n {

// crbm_cd_update's parameter updates (energy.hpp:353-374) from the step's partials, in a fixed
// order (deterministic, independent of the launch geometry of the producing kernels).
//   blocks [0, ckk]: WGRAD partial rows (patch rows + the ones row) -> K / bh
//   block ckk + 1  : visible partials -> bv, and the reconstruction error -> *recon
static __global__ void crbm_update_kernel(const float* __restrict__ ws, int chunks, int ckk, int kout,
                                          const float* __restrict__ vstat_f, const double* __restrict__ vstat_d,
                                          int nstat, int cin, float* P, float scale, double inv_bg, double* recon) {
    pdl_wait();
    const int j = blockIdx.x;
    if (j <= ckk) {
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
        float* dst = j < ckk ? P + (long long)n * ckk + j : P + (long long)kout * ckk + n;
        *dst += scale * s;
        return;
    }
    // visible bias + reconstruction: 256 threads stride the partials, then a fixed smem tree
    __shared__ float sf[256];
    __shared__ double sd[256];
    float* bv = P + (long long)kout * ckk + kout;
    double rsum = 0.0;
    for (int c = 0; c < cin; ++c) {
        float a = 0.0f;
        double d = 0.0;
        for (int i = threadIdx.x; i < nstat; i += 256) {
            a += vstat_f[(long long)i * cin + c];
            d += vstat_d[(long long)i * cin + c];
        }
        sf[threadIdx.x] = a;
        sd[threadIdx.x] = d;
        __syncthreads();
        for (int o = 128; o > 0; o >>= 1) {
            if (threadIdx.x < o) {
                sf[threadIdx.x] += sf[threadIdx.x + o];
                sd[threadIdx.x] += sd[threadIdx.x + o];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            bv[c] += scale * sf[0];
            rsum += sd[0];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *recon = rsum * inv_bg;
}

class Crbm {
  public:
    Crbm(int c, int h, int w, int k, int kh, int kw, int device, int precision)
        : device_(device), x3_(precision == B2N_TF32X3) {
        if (c < 1 || h < 1 || w < 1 || k < 1 || kh < 1 || kw < 1) throw Error(B2N_ESHAPE, "crbm extents must be positive");
        if (kh > h || kw > w) throw Error(B2N_ESHAPE, "crbm: kernel extents exceed visible extents");  // energy.hpp:257
        g_.c = c;
        g_.h = h;
        g_.w = w;
        g_.k = k;
        g_.kh = kh;
        g_.kw = kw;
        g_.pad = 0;
        g_.oh = h - kh + 1;
        g_.ow = w - kw + 1;
        conv_np(k);  // envelope checks (throw ShapeError)
        conv_np(c);
        conv_base(g_, 1, ACT_SIGMOID, false);
        ckk_ = (long long)c * kh * kw;
        nP_ = round_up((long long)k * ckk_ + k + c, 32);
        B2N_CUDA(cudaSetDevice(device));
        B2N_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
        P_.alloc(nP_ * 4);
        recon_.alloc(64);
    }
    ~Crbm() {
        plans_.clear();
        for (int j = 0; j < kCrbmStage; ++j)
            for (cudaEvent_t e : {ev_used_[j], ev_rng_[j], ev_ready_[j]})
                if (e) cudaEventDestroy(e);
        if (copy_stream_) cudaStreamDestroy(copy_stream_);
        if (stream_) cudaStreamDestroy(stream_);
    }

    // Crbm::init (energy.hpp:261): glorot_fill(kernels, c*kh*kw, k*kh*kw); biases stay zero
    void init(unsigned seed) {
        std::mt19937 rng(seed);
        const float limit = std::sqrt(6.0f / static_cast<float>(ckk_ + (long long)g_.k * g_.kh * g_.kw));
        UniformF32 dist(-limit, limit);
        std::vector<float> ker((size_t)(g_.k * ckk_));
        for (float& v : ker) v = dist(rng);
        std::vector<float> zk((size_t)g_.k, 0.0f), zc((size_t)g_.c, 0.0f);
        set(ker.data(), zc.data(), zk.data());
    }
    void set(const float* ker, const float* bv, const float* bh) {
        float* P = P_.as<float>();
        const long long nk = g_.k * ckk_;
        if (ker) B2N_CUDA(cudaMemcpyAsync(P, ker, nk * 4, cudaMemcpyHostToDevice, stream_));
        if (bh) B2N_CUDA(cudaMemcpyAsync(P + nk, bh, (size_t)g_.k * 4, cudaMemcpyHostToDevice, stream_));
        if (bv) B2N_CUDA(cudaMemcpyAsync(P + nk + g_.k, bv, (size_t)g_.c * 4, cudaMemcpyHostToDevice, stream_));
        B2N_CUDA(cudaStreamSynchronize(stream_));
    }
    void get(float* ker, float* bv, float* bh) {
        const float* P = P_.as<float>();
        const long long nk = g_.k * ckk_;
        if (ker) B2N_CUDA(cudaMemcpyAsync(ker, P, nk * 4, cudaMemcpyDeviceToHost, stream_));
        if (bh) B2N_CUDA(cudaMemcpyAsync(bh, P + nk, (size_t)g_.k * 4, cudaMemcpyDeviceToHost, stream_));
        if (bv) B2N_CUDA(cudaMemcpyAsync(bv, P + nk + g_.k, (size_t)g_.c * 4, cudaMemcpyDeviceToHost, stream_));
        B2N_CUDA(cudaStreamSynchronize(stream_));
    }

    // A stream of crbm_cd_update steps over host batches (the caller's loop, energy.hpp:333): step i
    // takes images [i B, (i + 1) B) of v0 and, with u == null, its draws from the device generator --
    // generated `gens` steps ahead with jump-ahead start states (mt19937.cuh), the 691,200 draws of a
    // MNIST-shape step taking ~450 us on one SM. The H2D of the next steps overlaps the current one.
    void train_stream(const float* v0, const double* u, long long steps, long long B, float lr, double* recon_out) {
        if (dp_) throw Error(B2N_EPARAM, "train_stream: data-parallel CRBMs step through run_staged");
        if (steps < 1 || B < 1) throw Error(B2N_ESHAPE, "train_stream: need steps >= 1 and batch >= 1");
        ensure_capacity(B);
        Plan& pl = plan_for(B, lr, B);
        if (!pl.fused || pl.keep) {  // the split path: staged copies + the step graph, in order
            for (long long i = 0; i < steps; ++i) {
                stage(v0 + i * B * vpix(), u ? u + i * B * hpix() : nullptr, B);
                run_staged(1, lr, B);
                recon_out[i] = recon();
            }
            return;
        }
        constexpr int kS = kCrbmStage;  // as deep as the generators in flight (one step's draws: ~550 us)
        for (int j = 0; j < kS; ++j) {
            if (sv_[j].bytes < (size_t)(B * vpix() * 4)) sv_[j].alloc((size_t)(B * vpix() * 4));
            if (su_[j].bytes < (size_t)(B * hpix() * 8)) su_[j].alloc((size_t)(B * hpix() * 8));
            for (cudaEvent_t* e : {&ev_used_[j], &ev_rng_[j], &ev_ready_[j]})
                if (!*e) B2N_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        }
        if (!copy_stream_) B2N_CUDA(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));
        // per-step recon slots, grown geometrically (no allocation inside a later, longer stream)
        if (rstream_.bytes < (size_t)steps * 8) rstream_.alloc(std::max<size_t>((size_t)steps * 8 * 2, 8192));
        for (int j = 0; j < kS; ++j) B2N_CUDA(cudaEventRecord(ev_used_[j], stream_));
        if (!u) rng_.stream_begin(B * hpix(), stream_, 24);
        for (long long i = 0; i < steps; ++i) {
            const int j = (int)(i % kS);
            B2N_CUDA(cudaStreamWaitEvent(copy_stream_, ev_used_[j], 0));
            B2N_CUDA(cudaMemcpyAsync(sv_[j].p, v0 + i * B * vpix(), (size_t)(B * vpix() * 4), cudaMemcpyDefault,
                                     copy_stream_));
            if (u)
                B2N_CUDA(cudaMemcpyAsync(su_[j].p, u + i * B * hpix(), (size_t)(B * hpix() * 8), cudaMemcpyDefault,
                                         copy_stream_));
            else {
                rng_.stream_step((int)i, (int)steps, su_[j].as<double>(), ev_used_[j], ev_rng_[j]);
                B2N_CUDA(cudaStreamWaitEvent(copy_stream_, ev_rng_[j], 0));
            }
            B2N_CUDA(cudaEventRecord(ev_ready_[j], copy_stream_));
            B2N_CUDA(cudaStreamWaitEvent(stream_, ev_ready_[j], 0));
            CrbmFusedParams fp = pl.fp;
            fp.v0 = sv_[j].as<float>();
            fp.u = su_[j].as<double>();
            fp.recon = rstream_.as<double>() + i;
            launch_ex(pl.fkern, dim3(pl.fgrid), dim3(kCfThreads), pl.fsmem, stream_, 1u, fp);
            B2N_CUDA(cudaEventRecord(ev_used_[j], stream_));
        }
        if (!u) rng_.stream_end((int)steps, stream_);
        B2N_CUDA(cudaMemcpyAsync(recon_out, rstream_.p, (size_t)steps * 8, cudaMemcpyDeviceToHost, stream_));
        spin_sync(stream_);
        last_B_ = B;
        last_kept_ = false;
    }

    // crbm_cd_update (energy.hpp:333) with the uniforms supplied: u[B][k][oh][ow]
    double cd_update(const float* v0, long long B, float lr, const double* u, long long Bg) {
        stage(v0, u, B);
        run_staged(1, lr, Bg);
        return recon();
    }
    void stage(const float* v0, const double* u, long long B) {
        if (B < 1) throw Error(B2N_ESHAPE, "crbm_cd_update: batch must be >= 1");
        ensure_capacity(B);
        B2N_CUDA(cudaMemcpyAsync(Vc_.p, v0, (size_t)(B * vpix()) * 4, cudaMemcpyHostToDevice, stream_));
        if (u)
            B2N_CUDA(cudaMemcpyAsync(U_.p, u, (size_t)(B * hpix()) * 8, cudaMemcpyHostToDevice, stream_));
        else  // u == null: the B * k * oh * ow draws from the device generator (set_rng)
            rng_.draw(U_.as<double>(), B * hpix(), stream_);
        staged_B_ = B;
    }
    void run_staged(int steps, float lr, long long Bg) {
        if (!staged_B_) throw Error(B2N_EPARAM, "run_staged before stage");
        Plan& pl = plan_for(staged_B_, lr, Bg ? Bg : staged_B_);
        for (int s = 0; s < steps; ++s) launch(pl);
        last_B_ = staged_B_;
        last_kept_ = pl.fused ? pl.keep : true;
    }
    double recon() {
        double r = 0.0;
        B2N_CUDA(cudaMemcpyAsync(h_recon_.p, recon_.p, 8, cudaMemcpyDeviceToHost, stream_));
        spin_sync(stream_);
        std::memcpy(&r, h_recon_.p, 8);
        return r;
    }
    // chain states of the last step (h0 mean, h sample, v1 mean, h1 mean), NCHW
    void last_states(float* h0, float* hs, float* v1, float* h1) {
        if (!last_kept_) throw Error(B2N_EPARAM, "crbm last_states: enable keep_states before the step");
        const long long B = last_B_, hp = hpix(), vp = vpix();
        const float* Hc = Hc_.as<float>();
        const auto D2H = cudaMemcpyDeviceToHost;
        if (h0) B2N_CUDA(cudaMemcpyAsync(h0, Hc, B * hp * 4, D2H, stream_));
        if (hs) B2N_CUDA(cudaMemcpyAsync(hs, HS_.p, B * hp * 4, D2H, stream_));
        if (v1) B2N_CUDA(cudaMemcpyAsync(v1, Vc_.as<float>() + B * vp, B * vp * 4, D2H, stream_));
        if (h1) B2N_CUDA(cudaMemcpyAsync(h1, Hc + B * hp, B * hp * 4, D2H, stream_));
        B2N_CUDA(cudaStreamSynchronize(stream_));
        if (h1)
            for (long long i = 0; i < B * hp; ++i) h1[i] = -h1[i];  // stored negated for the statistics
    }
    // the caller's std::mt19937 (625 words: state, position) for the steps that take no uniforms
    void set_rng(const uint32_t* st) { rng_.load(st, stream_); }
    void get_rng(uint32_t* st) { rng_.store(st, stream_); }
    cudaStream_t stream() const { return stream_; }
    void dp_init(const char id[128], int rank, int world) {
        dp_ = std::make_unique<DpComm>();
        dp_->init(id, rank, world);
        plans_.clear();
    }
    int kernels_per_step() const { return last_kernels_; }
    // write the chain states of every step (h0, hs, v1, -h1) to HBM for last_states (the fused
    // step otherwise keeps them in shared memory only)
    void keep_states(bool on) { keep_states_ = on; }
    std::vector<OpStats> profile(int steps, float lr, long long Bg) {
        if (!staged_B_) throw Error(B2N_EPARAM, "profile before stage");
        Plan& pl = plan_for(staged_B_, lr, Bg ? Bg : staged_B_);
        return profile_ops(pl.ops, steps, stream_);
    }

  private:
    struct Plan {
        long long B, Bg;
        float lr;
        bool keep = false, fused = false;
        std::vector<Op> ops;
        std::shared_ptr<DevMem> ws, vf, vd;
        cudaGraphExec_t graph = nullptr;
        CrbmFusedParams fp;  // the one-launch step (fused plans)
        int fgrid = 0;
        size_t fsmem = 0;
        void (*fkern)(CrbmFusedParams) = nullptr;
        ~Plan() {
            if (graph) cudaGraphExecDestroy(graph);
        }
    };
    long long vpix() const { return (long long)g_.c * g_.h * g_.w; }
    long long hpix() const { return (long long)g_.k * g_.oh * g_.ow; }

    void ensure_capacity(long long B) {
        if (B <= cap_) return;
        cap_ = B;
        plans_.clear();
        Vc_.alloc((size_t)(2 * B * vpix()) * 4);
        Hc_.alloc((size_t)(2 * B * hpix()) * 4);
        HS_.alloc((size_t)(B * hpix()) * 4);
        U_.alloc((size_t)(B * hpix()) * 8);
        if (!h_recon_.p) h_recon_.alloc(64);
    }

    Plan& plan_for(long long B, float lr, long long Bg) {
        for (auto& p : plans_)
            if (p->B == B && p->lr == lr && p->Bg == Bg && p->keep == keep_states_) return *p;
        auto pl = std::make_unique<Plan>();
        pl->B = B;
        pl->lr = lr;
        pl->Bg = Bg;
        pl->keep = keep_states_;
        build(*pl);
        plans_.push_back(std::move(pl));
        return *plans_.back();
    }

    bool fused_ok() const {
        const char* e = std::getenv("B2N_CRBM_FUSED");
        if (e && e[0] == '0') return false;
        return g_.kw <= 8 && g_.c <= 64 && crbm_fused_smem(g_.c, g_.h, g_.w, g_.k, g_.kh, g_.kw) <= 200 * 1024;
    }

    template <int KW>
    void build_fused_kw(Plan& pl) {
        const ConvGeom& g = g_;
        const size_t smem = crbm_fused_smem(g.c, g.h, g.w, g.k, g.kh, g.kw);
        B2N_CUDA(cudaFuncSetAttribute(crbm_cd1_fused_kernel<KW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        int occ = 0;
        B2N_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, crbm_cd1_fused_kernel<KW>, kCfThreads, smem));
        const int grid = (int)std::min<long long>(pl.B, (long long)sm_count() * std::max(occ, 1));
        const long long np = g.k * ckk_ + g.k + g.c;
        pl.ws = std::make_shared<DevMem>();
        pl.ws->alloc((size_t)(pl.B * round_up(np, 4)) * 4);
        pl.vd = std::make_shared<DevMem>();
        pl.vd->alloc((size_t)pl.B * 8 + 64);
        CrbmFusedParams p;
        std::memset(&p, 0, sizeof(p));
        p.C = g.c;
        p.H = g.h;
        p.W = g.w;
        p.K = g.k;
        p.KH = g.kh;
        p.KW = g.kw;
        p.OH = g.oh;
        p.OW = g.ow;
        p.HP = g.oh + 2 * (g.kh - 1);
        const CrbmPitches q = crbm_pitches(g.w, g.ow, g.kw);
        p.VP = q.VP;
        p.OP = q.OP;
        p.HPP = q.HPP;
        p.B = (int)pl.B;
        p.npart = (int)np;
        p.v0 = Vc_.as<float>();
        p.u = U_.as<double>();
        p.P = P_.as<float>();
        p.ws = pl.ws->as<float>();
        p.rws = pl.vd->as<double>();
        p.ticket = reinterpret_cast<unsigned*>(recon_.as<double>() + 1);
        p.recon = recon_.as<double>();
        p.scale = pl.lr / static_cast<float>(pl.Bg);
        p.inv_bg = 1.0 / (double)pl.Bg;
        p.stage_floats = (long long)(smem / 4) - round_up(np, 4) - 16;
        p.ws_pitch = (int)round_up(np, 4);
        p.trace = TraceRegistry::get().next();
        if (dp_) {
            pl.vf = std::make_shared<DevMem>();  // [G (npart floats) | pad | Gd (double)]
            pl.vf->alloc((size_t)(round_up(np, 2) * 4 + 64));
            p.G = pl.vf->as<float>();
            p.Gd = reinterpret_cast<double*>(p.G + round_up(np, 2));
        }
        if (pl.keep) {
            p.h0_out = Hc_.as<float>();
            p.h1_out = Hc_.as<float>() + pl.B * hpix();
            p.hs_out = HS_.as<float>();
            p.v1_out = Vc_.as<float>() + pl.B * vpix();
        }
        const double fl = 2.0 * pl.B * (3.0 * hpix() * ckk_ + (double)vpix() * g.k * g.kh * g.kw + 2.0 * hpix() * ckk_);
        const double by = 4.0 * pl.B * vpix() + 8.0 * pl.B * hpix() + 8.0 * np + 4.0 * 2 * pl.B * np;
        pl.ops.push_back(Op([=](cudaStream_t st) {
            launch_ex(crbm_cd1_fused_kernel<KW>, dim3(grid), dim3(kCfThreads), smem, st, 1u, p);
        }, "crbm.cd1_fused", fl, by));
        pl.fp = p;  // train_stream relaunches it with each step's buffers
        pl.fgrid = grid;
        pl.fsmem = smem;
        pl.fkern = crbm_cd1_fused_kernel<KW>;
        if (dp_) {  // one exchange step: the shards' parameter sums and recon sums, then the update
            DpComm* dp = dp_.get();
            float* G = p.G;
            double* Gd = p.Gd;
            float* P = p.P;
            double* rc = p.recon;
            const int n = (int)np;
            const float scale = p.scale;
            const double inv_bg = p.inv_bg;
            pl.ops.push_back(Op([=](cudaStream_t st) {
                dp->allreduce_f32(G, (size_t)n, st);
                dp->allreduce_f64(Gd, 1, st);
                launch_ex(crbm_dp_apply_kernel, dim3((n + 255) / 256), dim3(256), 0, st, 1u, P, (const float*)G, n, scale,
                          (const double*)Gd, rc, inv_bg);
            }, "allreduce+update", 0.0, 12.0 * np));
        }
        pl.fused = true;
    }

    void build(Plan& pl) {
        if (dp_ && !fused_ok())
            throw Error(B2N_EPARAM, "data-parallel CRBM steps need the one-launch kernel's shape envelope");
        if (fused_ok()) {
            switch (g_.kw) {
                case 1: build_fused_kw<1>(pl); break;
                case 2: build_fused_kw<2>(pl); break;
                case 3: build_fused_kw<3>(pl); break;
                case 4: build_fused_kw<4>(pl); break;
                case 5: build_fused_kw<5>(pl); break;
                case 6: build_fused_kw<6>(pl); break;
                case 7: build_fused_kw<7>(pl); break;
                default: build_fused_kw<8>(pl); break;
            }
            last_kernels_ = dp_ ? 2 : 1;
            return;
        }
        last_kernels_ = 5;
        const int B = (int)pl.B;
        const ConvGeom& g = g_;
        float* P = P_.as<float>();
        float* bh = P + g.k * ckk_;
        float* bv = bh + g.k;
        float* Vc = Vc_.as<float>();
        float* Hc = Hc_.as<float>();
        const long long vp = vpix(), hp = hpix();
        const int sms = sm_count();
        // hidden given visible (crbm_hidden_preact + unit mean / sample)
        auto hidden = [&](const float* vin, float* hout, bool sample, bool neg, const char* name) {
            ConvParams p = conv_base(g, B, ACT_SIGMOID, false);
            p.x = vin;
            p.ldx = vp;
            p.wk = P;
            p.bias = bh;
            p.y = hout;
            p.ldy = hp;
            p.npix = (long long)B * g.oh * g.ow;
            p.items = (int)((p.npix + 127) / 128);
            p.kblocks = (p.ckk + 31) / 32;
            p.neg_out = neg ? 1 : 0;
            if (sample) {
                p.u = U_.as<double>();
                p.ys = HS_.as<float>();
            }
            const int np = conv_np(g.k), grid = std::min(p.items, sms);
            const bool x3 = x3_;
            const double fl = 2.0 * p.npix * g.k * p.ckk;
            const double by = 4.0 * (B * vp + B * hp * (sample ? 2 : 1) + g.k * (p.ckk + 1)) + (sample ? 8.0 * B * hp : 0);
            pl.ops.push_back(Op([=](cudaStream_t st) { launch_conv<CONV_FWD>(p, np, x3, grid, st); }, name, fl, by));
        };
        hidden(Vc, Hc, true, false, "crbm.hidden+sample");
        // visible given hidden sample (crbm_visible_preact + unit mean) + bias / recon partials
        ConvParams pd = conv_base(g, B, ACT_SIGMOID, false);
        pd.dz = HS_.as<float>();
        pd.wk = P;
        pd.x = Vc;
        pd.ldx = vp;
        pd.dx = Vc + B * vp;
        pd.lddx = vp;
        pd.dg_bias = bv;
        pd.dg_act = ACT_SIGMOID;
        pd.npix = (long long)B * g.h * g.w;
        pd.items = (int)((pd.npix + 127) / 128);
        pd.kblocks = (pd.kkk + 31) / 32;
        const int nstat = pd.items * 4;
        pl.vf = std::make_shared<DevMem>();
        pl.vf->alloc((size_t)nstat * g.c * 4);
        pl.vd = std::make_shared<DevMem>();
        pl.vd->alloc((size_t)nstat * g.c * 8);
        pd.vstat_f = pl.vf->as<float>();
        pd.vstat_d = pl.vd->as<double>();
        {
            const int np = conv_np(g.c), grid = std::min(pd.items, sms);
            const bool x3 = x3_;
            const double fl = 2.0 * pd.npix * g.c * pd.kkk;
            const double by = 4.0 * (B * hp + 2 * B * vp + g.k * ckk_ + g.c);
            pl.ops.push_back(
                Op([=](cudaStream_t st) { launch_conv<CONV_DGRAD>(pd, np, x3, grid, st); }, "crbm.visible+stats", fl, by));
        }
        hidden(Vc + B * vp, Hc + B * hp, false, true, "crbm.neg_hidden");
        // pos - neg statistics over the 2B concatenated images (+ the ones row: sum(h0 - h1))
        ConvParams pw = conv_base(g, 2 * B, ACT_SIGMOID, false);
        pw.x = Vc;
        pw.ldx = vp;
        pw.dz = Hc;
        pw.npix = 2LL * B * g.oh * g.ow;
        pw.mtiles_w = (int)((ckk_ + 1 + 127) / 128);
        const long long want_items = 2LL * sms;
        long long chunks = std::max<long long>(1, want_items / pw.mtiles_w);
        long long chunk_px = (pw.npix + chunks - 1) / chunks;
        chunk_px = std::max<long long>(32, (chunk_px + 31) / 32 * 32);
        chunks = (pw.npix + chunk_px - 1) / chunk_px;
        pw.chunk_px = (int)chunk_px;
        pw.chunks = (int)chunks;
        pw.items = (int)(pw.mtiles_w * chunks);
        pw.kblocks = (int)(chunk_px / 32);
        pl.ws = std::make_shared<DevMem>();
        pl.ws->alloc((size_t)pw.items * 128 * 32 * 4);
        pw.ws = pl.ws->as<float>();
        {
            const int grid = std::min(pw.items, sms);
            const bool x3 = x3_;
            const double fl = 2.0 * pw.npix * g.k * (ckk_ + 1);
            const double by = 4.0 * 2 * B * (vp + hp) + 4.0 * pw.items * 128 * 32;
            pl.ops.push_back(
                Op([=](cudaStream_t st) { launch_conv<CONV_WGRAD>(pw, 32, x3, grid, st); }, "crbm.stats", fl, by));
        }
        {
            const float* ws = pw.ws;
            const int ch = pw.chunks, ckk = (int)ckk_, kout = g.k, cin = g.c;
            const float* vf = pd.vstat_f;
            const double* vd = pd.vstat_d;
            const float scale = pl.lr / static_cast<float>(pl.Bg);
            const double inv_bg = 1.0 / (double)pl.Bg;
            double* rc = recon_.as<double>();
            const double by = 4.0 * pw.items * 128 * 32 + 12.0 * nstat * g.c + 8.0 * (g.k * ckk_ + g.k + g.c);
            pl.ops.push_back(Op([=](cudaStream_t st) {
                launch_ex(crbm_update_kernel, dim3(ckk + 2), dim3(256), 0, st, 1u, ws, ch, ckk, kout, vf, vd, nstat, cin,
                          P, scale, inv_bg, rc);
            }, "crbm.update", 0.0, by));
        }
    }

    void launch(Plan& pl) {
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

    ConvGeom g_;
    int device_;
    bool x3_;
    long long ckk_ = 0, nP_ = 0, cap_ = 0;
    long long staged_B_ = 0, last_B_ = 0;
    bool keep_states_ = false, last_kept_ = false;
    int last_kernels_ = 1;
    cudaStream_t stream_ = nullptr;
    DevMem P_, Vc_, Hc_, HS_, U_, recon_;
    DevRng rng_;
    static constexpr int kCrbmStage = 24;
    DevMem sv_[kCrbmStage], su_[kCrbmStage], rstream_;  // train_stream: rotating v0 / draw buffers, per-step recon
    cudaEvent_t ev_used_[kCrbmStage] = {}, ev_rng_[kCrbmStage] = {}, ev_ready_[kCrbmStage] = {};
    cudaStream_t copy_stream_ = nullptr;
    HostPinned h_recon_;
    std::vector<std::unique_ptr<Plan>> plans_;
    std::unique_ptr<DpComm> dp_;
};

}  // namespace b2n
