// network.cuh -- device-resident replacement of fastnn::Network / train_minibatch
// (network.hpp:236-472). The layer list is planned once per (batch, global batch) into a fixed
// launch sequence, captured as one CUDA graph:
//
//   dense + activation       -> 1 tcgen05 GEMM, bias+act epilogue            (dense_forward+activation_apply)
//   last dense + softmax     -> 1 tcgen05 GEMM, softmax-xent epilogue         (+softmax_cross_entropy, argmax)
//   backward, per dense l    -> dX GEMM with act' epilogue (skipped for l=0: its dX is dead)
//                               dW GEMM over [X | 1] with the SGD-momentum epilogue (gradient of w and b
//                               in one GEMM: the ones column yields the bias gradient)
//   conv + act + maxpool     -> conv.cuh implicit-GEMM kernels
//
// Parameters live in one packed buffer: a dense layer is W_aug (out x ldw) with b in column `in`,
// so the forward bias and the SGD update of b ride on the W tiles. Velocity and gradient buffers
// mirror that layout, which makes the data-parallel allreduce a single NCCL call and the optimizer
// one vectorised pass.
#pragma once
#include <algorithm>
#include <chrono>
#include <functional>
#include <string>
#include <map>
#include <memory>
#include <random>

#include "conv.cuh"
#include "checkpoint.cuh"
#include "convx.cuh"
#include "nccl_dyn.cuh"
#include "runtime.cuh"

namespace b2n {

// one planned launch (or short launch sequence) of a step, with its algorithmic work
struct Op {
    std::function<void(cudaStream_t)> fn;
    std::string name;
    double flops = 0, bytes = 0;
    int kernels = 1;
    int branch = 0;  // 1: captured on the side stream after a fork from the main stream (a dense
                     // wgrad+SGD off the critical path), joined at the end of the graph
    bool is_gemm = false;
    GemmLaunch gemm;  // when is_gemm: launched directly (its PDL prefetch flags are per op list)
    Op() = default;
    template <class F>
    Op(F f, std::string n = "op", double fl = 0, double by = 0, int k = 1)
        : fn(std::move(f)), name(std::move(n)), flops(fl), bytes(by), kernels(k) {}
    void operator()(cudaStream_t s) const {
        if (is_gemm)
            gemm.run(s);
        else
            fn(s);
    }
};
inline Op gemm_op(const GemmLaunch& g, const std::string& name) {
    Op o;
    o.name = name;
    o.flops = g.flops;
    o.bytes = g.bytes;
    o.is_gemm = true;
    o.gemm = g;
    return o;
}
// PDL prefetch analysis over one captured op list: a GEMM operand may be loaded before
// griddepcontrol.wait iff the immediately preceding op OF THE SAME STREAM does not write it (kernel
// N-2 has always completed when kernel N launches). Non-GEMM ops count as writing everything; ops on
// the side branch (fork / join through events) never prefetch.
// B2N_BRANCH=0 keeps every op of the step on one stream (A/B measurement of the fork)
inline bool branch_wgrad() {
    static const bool on = [] {
        const char* e = std::getenv("B2N_BRANCH");
        return !(e && e[0] == '0');
    }();
    return on;
}
inline void assign_prefetch(std::vector<Op>& ops) {
    const Op* prev_main = nullptr;
    for (size_t i = 0; i < ops.size(); ++i) {
        Op& op = ops[i];
        if (op.branch) {
            if (op.is_gemm) op.gemm.p.pre_a = op.gemm.p.pre_b = 0;
            continue;
        }
        const Op* prev = prev_main;
        prev_main = &op;
        if (!op.is_gemm) continue;
        GemmLaunch& g = op.gemm;
        if (!prev) {  // first main-stream node of a graph: no in-graph predecessor
            g.p.pre_a = g.p.pre_b = i == 0 ? 1 : 0;
            continue;
        }
        if (!prev->is_gemm) {
            g.p.pre_a = g.p.pre_b = 0;
            continue;
        }
        bool wa = false, wb = false;
        for (const auto& w : prev->gemm.writes) {
            wa = wa || overlaps(w, g.a_rng);
            wb = wb || overlaps(w, g.b_rng);
        }
        g.p.pre_a = !wa;
        g.p.pre_b = !wb;
    }
}

// per-op device time of `steps` un-graphed runs of an op list (CUDA events between ops)
struct OpStats {
    std::string name;
    double ms = 0, flops = 0, bytes = 0;
    int kernels = 1;
};
inline std::vector<OpStats> profile_ops(const std::vector<Op>& ops, int steps, cudaStream_t st) {
    std::vector<cudaEvent_t> ev(ops.size() + 1);
    for (auto& e : ev) B2N_CUDA(cudaEventCreate(&e));
    std::vector<OpStats> out(ops.size());
    for (size_t i = 0; i < ops.size(); ++i) out[i] = {ops[i].name, 0.0, ops[i].flops, ops[i].bytes, ops[i].kernels};
    for (int s = 0; s < steps + 1; ++s) {  // first pass warms up
        for (size_t i = 0; i < ops.size(); ++i) {
            B2N_CUDA(cudaEventRecord(ev[i], st));
            ops[i](st);
        }
        B2N_CUDA(cudaEventRecord(ev[ops.size()], st));
        B2N_CUDA(cudaEventSynchronize(ev[ops.size()]));
        if (s == 0) continue;
        for (size_t i = 0; i < ops.size(); ++i) {
            float ms = 0;
            B2N_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
            out[i].ms += ms / steps;
        }
    }
    for (auto& e : ev) cudaEventDestroy(e);
    return out;
}

struct ParamView {  // one fastnn ParamRef (w or b of a layer) inside the packed buffers
    std::vector<long long> dims;
    long long off;      // float offset of element (0,0) in the packed buffers
    long long rows, cols, pitch;  // 2-D view: rows x cols with row pitch (floats)
};

inline long long numel(const std::vector<long long>& s) {
    long long n = 1;
    for (long long e : s) n *= e;
    return n;
}

// ---- device-resident epoch loop (fit / evaluate, network.hpp:474-511, data.hpp:243-266): the dataset
// lives in HBM, each batch is gathered on the device in the shuffled order, and a device-side batch
// cursor lets one CUDA graph (gather + step + loss / accuracy accumulation) be relaunched per batch
// with no host synchronisation inside an epoch.
struct FitState {
    long long pos;          // first order index of the next batch
    double loss_sum;        // sum of per-row losses of the epoch (network.hpp:500)
    unsigned long long correct;  // evaluate(): rows whose argmax equals the label
};

static __global__ void fit_gather_kernel(const float* __restrict__ ds, long long per, const int* __restrict__ ds_y,
                                         const int* __restrict__ order, const FitState* st, int count,
                                         float* __restrict__ X, long long ldx, int* __restrict__ labels) {
    pdl_wait();
    const long long pos = st->pos;
    const bool vec = (per & 3) == 0 && (ldx & 3) == 0;
    const long long n = (long long)count * (vec ? per / 4 : per);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        if (vec) {
            const long long r = i / (per / 4), c = i - r * (per / 4);
            const long long src = order[pos + r];
            reinterpret_cast<float4*>(X + r * ldx)[c] = __ldg(reinterpret_cast<const float4*>(ds + src * per) + c);
        } else {
            const long long r = i / per, c = i - r * per;
            X[r * ldx + c] = __ldg(ds + order[pos + r] * per + c);
        }
    }
    if (blockIdx.x == 0)
        for (int r = threadIdx.x; r < count; r += blockDim.x) labels[r] = ds_y[order[pos + r]];
}

// after a training step: loss_sum += sum of the batch's row losses in row order; advance the cursor
static __global__ void fit_advance_kernel(const double* __restrict__ row_loss, int count, FitState* st, int eval,
                                          const int* __restrict__ argmax, const int* __restrict__ labels) {
    pdl_wait();
    if (threadIdx.x != 0) return;
    if (eval) {
        unsigned long long c = 0;
        for (int r = 0; r < count; ++r) c += argmax[r] == labels[r];
        st->correct += c;
    } else {
        double s = 0.0;
        for (int r = 0; r < count; ++r) s += row_loss[r];
        st->loss_sum += s;
    }
    st->pos += count;
}

// train_stream: the step's loss (row losses summed in row order, network.hpp:433-435) into the
// next slot of the per-step array
static __global__ void stream_loss_kernel(const double* __restrict__ row_loss, int count, double* out) {
    pdl_wait();
    if (threadIdx.x != 0) return;
    double s = 0.0;
    for (int r = 0; r < count; ++r) s += row_loss[r];
    unsigned long long* idx = reinterpret_cast<unsigned long long*>(out - 1);
    out[*idx] = s;
    *idx += 1;
}

// BatchIterator's order (data.hpp:224-238): iota, then std::shuffle with mt19937(seed) at construction
// and mt19937(seed + epoch) on the current order for every later epoch (network.hpp:495)
inline void batch_order(std::vector<long long>& order, long long N, unsigned seed, int epoch) {
    std::vector<std::size_t> o((size_t)N);
    for (long long i = 0; i < N; ++i) o[(size_t)i] = (std::size_t)i;
    {
        std::mt19937 rng(seed);
        std::shuffle(o.begin(), o.end(), rng);
    }
    for (int e = 1; e <= epoch; ++e) {
        std::mt19937 rng(seed + (unsigned)e);
        std::shuffle(o.begin(), o.end(), rng);
    }
    order.assign(o.begin(), o.end());
}

class Net {
  public:
    struct Layer {
        int kind = B2N_DENSE;
        std::vector<long long> in_shape, out_shape;
        // dense
        long long in = 0, out = 0, ldw = 0, off = 0;
        // conv (+ fused act + pool)
        ConvGeom g;
        long long kern_off = 0, bias_off = 0;
        // fused epilogue choices
        int act = ACT_NONE;
        bool pool_after = false;
        bool softmax_after = false;
        // activations (device)
        float* Ain = nullptr;
        long long ld_in = 0;
        float* Aout = nullptr;
        long long ld_out = 0;
        float* D = nullptr;  // gradient w.r.t. this layer's (pre-activation / pooled) output
        long long ldd = 0;
        uint8_t* arg = nullptr;  // pool argmax codes
        float* Dx = nullptr;     // gradient w.r.t. this layer's input (conv dgrad output)
        // halo-tile conv path (convt.cuh): output / D row-blocked when a conv consumes them
        bool blocked_out = false;
        long long codes_bstride = 0;
        int codes_pw = 0;
    };

    Net(const b2n_network_spec& spec, int device, int precision);
    ~Net();

    int num_params() const { return (int)params_.size(); }
    const ParamView& param(int i) const { return params_.at(i); }
    void get_param(int idx, int which, float* host);
    void set_param(int idx, int which, const float* host);
    long long num_layers() const { return (long long)layers_.size(); }
    void layer_output(int li, long long batch, float* host, uint8_t* codes_host);
    void set_hparams(float lr, float mom, float wd) {
        lr_ = lr;
        mom_ = mom;
        wd_ = wd;
        invalidate_plans();
    }

    double train(const float* x, const int* labels, long long B);
    // `steps` train_minibatch calls over consecutive host batches (rows [i B, (i + 1) B) of x / labels);
    // the H2D of step i + 1 runs on a copy stream into the other of two device staging buffers while
    // step i computes. loss_out[i] = step i's train_minibatch return value.
    void train_stream(const float* x, const int* labels, long long steps, long long B, double* loss_out);
    double forward_backward(const float* x, const int* labels, long long B, long long Bg);
    void apply_update();
    void forward(const float* x, long long B, float* probs, int* argmax);
    void stage(const float* x, const int* labels, long long B);
    struct FitEpoch {
        double loss, accuracy, seconds;
    };
    // fit (network.hpp:488-511): `epochs` shuffled passes over a dataset of N samples held in HBM;
    // per-epoch mean loss, train accuracy (evaluate) and batch-loop wall time
    std::vector<FitEpoch> fit(const float* images, const int* labels, long long N, int epochs);
    double evaluate(const float* images, const int* labels, long long N);  // network.hpp:474-484
    void save(const std::string& path, bool with_state);  // network.hpp:552-573 (+ sidecar)
    void load(const std::string& path, bool with_state);  // network.hpp:575-607 (+ sidecar)
    void run_staged(int steps, long long Bg);
    double loss();
    int kernels_per_step(long long B);
    std::vector<OpStats> profile(long long B, int steps) {
        ensure_capacity(B);
        Plan& pl = plan_for(B, B);
        return profile_ops(pl.ops[TRAIN], steps, stream_);
    }
    void dp_init(const char id[128], int rank, int world) {
        dp_ = std::make_unique<DpComm>();
        dp_->init(id, rank, world);
        invalidate_plans();
    }
    cudaStream_t stream() const { return stream_; }
    float* grad_buffer() const { return G_.as<float>(); }
    long long packed_floats() const { return n_packed_; }

  private:
    // TRAIN = the whole training step of this net: FUSED (SGD epilogues in the backward kernels) when
    // the optimizer is SGD-momentum on one GPU, else SPLIT + SPLIT_APPLY (allreduce and / or the
    // packed optimizer kernel), SPLIT alone when lr == 0
    enum Mode { FUSED = 0, SPLIT = 1, FWD = 2, SPLIT_APPLY = 3, FIT = 4, EVAL = 5, TRAIN = 6, STREAM0 = 7, STREAM1 = 8,
                NMODES = 9 };
    struct Plan {
        long long B = 0, Bg = 0;
        std::vector<Op> ops[NMODES];
        cudaGraphExec_t graph[NMODES] = {};
        int nkernels[NMODES] = {};
        ~Plan() {
            for (auto& g : graph)
                if (g) cudaGraphExecDestroy(g);
        }
    };

    void ensure_capacity(long long B);
    void alloc_activations();
    Plan& plan_for(long long B, long long Bg);
    void build_plan(Plan& pl);
    void launch(Plan& pl, int mode);
    void stage_inputs(const float* x, const int* labels, long long B);
    void build_stream_ops(Plan& pl, int j);
    DevMem sx_[2], sl_[2];   // train_stream: double-buffered device staging of x / labels
    DevMem sloss_;           // train_stream: per-step loss sums [kStreamChunk] + step counter
    static constexpr long long kStreamChunk = 4096;
    cudaEvent_t ev_copied_[2] = {nullptr, nullptr}, ev_used_[2] = {nullptr, nullptr};
    cudaStream_t copy_stream_ = nullptr;
    double read_loss(long long B);
    void invalidate_plans() { plans_.clear(); }
    void check_train_params() const;

    int device_;
    bool x3_;
    cudaStream_t stream_ = nullptr;
    cudaStream_t side_ = nullptr;  // graph-capture side branch (dense wgrad+SGD off the critical path)
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
    std::vector<long long> input_;
    std::vector<Layer> layers_;
    std::vector<ParamView> params_;
    long long n_packed_ = 0;
    long long classes_ = 0;
    float lr_, mom_, wd_;
    long long cap_ = 0;
    DevMem P_, V_, G_;
    DevMem act_;
    float* X_ = nullptr;  // network input (augmented with a ones column for a first dense layer)
    long long ldx_ = 0;
    int* labels_ = nullptr;
    double* row_loss_ = nullptr;
    int* argmax_ = nullptr;
    float* probs_ = nullptr;
    float* logits_ = nullptr;  // only when classes > 256 (standalone softmax kernel)
    long long ldlog_ = 0;
    HostPinned h_loss_;
    long long last_B_ = 0, last_Bg_ = 0;
    std::map<std::pair<long long, long long>, std::unique_ptr<Plan>> plans_;
    std::unique_ptr<DpComm> dp_;
    DevMem loss_sum_;  // dp: double partial loss
    bool tconv_ = false;     // conv layers on the halo-tile kernels (convt.cuh) instead of conv.cuh
    bool conv_fwd_tc_ = false;  // conv forward on the tensor cores (convt FWD) instead of the exact convx
    DevMem ds_x_, ds_y_, ds_order_, fit_state_;  // device-resident dataset, order, cursor / sums
    long long ds_n_ = 0;
    unsigned seed_ = 0;
    long long batch_size_ = 1;
    std::vector<int> spec_kinds_;  // the spec's layer list (checkpoint tags, network.hpp:560)
    int opt_ = 0;                  // OptimizerKind (optim.hpp:11)
    DevMem S1_, S2_;               // adagrad / adadelta / adam state (packed like P_)
    DevMem opt_ctab_, opt_cnt_;    // adam bias-correction table + device step counter
    long long opt_steps_ = 0, opt_ctab_filled_ = 0;  // host view of the adam step count / table fill
    static constexpr long long kCtabCap = 1ll << 24;
    void note_opt_step();
    DevMem& state_buffer(int which);
    void gather_params(const std::vector<float>& packed, int idx, float* out) const;
    void scatter_params(std::vector<float>& packed, int idx, const float* in) const;
    void upload_dataset(const float* images, const int* labels, long long N);
    void build_fit_ops(Plan& pl, int mode);
    double run_epoch_eval(long long N);
    float* Xb_ = nullptr;    // row-blocked copy of a conv network's input
    long long xb_bstride_ = 0;
    TLayout out_layout(const Layer& L, float* p, long long ld) const {
        TLayout t;
        t.p = p;
        t.bstride = ld;
        t.blocked = L.blocked_out ? 1 : 0;
        t.C = (int)L.out_shape[0];
        t.H = (int)L.out_shape[1];
        t.W = (int)L.out_shape[2];
        return t;
    }
};

// --------------------------------------------------------------------------- construction
inline Net::Net(const b2n_network_spec& spec, int device, int precision)
    : device_(device), x3_(precision == B2N_TF32X3), lr_(spec.lr), mom_(spec.momentum), wd_(spec.weight_decay) {
    seed_ = spec.seed;
    batch_size_ = spec.batch_size;
    // validation mirrors build_network (network.hpp:285-300, :303-367)
    if (spec.n_layers < 1 || !spec.layers) throw Error(B2N_ESPEC, "network spec has no layers");
    if (spec.input_rank != 1 && spec.input_rank != 3)
        throw Error(B2N_ESPEC, "network spec input must have 1 or 3 extents; got " + std::to_string(spec.input_rank));
    for (int i = 0; i < spec.input_rank; ++i)
        if (spec.input[i] < 1) throw Error(B2N_ESPEC, "network spec input extents must be positive");
    if (spec.batch_size < 1) throw Error(B2N_ESPEC, "network spec batch_size must be >= 1");
    if (spec.optimizer < 0 || spec.optimizer > OPT_ADAM) throw Error(B2N_ESPEC, "unknown optimizer kind");
    opt_ = spec.optimizer;
    input_.assign(spec.input, spec.input + spec.input_rank);

    auto shape_str = [](const std::vector<long long>& s) {
        std::string o = "(";
        for (size_t i = 0; i < s.size(); ++i) o += (i ? "x" : "") + std::to_string(s[i]);
        return o + ")";
    };
    auto mismatch = [&](int idx, const std::vector<long long>& got, const std::string& need) {
        throw Error(B2N_ESPEC, "network spec: " + (idx == 1 ? std::string("input") : "layer " + std::to_string(idx - 1)) +
                                   " produces " + shape_str(got) + " but layer " + std::to_string(idx) + " expects " +
                                   need);
    };
    std::vector<long long> cur = input_;
    for (int i = 0; i < spec.n_layers; ++i) {
        const b2n_layer_desc& d = spec.layers[i];
        const int idx = i + 1;
        // the reference's node list (checkpoint layer count / tags): an implicit FlattenNode before a
        // dense layer that follows feature maps (network.hpp:309-312)
        if (d.kind == B2N_DENSE && cur.size() == 3) spec_kinds_.push_back(B2N_FLATTEN);
        spec_kinds_.push_back(d.kind);
        switch (d.kind) {
            case B2N_DENSE: {
                if (cur.size() == 3) cur = {cur[0] * cur[1] * cur[2]};  // implicit flatten (network.hpp:309-312)
                if (cur[0] != d.in) mismatch(idx, cur, "dense input extent " + std::to_string(d.in));
                if (d.out < 1) throw Error(B2N_ESPEC, "dense output extent must be positive");
                Layer L;
                L.kind = B2N_DENSE;
                L.in_shape = cur;
                L.in = d.in;
                L.out = d.out;
                L.ldw = round_up(d.in + 1, 8);
                cur = {d.out};
                L.out_shape = cur;
                layers_.push_back(L);
                break;
            }
            case B2N_CONV: {
                if (cur.size() != 3) mismatch(idx, cur, "feature maps (c, h, w) for conv");
                if (d.kh > cur[1] + 2 * d.pad || d.kw > cur[2] + 2 * d.pad)
                    mismatch(idx, cur, "extents >= the " + std::to_string(d.kh) + "x" + std::to_string(d.kw) + " kernel");
                if (d.k < 1 || d.kh < 1 || d.kw < 1 || d.pad < 0) throw Error(B2N_ESPEC, "bad conv extents");
                Layer L;
                L.kind = B2N_CONV;
                L.in_shape = cur;
                L.g.c = (int)cur[0];
                L.g.h = (int)cur[1];
                L.g.w = (int)cur[2];
                L.g.k = (int)d.k;
                L.g.kh = (int)d.kh;
                L.g.kw = (int)d.kw;
                L.g.pad = (int)d.pad;
                L.g.oh = L.g.h + 2 * L.g.pad - L.g.kh + 1;
                L.g.ow = L.g.w + 2 * L.g.pad - L.g.kw + 1;
                cur = {d.k, L.g.oh, L.g.ow};
                L.out_shape = cur;
                layers_.push_back(L);
                break;
            }
            case B2N_MAXPOOL: {
                if (cur.size() != 3) mismatch(idx, cur, "feature maps (c, h, w) for maxpool");
                if (cur[1] % 2 || cur[2] % 2) mismatch(idx, cur, "even spatial extents for 2x2 pooling");
                if (layers_.empty() || layers_.back().kind != B2N_CONV || layers_.back().pool_after)
                    throw Error(B2N_ESPEC, "b200nn: maxpool must follow a conv (+activation) to fuse into its epilogue");
                layers_.back().pool_after = true;
                cur = {cur[0], cur[1] / 2, cur[2] / 2};
                layers_.back().out_shape = cur;
                break;
            }
            case B2N_SIGMOID:
            case B2N_RELU: {
                const int a = d.kind == B2N_SIGMOID ? ACT_SIGMOID : ACT_RELU;
                if (layers_.empty() || layers_.back().act != ACT_NONE || layers_.back().pool_after)
                    throw Error(B2N_ESPEC, "b200nn: an activation must directly follow a dense or conv layer");
                layers_.back().act = a;
                break;
            }
            case B2N_SOFTMAX:
                if (cur.size() != 1) mismatch(idx, cur, "a flat vector for softmax");
                if (i + 1 != spec.n_layers)
                    throw Error(B2N_ESPEC, "network spec: softmax (layer " + std::to_string(idx) + ") must be the final layer");
                if (layers_.empty() || layers_.back().kind != B2N_DENSE || layers_.back().act != ACT_NONE)
                    throw Error(B2N_ESPEC, "b200nn: softmax must follow a dense layer");
                layers_.back().softmax_after = true;
                break;
            case B2N_FLATTEN:
                if (cur.size() != 3) mismatch(idx, cur, "feature maps (c, h, w) for flatten");
                cur = {cur[0] * cur[1] * cur[2]};
                break;
            case B2N_DROPOUT:
            case B2N_BATCHNORM:
                throw Error(B2N_ESPEC, "b200nn: dropout / batchnorm are outside the B200 hot path (SURVEY 2.1 #9)");
            default: throw Error(B2N_ESPEC, "unknown layer kind " + std::to_string(d.kind));
        }
    }
    if (!layers_.back().softmax_after || layers_.back().kind != B2N_DENSE)
        throw Error(B2N_ESPEC, "b200nn: the training step needs a dense + softmax output (network.hpp:465)");
    for (const Layer& L : layers_)
        if (L.kind == B2N_CONV && L.pool_after && (L.g.oh % 2 || L.g.ow % 2))
            throw Error(B2N_ESPEC, "maxpool needs even extents");
    classes_ = layers_.back().out;
    {  // the halo-tile conv kernels cover 3x3 / 5x5 filters with <= 32 channels and kernels
        const char* e = std::getenv("B2N_CONV_LEGACY");
        tconv_ = !(e && e[0] == '1');
        const char* f = std::getenv("B2N_CONV_FWD");
        conv_fwd_tc_ = f && std::string(f) == "tc";
        auto nk = [](int n) { return n <= 8 ? 8 : n <= 16 ? 16 : 32; };
        for (const Layer& L : layers_) {
            if (L.kind != B2N_CONV) continue;
            const bool shape_ok = L.g.kh == L.g.kw && (L.g.kh == 3 || L.g.kh == 5) && L.g.k <= 32 && L.g.c <= 32;
            // two TMEM buffers of >= 2 + 2(kh-1) row slots of NK columns (fwd: NK(k), dgrad: NK(c))
            const int slots = 2 + 2 * (L.g.kh - 1);
            const bool tmem_ok = 2 * slots * nk(L.g.k) <= 512 && 2 * slots * nk(L.g.c) <= 512;
            if (!shape_ok || !tmem_ok) tconv_ = false;
        }
    }

    // packed parameter layout, trainable() order
    long long off = 0;
    auto take = [&](long long n) {
        const long long o = off;
        off = round_up(off + n, 32);
        return o;
    };
    for (Layer& L : layers_) {
        if (L.kind == B2N_DENSE) {
            L.off = take(L.out * L.ldw);
            params_.push_back({{L.out, L.in}, L.off, L.out, L.in, L.ldw});
            params_.push_back({{L.out}, L.off + L.in, L.out, 1, L.ldw});
        } else {
            const long long kn = (long long)L.g.k * L.g.c * L.g.kh * L.g.kw;
            L.kern_off = take(kn);
            L.bias_off = take(L.g.k);
            params_.push_back({{L.g.k, L.g.c, L.g.kh, L.g.kw}, L.kern_off, 1, kn, kn});
            params_.push_back({{L.g.k}, L.bias_off, 1, L.g.k, L.g.k});
        }
    }
    n_packed_ = round_up(off, 32);
    // the spec is valid: from here on device work (spec errors above never touch the GPU)
    B2N_CUDA(cudaSetDevice(device));
    B2N_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    P_.alloc(n_packed_ * 4);
    V_.alloc(n_packed_ * 4);
    G_.alloc(n_packed_ * 4);
    if (opt_ != 0) {
        S1_.alloc(n_packed_ * 4);
        if (opt_ != OPT_ADAGRAD) S2_.alloc(n_packed_ * 4);
        opt_cnt_.alloc(sizeof(OptCounter));
        if (opt_ == OPT_ADAM) opt_ctab_.alloc(kCtabCap * sizeof(float2));
    }
    loss_sum_.alloc(64);
    // seeded Glorot init in layer order (network.hpp:369-373, layers.hpp:40-48), same draws
    std::mt19937 rng(spec.seed);
    std::vector<float> host(n_packed_, 0.0f);
    for (Layer& L : layers_) {
        long long fan_in, fan_out, rows, cols, pitch, base;
        if (L.kind == B2N_DENSE) {
            fan_in = L.in, fan_out = L.out, rows = L.out, cols = L.in, pitch = L.ldw, base = L.off;
        } else {
            fan_in = (long long)L.g.c * L.g.kh * L.g.kw, fan_out = (long long)L.g.k * L.g.kh * L.g.kw;
            rows = 1, cols = (long long)L.g.k * fan_in, pitch = cols, base = L.kern_off;
        }
        const float limit = std::sqrt(6.0f / static_cast<float>(fan_in + fan_out));
        UniformF32 dist(-limit, limit);
        for (long long r = 0; r < rows; ++r)
            for (long long j = 0; j < cols; ++j) host[base + r * pitch + j] = dist(rng);
    }
    B2N_CUDA(cudaMemcpyAsync(P_.p, host.data(), n_packed_ * 4, cudaMemcpyHostToDevice, stream_));
    B2N_CUDA(cudaStreamSynchronize(stream_));
    h_loss_.alloc(sizeof(double) * 4096);
    ensure_capacity(spec.batch_size);
}

inline Net::~Net() {
    plans_.clear();
    for (int j = 0; j < 2; ++j) {
        if (ev_copied_[j]) cudaEventDestroy(ev_copied_[j]);
        if (ev_used_[j]) cudaEventDestroy(ev_used_[j]);
    }
    if (copy_stream_) cudaStreamDestroy(copy_stream_);
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_join_) cudaEventDestroy(ev_join_);
    if (side_) cudaStreamDestroy(side_);
    if (stream_) cudaStreamDestroy(stream_);
}

inline void Net::ensure_capacity(long long B) {
    if (B <= cap_) return;
    cap_ = std::max(B, cap_);
    invalidate_plans();
    alloc_activations();
}

inline void Net::alloc_activations() {
    // one allocation, carved per layer; 256 B alignment per buffer
    struct Req {
        void** dst;
        size_t bytes;
    };
    std::vector<Req> reqs;
    const long long cap = cap_;
    auto req = [&](void** dst, size_t bytes) { reqs.push_back({dst, (bytes + 255) / 256 * 256}); };
    const Layer& first = layers_.front();
    const long long in0 = numel(input_);
    ldx_ = first.kind == B2N_DENSE ? round_up(in0 + 1, 8) : in0;
    req((void**)&X_, cap * ldx_ * 4);
    for (size_t i = 0; i < layers_.size(); ++i) {
        Layer& L = layers_[i];
        const bool last = i + 1 == layers_.size();
        const bool next_dense = !last && layers_[i + 1].kind == B2N_DENSE;
        if (L.kind == B2N_DENSE) {
            L.ld_out = round_up(L.out + (next_dense ? 1 : 0), 8);
            if (!last) req((void**)&L.Aout, cap * L.ld_out * 4);
            // the standalone (classes > 256) softmax kernel keeps its row sum in column `out`
            L.ldd = round_up(L.out + (last && L.out > 256 ? 1 : 0), 8);
            req((void**)&L.D, cap * L.ldd * 4);
        } else {
            const long long per = numel(L.out_shape);
            const long long kq = (L.g.k + 3) / 4, oh = L.out_shape[1], ow = L.out_shape[2];
            L.blocked_out = tconv_ && !next_dense && !last;
            // pooled (or plain) conv output; an augmented row when a dense layer consumes it
            L.ld_out = next_dense ? round_up(per + 1, 8) : L.blocked_out ? oh * kq * ow * 4 : per;
            req((void**)&L.Aout, cap * L.ld_out * 4);
            L.ldd = next_dense ? round_up(per, 8) : L.blocked_out ? L.ld_out : per;
            req((void**)&L.D, cap * L.ldd * 4);
            L.codes_pw = (int)round_up(ow, 4);
            L.codes_bstride = tconv_ ? oh * kq * L.codes_pw * 4 : per;
            if (L.pool_after) req((void**)&L.arg, cap * L.codes_bstride);
        }
    }
    if (tconv_ && first.kind == B2N_CONV) {
        xb_bstride_ = (long long)first.g.h * ((first.g.c + 3) / 4) * first.g.w * 4;
        req((void**)&Xb_, cap * xb_bstride_ * 4);
    }
    if (classes_ > 256) {
        ldlog_ = round_up(classes_ + 1, 8);
        req((void**)&logits_, cap * ldlog_ * 4);
    }
    req((void**)&labels_, cap * 4);
    req((void**)&row_loss_, cap * 8);
    req((void**)&argmax_, cap * 4);
    req((void**)&probs_, cap * classes_ * 4);
    size_t total = 0;
    for (auto& r : reqs) total += r.bytes;
    act_.alloc(total);
    size_t o = 0;
    for (auto& r : reqs) {
        *r.dst = static_cast<char*>(act_.p) + o;
        o += r.bytes;
    }
    // wire inputs and ones columns
    float* prev = X_;
    long long ld_prev = ldx_;
    for (size_t i = 0; i < layers_.size(); ++i) {
        Layer& L = layers_[i];
        L.Ain = prev;
        L.ld_in = ld_prev;
        if (L.kind == B2N_DENSE) {
            set_column_kernel<<<grid_for(cap), 256, 0, stream_>>>(L.Ain, cap, L.ld_in, L.in, 1.0f);
            B2N_CUDA(cudaGetLastError());
        }
        prev = L.Aout;
        ld_prev = L.ld_out;
    }
    // conv dgrad targets: the D buffer of the previous layer
    for (size_t i = 1; i < layers_.size(); ++i) layers_[i].Dx = layers_[i - 1].D;
    B2N_CUDA(cudaStreamSynchronize(stream_));
}

inline void Net::check_train_params() const {  // optim.hpp:51-55, only reached when lr != 0 (network.hpp:468)
    if (lr_ != 0.0f) {
        if (!(lr_ > 0.0f)) throw Error(B2N_EPARAM, "optimizer step: lr must be > 0");
        if (mom_ < 0.0f || mom_ >= 1.0f) throw Error(B2N_EPARAM, "optimizer step: momentum must be in [0, 1)");
    }
}

// --------------------------------------------------------------------------- planning
inline Net::Plan& Net::plan_for(long long B, long long Bg) {
    auto key = std::make_pair(B, Bg);
    auto it = plans_.find(key);
    if (it != plans_.end()) return *it->second;
    auto pl = std::make_unique<Plan>();
    pl->B = B;
    pl->Bg = Bg;
    build_plan(*pl);
    Plan& ref = *pl;
    plans_[key] = std::move(pl);
    return ref;
}

inline void Net::build_plan(Plan& pl) {
    const int B = (int)pl.B;
    float* P = P_.as<float>();
    float* Vv = V_.as<float>();
    float* G = G_.as<float>();
    std::vector<Op> fwd, bwd_fused, bwd_split;
    int nk_fwd = 0, nk_fused = 0, nk_split = 0;
    const size_t nl = layers_.size();
    std::vector<ConvTLaunch> tfwd(nl);  // halo-tile conv forward plans (their tiles / X maps feed wgrad)

    // ---------------- forward
    for (size_t i = 0; i < nl; ++i) {
        Layer& L = layers_[i];
        if (L.kind == B2N_DENSE) {
            EpiParams e = epi_default();
            e.bias = P + L.off + L.in;
            e.bias_stride = L.ldw;
            const bool fused_softmax = L.softmax_after && L.out <= 256;
            if (fused_softmax) {
                e.C = L.D;
                e.ldc = L.ldd;
                e.labels = labels_;
                e.batch_div = (float)pl.Bg;
                e.row_loss = row_loss_;
                e.argmax = argmax_;
                e.probs = probs_;
                e.ld_probs = classes_;
            } else if (L.softmax_after) {
                e.C = logits_;
                e.ldc = ldlog_;
                e.act = ACT_NONE;
            } else {
                e.C = L.Aout;
                e.ldc = L.ld_out;
                e.act = L.act;
            }
            GemmLaunch g = plan_gemm(B, (int)L.out, (int)L.in, {L.Ain, L.ld_in, false}, {P + L.off, L.ldw, false},
                                     fused_softmax ? EPI_SOFTMAX_XENT : EPI_BIAS_ACT, e, x3_);
            fwd.push_back(gemm_op(g, "dense" + std::to_string(i) + (fused_softmax ? ".fwd+softmax_xent" : ".fwd+act")));
            ++nk_fwd;
            if (L.softmax_after && !fused_softmax) {
                float* lg = logits_;
                long long ldl = ldlog_, C = classes_;
                float* D = L.D;
                long long ldd = L.ldd;
                int* lab = labels_;
                double* rl = row_loss_;
                int* am = argmax_;
                float* pr = probs_;
                float bd = (float)pl.Bg;
                // one CTA per row, the row staged in shared memory
                const size_t smem = (size_t)((C + 3) & ~3LL) * 4;
                if (smem > 200 * 1024) throw Error(B2N_ESHAPE, "softmax: more than 51,200 classes");
                static bool sx_attr = [] {
                    B2N_CUDA(cudaFuncSetAttribute(softmax_xent_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  200 * 1024));
                    return true;
                }();
                (void)sx_attr;
                fwd.push_back(Op([=](cudaStream_t s) {
                    launch_ex(softmax_xent_rows_kernel, dim3(B), dim3(kSxThreads), smem, s, 1u, (const float*)lg, ldl, B,
                              (int)C, (const int*)lab, bd, D, ldd, rl, am, pr, C);
                }, "softmax_xent", 0.0, (double)B * C * 16));
                ++nk_fwd;
                if (ldd < C + 1) throw Error(B2N_EINTERNAL, "dlogits pitch");
            }
        } else {
            if (tconv_) {
                const ConvGeom& g = L.g;
                const int Cp = (g.c + 3) & ~3;
                const float* in = L.Ain;
                long long in_bs = L.ld_in;
                if (i == 0) {  // network input NCHW -> row-blocked (channel quads)
                    float* xs = X_;
                    long long ldx = ldx_, xbs = xb_bstride_;
                    float* xb = Xb_;
                    const long long n = (long long)B * g.h * (Cp / 4) * g.w;
                    fwd.push_back(Op([=](cudaStream_t s) {
                        launch_ex(convt_repack_kernel, dim3(grid_for(n)), dim3(256), 0, s, 1u, (const float*)xs, ldx, B,
                                  g.c, g.h, g.w, xb, xbs);
                    }, "conv0.repack", 0.0, (double)B * g.h * g.w * (g.c + Cp) * 4));
                    in = Xb_;
                    in_bs = xb_bstride_;
                }
                ConvTLaunch f = plan_convt(CT_FWD, B, Cp, g.h, g.w, g.kh, g.kw, g.pad, g.k, x3_);
                f.map = make_map_blocked(in, B, Cp / 4, g.h, g.w, in_bs, f.p.P, f.p.HR);
                f.p.x = in;
                f.p.x_bstride = in_bs;
                f.p.act = L.act;
                f.p.pool = L.pool_after ? 1 : 0;
                f.p.bias = P + L.bias_off;
                f.p.out = out_layout(L, L.Aout, L.ld_out);
                f.p.codes = L.arg;
                f.p.codes_bstride = L.codes_bstride;
                f.p.codes_pw = L.codes_pw;
                f.p.wk = P + L.kern_off;
                f.p.wk_K = g.k;
                f.p.wk_C = g.c;
                const double outn = (double)B * numel(L.out_shape);
                f.bytes = (double)B * g.c * g.h * g.w * 4 + outn * (L.pool_after ? 5 : 4) + (double)g.k * (g.c * g.kh * g.kw + 1) * 4;
                f.flops = 2.0 * B * g.oh * g.ow * g.k * (double)g.c * g.kh * g.kw;
                tfwd[i] = f;  // its tiles and input map also plan the weight gradient
                if (conv_fwd_tc_) {  // 3xTF32 tensor-core forward (B2N_CONV_FWD=tc), near-tie fix-up
                    if (!std::getenv("B2N_CT_NOFIX")) convt_enable_fix(f, f.fix);
                    fwd.push_back(Op([f](cudaStream_t s) { f.run(s); }, "conv" + std::to_string(i) + ".fwd", f.flops, f.bytes));
                } else {  // the reference's own fma chains: bit-identical activations and pool decisions
                    ConvXLaunch xf = plan_convx_fwd(B, g.c, g.h, g.w, g.kh, g.kw, g.pad, g.k);
                    xf.p.x = in;
                    xf.p.x_bstride = in_bs;
                    xf.p.wk = P + L.kern_off;
                    xf.p.bias = P + L.bias_off;
                    xf.p.act = L.act;
                    xf.p.pool = L.pool_after ? 1 : 0;
                    xf.p.out = out_layout(L, L.Aout, L.ld_out);
                    xf.p.codes = L.arg;
                    xf.p.codes_bstride = L.codes_bstride;
                    xf.p.codes_pw = L.codes_pw;
                    xf.bytes = f.bytes;
                    fwd.push_back(Op([xf](cudaStream_t s) { xf.run(s); }, "conv" + std::to_string(i) + ".fwd", xf.flops, xf.bytes));
                }
                ++nk_fwd;
                continue;
            }
            ConvFwdLaunch c = plan_conv_fwd(L.g, B, L.Ain, L.ld_in, P + L.kern_off, P + L.bias_off, L.act, L.pool_after,
                                            L.Aout, L.ld_out, L.arg, x3_);
            fwd.push_back(Op([c](cudaStream_t s) { c.run(s); }, "conv" + std::to_string(i) + ".fwd", c.flops, c.bytes));
            ++nk_fwd;
        }
    }
    // ---------------- backward
    for (size_t ii = nl; ii-- > 0;) {
        Layer& L = layers_[ii];
        if (L.kind == B2N_DENSE) {
            if (ii > 0) {  // dX with the previous layer's activation derivative fused
                Layer& Prev = layers_[ii - 1];
                if (Prev.kind == B2N_DENSE) {
                    EpiParams e = epi_default();
                    e.C = Prev.D;
                    e.ldc = Prev.ldd;
                    e.aux = Prev.Aout;
                    e.ld_aux = Prev.ld_out;
                    e.act = Prev.act;
                    GemmLaunch g = plan_gemm(B, (int)L.in, (int)L.out, {L.D, L.ldd, false}, {P + L.off, L.ldw, true},
                                             Prev.act == ACT_NONE ? EPI_STORE : EPI_DACT, e, x3_);
                    bwd_fused.push_back(gemm_op(g, "dense" + std::to_string(ii) + ".dgrad+dact"));
                    bwd_split.push_back(gemm_op(g, "dense" + std::to_string(ii) + ".dgrad+dact"));
                } else {  // conv below: plain dX into the pooled-gradient buffer (act' applied by the conv gather)
                    EpiParams e = epi_default();
                    e.C = Prev.D;
                    e.ldc = Prev.ldd;
                    GemmLaunch g = plan_gemm(B, (int)L.in, (int)L.out, {L.D, L.ldd, false}, {P + L.off, L.ldw, true},
                                             EPI_STORE, e, x3_);
                    bwd_fused.push_back(gemm_op(g, "dense" + std::to_string(ii) + ".dgrad"));
                    bwd_split.push_back(gemm_op(g, "dense" + std::to_string(ii) + ".dgrad"));
                }
                ++nk_fused;
                ++nk_split;
            }
            // dW (+ db through the ones column): M = out, N = in + 1, K = batch
            EpiParams ef = epi_default();
            ef.C = P + L.off;
            ef.ldc = L.ldw;
            ef.V = Vv + L.off;
            ef.ldv = L.ldw;
            ef.lr = lr_;
            ef.mom = mom_;
            ef.wd = wd_;
            GemmLaunch gf = plan_gemm((int)L.out, (int)L.in + 1, B, {L.D, L.ldd, true}, {L.Ain, L.ld_in, true},
                                      EPI_SGD, ef, x3_);
            EpiParams es = epi_default();
            es.C = G + L.off;
            es.ldc = L.ldw;
            GemmLaunch gs = plan_gemm((int)L.out, (int)L.in + 1, B, {L.D, L.ldd, true}, {L.Ain, L.ld_in, true},
                                      EPI_STORE, es, x3_);
            bwd_fused.push_back(gemm_op(gf, "dense" + std::to_string(ii) + ".wgrad+sgd"));
            // off the critical path: only the next step's forward (after the graph's join) reads the
            // updated W / V, and this layer's dgrad (which reads W) precedes the fork
            if (branch_wgrad()) bwd_fused.back().branch = 1;
            bwd_split.push_back(gemm_op(gs, "dense" + std::to_string(ii) + ".wgrad"));
            ++nk_fused;
            ++nk_split;
        } else if (tconv_) {
            const ConvGeom& g = L.g;
            const int Kp = (g.k + 3) & ~3;
            const TLayout dP = out_layout(L, L.D, L.ldd), Pv = out_layout(L, L.Aout, L.ld_out);
            const bool has_d = ii > 0;
            DZSrc z;
            std::memset(&z, 0, sizeof(z));
            z.dP = dP;
            z.P = Pv;
            z.codes = L.arg;
            z.codes_bstride = L.codes_bstride;
            z.PWc = L.codes_pw;
            z.act = L.act;
            z.pool = L.pool_after ? 1 : 0;
            z.OHz = g.oh;
            z.OWz = g.ow;
            z.tma = L.blocked_out ? 1 : 0;
            z.Kq = Kp / 4;
            ConvTLaunch d;
            if (has_d) {  // dX = the previous conv's pooled-output gradient (row-blocked)
                const Layer& Prev = layers_[ii - 1];
                d = plan_convt(CT_DGRAD, B, Kp, g.oh, g.ow, g.kh, g.kw, g.kh - 1 - g.pad, g.c, x3_, &z);
                std::memset(&d.map, 0, sizeof(d.map));
                d.p.out = out_layout(Prev, Prev.D, Prev.ldd);
                d.p.wk = P + L.kern_off;
                d.p.wk_K = g.k;
                d.p.wk_C = g.c;
                const double pooled = (double)B * numel(L.out_shape);
                d.bytes = pooled * 9 + (double)B * g.c * g.h * g.w * 4;
                d.flops = 2.0 * B * g.h * g.w * g.c * (double)g.k * g.kh * g.kw;
            }
            auto wplan = [&](bool fused) {
                ConvTWLaunch w = plan_convt_wgrad(tfwd[ii], g.k, g.c, z);
                w.kern = P + L.kern_off;
                w.kvel = Vv + L.kern_off;
                w.bias = P + L.bias_off;
                w.bvel = Vv + L.bias_off;
                w.gk = G + L.kern_off;
                w.gb = G + L.bias_off;
                w.lr = lr_;
                w.mom = mom_;
                w.wd = wd_;
                (void)fused;
                return w;
            };
            const ConvTWLaunch wf = wplan(true), wsp = wplan(false);
            const double fl = wf.flops + (has_d ? d.flops : 0.0), by = wf.bytes + (has_d ? d.bytes : 0.0);
            const int nk = has_d ? 3 : 2;
            // dgrad on the main chain, then the weight gradient + SGD forked onto the side branch:
            // it must follow this layer's dgrad (which reads the kernels it updates) but nothing
            // on the main chain below reads its outputs before the graph's join
            if (has_d)
                bwd_fused.push_back(Op([d](cudaStream_t s) { d.run(s); }, "conv" + std::to_string(ii) + ".dgrad", d.flops,
                                       d.bytes, 1));
            bwd_fused.push_back(Op([wf](cudaStream_t s) { wf.run(s, true); }, "conv" + std::to_string(ii) + ".wgrad+sgd",
                                   wf.flops, wf.bytes, 2));
            if (branch_wgrad()) bwd_fused.back().branch = 1;
            bwd_split.push_back(Op([d, wsp, has_d](cudaStream_t s) {
                if (has_d) d.run(s);
                wsp.run(s, false);
            }, "conv" + std::to_string(ii) + ".bwd", fl, by, nk));
        } else {
            // conv: dgrad (unless first layer), then wgrad (+ fused SGD on the reduce)
            const bool first = ii == 0;
            ConvBwdLaunch cb = plan_conv_bwd(L.g, B, L.Ain, L.ld_in, P + L.kern_off, P + L.bias_off, L.act,
                                             L.pool_after, L.Aout, L.ld_out, L.arg, L.D, L.ldd,
                                             first ? nullptr : layers_[ii - 1].D, first ? 0 : layers_[ii - 1].ldd,
                                             P + L.kern_off, Vv + L.kern_off, P + L.bias_off, Vv + L.bias_off,
                                             G + L.kern_off, G + L.bias_off, lr_, mom_, wd_, x3_);
            bwd_fused.push_back(Op([cb](cudaStream_t s) { cb.run(s, true); }, "conv" + std::to_string(ii) + ".bwd+sgd",
                                   cb.flops, cb.bytes, cb.kernels()));
            bwd_split.push_back(Op([cb](cudaStream_t s) { cb.run(s, false); }, "conv" + std::to_string(ii) + ".bwd",
                                   cb.flops, cb.bytes, cb.kernels()));
            nk_fused += cb.kernels();
            nk_split += cb.kernels();
        }
    }
    (void)nk_fwd;
    (void)nk_fused;
    (void)nk_split;
    auto count = [](const std::vector<Op>& v) {
        int n = 0;
        for (const Op& o : v) n += o.kernels;
        return n;
    };
    // the step's last op stays on the main stream (it then runs beside the side chain)
    if (!bwd_fused.empty()) bwd_fused.back().branch = 0;
    nk_fwd = count(fwd);
    nk_fused = count(bwd_fused);
    nk_split = count(bwd_split);
    pl.ops[FWD] = fwd;
    pl.nkernels[FWD] = nk_fwd;
    pl.ops[FUSED] = fwd;
    pl.ops[FUSED].insert(pl.ops[FUSED].end(), bwd_fused.begin(), bwd_fused.end());
    pl.nkernels[FUSED] = nk_fwd + nk_fused;
    pl.ops[SPLIT] = fwd;
    pl.ops[SPLIT].insert(pl.ops[SPLIT].end(), bwd_split.begin(), bwd_split.end());
    pl.nkernels[SPLIT] = nk_fwd + nk_split;
    for (int m : {FWD, FUSED, SPLIT}) assign_prefetch(pl.ops[m]);
    // data-parallel apply: allreduce(G) then the packed optimizer pass
    float* Pp = P;
    long long n4 = n_packed_ / 4;
    float lr = lr_, mom = mom_, wd = wd_;
    DpComm* dp = dp_.get();
    long long npk = n_packed_;
    const int opt = opt_;
    float* S1 = S1_.as<float>();
    float* S2 = opt_ == OPT_ADAGRAD ? S1 : S2_.as<float>();
    const float2* ctab = opt_ctab_.as<float2>();
    OptCounter* cnt = opt_cnt_.as<OptCounter>();
    static const char* opt_names[] = {"sgd", "adagrad", "adadelta", "adam"};
    const double opt_bytes = (double)npk * (opt == 0 ? 20 : opt == OPT_ADAGRAD ? 20 : 28);
    pl.ops[SPLIT_APPLY].push_back(Op([=](cudaStream_t s) {
        if (dp) dp->allreduce_f32(G, (size_t)npk, s);
        float4* p4 = reinterpret_cast<float4*>(Pp);
        const float4* g4 = reinterpret_cast<const float4*>(G);
        float4* a4 = reinterpret_cast<float4*>(S1);
        float4* b4 = reinterpret_cast<float4*>(S2);
        // OptimizerState defaults (optim.hpp:18-21): eps 1e-8, beta1 0.9, beta2 0.999, rho 0.95
        switch (opt) {
            case 0:
                launch_ex(sgd_packed_kernel, dim3(grid_for(n4)), dim3(256), 0, s, 1u, p4,
                          reinterpret_cast<float4*>(Vv), g4, n4, lr, mom, wd);
                break;
            case OPT_ADAGRAD:
                launch_ex(opt_packed_kernel<OPT_ADAGRAD>, dim3(grid_for(n4)), dim3(256), 0, s, 1u, p4, a4, b4, g4, n4,
                          lr, 1e-8f, 0.95f, 0.9f, 0.999f, ctab, cnt);
                break;
            case OPT_ADADELTA:
                launch_ex(opt_packed_kernel<OPT_ADADELTA>, dim3(grid_for(n4)), dim3(256), 0, s, 1u, p4, a4, b4, g4,
                          n4, lr, 1e-8f, 0.95f, 0.9f, 0.999f, ctab, cnt);
                break;
            default:
                launch_ex(opt_packed_kernel<OPT_ADAM>, dim3(grid_for(n4)), dim3(256), 0, s, 1u, p4, a4, b4, g4, n4,
                          lr, 1e-8f, 0.95f, 0.9f, 0.999f, ctab, cnt);
        }
    }, std::string(dp ? "allreduce+" : "") + opt_names[opt], 0.0, opt_bytes));
    pl.nkernels[SPLIT_APPLY] = 1;
    // the whole step
    if (!dp_ && opt_ == 0 && lr_ != 0.0f) {
        pl.ops[TRAIN] = pl.ops[FUSED];
        pl.nkernels[TRAIN] = pl.nkernels[FUSED];
    } else {
        pl.ops[TRAIN] = pl.ops[SPLIT];
        pl.nkernels[TRAIN] = pl.nkernels[SPLIT];
        if (dp_ || lr_ != 0.0f) {
            pl.ops[TRAIN].insert(pl.ops[TRAIN].end(), pl.ops[SPLIT_APPLY].begin(), pl.ops[SPLIT_APPLY].end());
            pl.nkernels[TRAIN] += pl.nkernels[SPLIT_APPLY];
        }
    }
}

// the host's count of adam steps keeps the bias-correction table filled ahead of the device counter
inline void Net::note_opt_step() {
    if (opt_ != OPT_ADAM) return;
    ++opt_steps_;
    if (opt_steps_ + 1 < opt_ctab_filled_) return;
    if (opt_steps_ + 2 > kCtabCap) throw Error(B2N_EPARAM, "adam: step counter exceeds the bias-correction table");
    const long long lo = opt_ctab_filled_, hi = std::min(kCtabCap, std::max(lo + 65536, opt_steps_ + 2));
    std::vector<float2> c((size_t)(hi - lo));
    for (long long t = lo; t < hi; ++t)  // adam_step (optim.hpp:118-119)
        c[(size_t)(t - lo)] = make_float2(1.0f - std::pow(0.9f, static_cast<float>(t)),
                                          1.0f - std::pow(0.999f, static_cast<float>(t)));
    B2N_CUDA(cudaMemcpyAsync(opt_ctab_.as<float2>() + lo, c.data(), c.size() * sizeof(float2), cudaMemcpyHostToDevice,
                             stream_));
    B2N_CUDA(cudaStreamSynchronize(stream_));
    opt_ctab_filled_ = hi;
}

inline void Net::launch(Plan& pl, int mode) {
    if (opt_ == OPT_ADAM && lr_ != 0.0f && (mode == TRAIN || mode == SPLIT_APPLY || mode == FIT || mode == STREAM0 ||
                                          mode == STREAM1))
        note_opt_step();
    if (!pl.graph[mode]) {
        cudaGraph_t graph;
        bool branched = false;
        for (const auto& op : pl.ops[mode]) branched = branched || op.branch;
        if (branched && !side_) {
            B2N_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
            B2N_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
            B2N_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
        }
        B2N_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
        try {
            // side-branch ops fork from the main stream right after the op before them (whose
            // outputs they read) and run beside the rest of the main chain; one join at the end
            for (auto& op : pl.ops[mode]) {
                if (op.branch) {
                    B2N_CUDA(cudaEventRecord(ev_fork_, stream_));
                    B2N_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
                    op(side_);
                } else {
                    op(stream_);
                }
            }
            if (branched) {
                B2N_CUDA(cudaEventRecord(ev_join_, side_));
                B2N_CUDA(cudaStreamWaitEvent(stream_, ev_join_, 0));
            }
        } catch (...) {
            cudaStreamEndCapture(stream_, &graph);
            throw;
        }
        B2N_CUDA(cudaStreamEndCapture(stream_, &graph));
        B2N_CUDA(cudaGraphInstantiate(&pl.graph[mode], graph, 0));
        cudaGraphDestroy(graph);
    }
    B2N_CUDA(cudaGraphLaunch(pl.graph[mode], stream_));
}

// --------------------------------------------------------------------------- stepping
inline void Net::stage_inputs(const float* x, const int* labels, long long B) {
    const long long in0 = numel(input_);
    B2N_CUDA(cudaMemcpy2DAsync(X_, ldx_ * 4, x, in0 * 4, in0 * 4, B, cudaMemcpyHostToDevice, stream_));
    if (labels) {
        for (long long r = 0; r < B; ++r)
            if (labels[r] < 0 || labels[r] >= classes_)
                throw Error(B2N_ELABEL, "softmax_cross_entropy: labels must be one-hot; row " + std::to_string(r));
        B2N_CUDA(cudaMemcpyAsync(labels_, labels, B * 4, cudaMemcpyHostToDevice, stream_));
    } else {
        B2N_CUDA(cudaMemsetAsync(labels_, 0, B * 4, stream_));
    }
}

inline double Net::read_loss(long long B) {
    B2N_CUDA(cudaMemcpyAsync(h_loss_.p, row_loss_, B * 8, cudaMemcpyDeviceToHost, stream_));
    spin_sync(stream_);
    double loss = 0.0;  // network.hpp:433-435: sequential over rows, then / batch
    const double* rl = h_loss_.as<double>();
    for (long long r = 0; r < B; ++r) loss += rl[r];
    return loss;
}

inline double Net::train(const float* x, const int* labels, long long B) {
    if (B < 1) throw Error(B2N_ESHAPE, "network input expects (batch >= 1, ...)");
    check_train_params();
    ensure_capacity(B);
    if (B > 4096) h_loss_.alloc(B * 8);
    stage_inputs(x, labels, B);
    if (dp_) {
        throw Error(B2N_EPARAM, "data-parallel nets step through forward_backward + apply_update");
    }
    Plan& pl = plan_for(B, B);
    launch(pl, TRAIN);
    last_B_ = B;
    last_Bg_ = B;
    return read_loss(B) / (double)B;
}

inline void Net::build_stream_ops(Plan& pl, int j) {
    const long long B = pl.B;
    const long long per = numel(input_);
    float* X = X_;
    const long long ldx = ldx_;
    int* lab = labels_;
    const float* sx = sx_[j].as<float>();
    const int* sl = sl_[j].as<int>();
    std::vector<Op> ops;
    ops.push_back(Op([=](cudaStream_t s) {  // staging buffer j -> the step's input / label buffers
        B2N_CUDA(cudaMemcpy2DAsync(X, ldx * 4, sx, per * 4, per * 4, B, cudaMemcpyDeviceToDevice, s));
        B2N_CUDA(cudaMemcpyAsync(lab, sl, B * 4, cudaMemcpyDeviceToDevice, s));
    }, "stream.stage", 0.0, (double)B * (per + 1) * 8, 0));
    const std::vector<Op>& body = pl.ops[TRAIN];
    ops.insert(ops.end(), body.begin(), body.end());
    const double* rl = row_loss_;
    double* out = sloss_.as<double>() + 1;
    ops.push_back(Op([=](cudaStream_t s) {
        launch_ex(stream_loss_kernel, dim3(1), dim3(32), 0, s, 1u, rl, (int)B, out);
    }, "stream.loss", 0.0, (double)B * 8));
    assign_prefetch(ops);
    pl.ops[STREAM0 + j] = ops;
    int n = 0;
    for (const Op& o : ops) n += o.kernels;
    pl.nkernels[STREAM0 + j] = n;
}

inline void Net::train_stream(const float* x, const int* labels, long long steps, long long B, double* loss_out) {
    if (B < 1 || steps < 1) throw Error(B2N_ESHAPE, "train_stream: need steps >= 1 and batch >= 1");
    if (dp_) throw Error(B2N_EPARAM, "data-parallel nets step through forward_backward + apply_update");
    check_train_params();
    for (long long r = 0; r < steps * B; ++r)  // softmax_cross_entropy's one-hot check (network.hpp:423-432)
        if (labels[r] < 0 || labels[r] >= classes_)
            throw Error(B2N_ELABEL, "softmax_cross_entropy: labels must be one-hot; row " + std::to_string(r % B));
    ensure_capacity(B);
    const long long per = numel(input_);
    if (sx_[0].bytes < (size_t)(cap_ * per * 4) || !sloss_.p) {
        for (int j = 0; j < 2; ++j) {
            sx_[j].alloc((size_t)(cap_ * per * 4));
            sl_[j].alloc((size_t)cap_ * 4);
        }
        sloss_.alloc((size_t)(kStreamChunk + 1) * 8);
        for (auto& kv : plans_)  // stream graphs captured the old staging pointers
            for (int m : {STREAM0, STREAM1}) {
                if (kv.second->graph[m]) cudaGraphExecDestroy(kv.second->graph[m]);
                kv.second->graph[m] = nullptr;
                kv.second->ops[m].clear();
            }
    }
    for (int j = 0; j < 2; ++j) {
        if (!ev_copied_[j]) B2N_CUDA(cudaEventCreateWithFlags(&ev_copied_[j], cudaEventDisableTiming));
        if (!ev_used_[j]) B2N_CUDA(cudaEventCreateWithFlags(&ev_used_[j], cudaEventDisableTiming));
    }
    if (!copy_stream_) B2N_CUDA(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));
    Plan& pl = plan_for(B, B);
    for (int j = 0; j < 2; ++j)
        if (pl.ops[STREAM0 + j].empty()) build_stream_ops(pl, j);
    B2N_CUDA(cudaEventRecord(ev_used_[0], stream_));  // staging buffers free after prior work
    B2N_CUDA(cudaEventRecord(ev_used_[1], stream_));
    for (long long c0 = 0; c0 < steps; c0 += kStreamChunk) {
        const long long n = std::min(kStreamChunk, steps - c0);
        B2N_CUDA(cudaMemsetAsync(sloss_.p, 0, 8, stream_));  // step counter
        for (long long i = c0; i < c0 + n; ++i) {
            const int j = (int)(i & 1);
            B2N_CUDA(cudaStreamWaitEvent(copy_stream_, ev_used_[j], 0));  // step i - 2 done with buffer j
            B2N_CUDA(cudaMemcpyAsync(sx_[j].p, x + i * B * per, (size_t)(B * per * 4), cudaMemcpyHostToDevice,
                                     copy_stream_));
            B2N_CUDA(cudaMemcpyAsync(sl_[j].p, labels + i * B, (size_t)B * 4, cudaMemcpyHostToDevice, copy_stream_));
            B2N_CUDA(cudaEventRecord(ev_copied_[j], copy_stream_));
            B2N_CUDA(cudaStreamWaitEvent(stream_, ev_copied_[j], 0));
            launch(pl, STREAM0 + j);
            B2N_CUDA(cudaEventRecord(ev_used_[j], stream_));
        }
        std::vector<double> h((size_t)n);
        B2N_CUDA(cudaMemcpyAsync(h.data(), sloss_.as<double>() + 1, (size_t)n * 8, cudaMemcpyDeviceToHost, stream_));
        spin_sync(stream_);
        for (long long i = 0; i < n; ++i) loss_out[c0 + i] = h[(size_t)i] / (double)B;
    }
    last_B_ = B;
    last_Bg_ = B;
}

inline double Net::forward_backward(const float* x, const int* labels, long long B, long long Bg) {
    if (B < 1 || Bg < B) throw Error(B2N_ESHAPE, "forward_backward: need 1 <= batch <= batch_global");
    ensure_capacity(B);
    stage_inputs(x, labels, B);
    Plan& pl = plan_for(B, Bg);
    launch(pl, SPLIT);
    last_B_ = B;
    last_Bg_ = Bg;
    return read_loss(B) / (double)Bg;
}

inline void Net::apply_update() {
    check_train_params();
    if (!last_B_) throw Error(B2N_EPARAM, "apply_update before forward_backward");
    Plan& pl = plan_for(last_B_, last_Bg_);
    if (lr_ != 0.0f) launch(pl, SPLIT_APPLY);
    B2N_CUDA(cudaStreamSynchronize(stream_));
}

inline void Net::forward(const float* x, long long B, float* probs, int* argmax) {
    if (B < 1) throw Error(B2N_ESHAPE, "forward_batch: batch must be >= 1");
    ensure_capacity(B);
    stage_inputs(x, nullptr, B);
    Plan& pl = plan_for(B, B);
    launch(pl, FWD);
    if (probs) B2N_CUDA(cudaMemcpyAsync(probs, probs_, B * classes_ * 4, cudaMemcpyDeviceToHost, stream_));
    if (argmax) B2N_CUDA(cudaMemcpyAsync(argmax, argmax_, B * 4, cudaMemcpyDeviceToHost, stream_));
    B2N_CUDA(cudaStreamSynchronize(stream_));
}

inline void Net::stage(const float* x, const int* labels, long long B) {
    ensure_capacity(B);
    stage_inputs(x, labels, B);
    B2N_CUDA(cudaStreamSynchronize(stream_));
    last_B_ = B;
}

inline void Net::run_staged(int steps, long long Bg) {
    if (!last_B_) throw Error(B2N_EPARAM, "run_staged before stage");
    check_train_params();
    Plan& pl = plan_for(last_B_, Bg ? Bg : last_B_);
    last_Bg_ = pl.Bg;
    for (int s = 0; s < steps; ++s) launch(pl, TRAIN);
}

inline double Net::loss() { return read_loss(last_B_) / (double)(last_Bg_ ? last_Bg_ : last_B_); }

inline int Net::kernels_per_step(long long B) {
    Plan& pl = plan_for(B, B);
    return pl.nkernels[TRAIN];
}

// --------------------------------------------------------------------------- fit / evaluate
inline void Net::upload_dataset(const float* images, const int* labels, long long N) {
    const long long per = numel(input_);
    for (long long r = 0; r < N; ++r)  // data.hpp:257-260 (BatchIterator::next)
        if (labels[r] < 0 || labels[r] >= classes_)
            throw Error(B2N_ECONSISTENCY, "batch_iterator: label " + std::to_string(labels[r]) + " outside [0, " +
                                        std::to_string(classes_) + ")");
    bool moved = false;  // the FIT / EVAL graphs bake these addresses in
    if (ds_x_.bytes < (size_t)(N * per * 4)) ds_x_.alloc((size_t)(N * per * 4)), moved = true;
    if (ds_y_.bytes < (size_t)(N * 4)) ds_y_.alloc((size_t)(N * 4)), moved = true;
    if (ds_order_.bytes < (size_t)(N * 4)) ds_order_.alloc((size_t)(N * 4)), moved = true;
    if (!fit_state_.p) fit_state_.alloc(sizeof(FitState)), moved = true;
    if (moved)
        for (auto& kv : plans_)
            for (int m : {FIT, EVAL}) {
                kv.second->ops[m].clear();
                if (kv.second->graph[m]) cudaGraphExecDestroy(kv.second->graph[m]);
                kv.second->graph[m] = nullptr;
            }
    B2N_CUDA(cudaMemcpyAsync(ds_x_.p, images, (size_t)(N * per * 4), cudaMemcpyHostToDevice, stream_));
    B2N_CUDA(cudaMemcpyAsync(ds_y_.p, labels, (size_t)(N * 4), cudaMemcpyHostToDevice, stream_));
    ds_n_ = N;
}

// FIT: gather -> training step -> loss sum + cursor; EVAL: gather -> forward -> correct count + cursor
inline void Net::build_fit_ops(Plan& pl, int mode) {
    const int count = (int)pl.B;
    const long long per = numel(input_);
    const float* ds = ds_x_.as<float>();
    const int* dy = ds_y_.as<int>();
    const int* ord = ds_order_.as<int>();
    FitState* st = fit_state_.as<FitState>();
    float* X = X_;
    long long ldx = ldx_;
    int* lab = labels_;
    std::vector<Op> ops;
    ops.push_back(Op([=](cudaStream_t s) {
        const long long n = (long long)count * per / 4 + 1;
        launch_ex(fit_gather_kernel, dim3(grid_for(n)), dim3(256), 0, s, 1u, ds, per, dy, ord, (const FitState*)st, count,
                  X, ldx, lab);
    }, "fit.gather", 0.0, (double)count * per * 8));
    const std::vector<Op>& body = pl.ops[mode == FIT ? TRAIN : FWD];
    ops.insert(ops.end(), body.begin(), body.end());
    const double* rl = row_loss_;
    const int* am = argmax_;
    const int eval = mode == EVAL;
    ops.push_back(Op([=](cudaStream_t s) {
        launch_ex(fit_advance_kernel, dim3(1), dim3(32), 0, s, 1u, rl, count, st, eval, am, (const int*)lab);
    }, "fit.advance", 0.0, (double)count * 16));
    assign_prefetch(ops);
    pl.ops[mode] = ops;
    int n = 0;
    for (const Op& o : ops) n += o.kernels;
    pl.nkernels[mode] = n;
}

inline double Net::run_epoch_eval(long long N) {
    B2N_CUDA(cudaMemsetAsync(fit_state_.p, 0, sizeof(FitState), stream_));
    const long long B = batch_size_;  // network.hpp:477
    for (long long pos = 0; pos < N; pos += B) {
        const long long count = std::min(B, N - pos);
        Plan& pl = plan_for(count, count);
        if (pl.ops[EVAL].empty()) build_fit_ops(pl, EVAL);
        launch(pl, EVAL);
    }
    FitState h;
    B2N_CUDA(cudaMemcpyAsync(&h, fit_state_.p, sizeof(FitState), cudaMemcpyDeviceToHost, stream_));
    spin_sync(stream_);
    return (double)h.correct / (double)N;
}

inline std::vector<Net::FitEpoch> Net::fit(const float* images, const int* labels, long long N, int epochs) {
    const unsigned seed = seed_;  // BatchIterator(train, net.batch_size, net.seed)
    if (N < 1) throw Error(B2N_EDATA, "fit: empty dataset");
    if (epochs < 1) throw Error(B2N_EPARAM, "fit: epochs must be >= 1");
    if (dp_) throw Error(B2N_EPARAM, "fit: data-parallel nets step through forward_backward + apply_update");
    check_train_params();
    const long long B = batch_size_;  // network.hpp:494
    ensure_capacity(B);
    upload_dataset(images, labels, N);
    std::vector<long long> order;
    std::vector<int> order32((size_t)N);
    std::vector<FitEpoch> out;
    for (int e = 0; e < epochs; ++e) {
        batch_order(order, N, seed, e);
        for (long long i = 0; i < N; ++i) order32[(size_t)i] = (int)order[(size_t)i];
        B2N_CUDA(cudaMemcpyAsync(ds_order_.p, order32.data(), (size_t)N * 4, cudaMemcpyHostToDevice, stream_));
        B2N_CUDA(cudaMemsetAsync(fit_state_.p, 0, sizeof(FitState), stream_));
        spin_sync(stream_);  // the order buffer is a pageable host copy: complete before it changes
        const auto t0 = std::chrono::steady_clock::now();
        for (long long pos = 0; pos < N; pos += B) {
            const long long count = std::min(B, N - pos);
            Plan& pl = plan_for(count, count);
            if (pl.ops[FIT].empty()) build_fit_ops(pl, FIT);
            launch(pl, FIT);
        }
        FitState h;
        B2N_CUDA(cudaMemcpyAsync(&h, fit_state_.p, sizeof(FitState), cudaMemcpyDeviceToHost, stream_));
        spin_sync(stream_);
        const auto t1 = std::chrono::steady_clock::now();
        FitEpoch fe;
        fe.loss = h.loss_sum / (double)N;
        fe.seconds = std::chrono::duration<double>(t1 - t0).count();
        fe.accuracy = run_epoch_eval(N);  // evaluate(net, train) over the same resident data, in order
        out.push_back(fe);
    }
    return out;
}

inline double Net::evaluate(const float* images, const int* labels, long long N) {
    if (N < 1) throw Error(B2N_EDATA, "evaluate: empty dataset");
    ensure_capacity(batch_size_);
    upload_dataset(images, labels, N);
    std::vector<int> iota((size_t)N);
    for (long long i = 0; i < N; ++i) iota[(size_t)i] = (int)i;
    B2N_CUDA(cudaMemcpyAsync(ds_order_.p, iota.data(), (size_t)N * 4, cudaMemcpyHostToDevice, stream_));
    spin_sync(stream_);
    return run_epoch_eval(N);
}

// --------------------------------------------------------------------------- checkpoint
inline void Net::gather_params(const std::vector<float>& packed, int idx, float* out) const {
    const ParamView& v = params_[idx];
    for (long long r = 0; r < v.rows; ++r)
        for (long long c = 0; c < v.cols; ++c) out[r * v.cols + c] = packed[(size_t)(v.off + r * v.pitch + c)];
}
inline void Net::scatter_params(std::vector<float>& packed, int idx, const float* in) const {
    const ParamView& v = params_[idx];
    for (long long r = 0; r < v.rows; ++r)
        for (long long c = 0; c < v.cols; ++c) packed[(size_t)(v.off + r * v.pitch + c)] = in[r * v.cols + c];
}

inline void Net::save(const std::string& path, bool with_state) {
    std::vector<float> packed((size_t)n_packed_), tmp;
    B2N_CUDA(cudaMemcpyAsync(packed.data(), P_.p, (size_t)n_packed_ * 4, cudaMemcpyDeviceToHost, stream_));
    B2N_CUDA(cudaStreamSynchronize(stream_));
    std::string o;
    o.append("FNN1", 4);
    ckpt::put_u32(o, (uint32_t)spec_kinds_.size());
    int pi = 0;
    auto put_tensor = [&](const std::vector<float>& src, int idx) {
        const ParamView& v = params_[idx];
        ckpt::put_u32(o, (uint32_t)v.dims.size());
        for (long long e : v.dims) ckpt::put_u64(o, (uint64_t)e);
        tmp.resize((size_t)numel(v.dims));
        gather_params(src, idx, tmp.data());
        ckpt::put_f32s(o, tmp.data(), tmp.size());
    };
    for (int kind : spec_kinds_) {
        const std::string tag = ckpt::tag_of(kind);
        ckpt::put_u32(o, (uint32_t)tag.size());
        o.append(tag);
        const int n = kind == B2N_DENSE || kind == B2N_CONV ? 2 : 0;
        ckpt::put_u32(o, (uint32_t)n);
        for (int t = 0; t < n; ++t) put_tensor(packed, pi++);
    }
    ckpt::write_file(path, o, "save_network");
    if (!with_state) return;
    o.clear();
    o.append("B2NS", 4);
    ckpt::put_u32(o, 2);
    ckpt::put_u32(o, (uint32_t)opt_);
    OptCounter oc{};
    if (opt_cnt_.p) B2N_CUDA(cudaMemcpyAsync(&oc, opt_cnt_.p, sizeof(oc), cudaMemcpyDeviceToHost, stream_));
    B2N_CUDA(cudaStreamSynchronize(stream_));
    ckpt::put_u64(o, (uint64_t)oc.t);
    const float hp[3] = {lr_, mom_, wd_};
    ckpt::put_f32s(o, hp, 3);
    const int nbuf = opt_ == 0 ? 1 : opt_ == OPT_ADAGRAD ? 1 : 2;
    ckpt::put_u32(o, (uint32_t)nbuf);
    for (int b = 0; b < nbuf; ++b) {  // velocity (sgd) or the optimizer's state buffers
        DevMem& src = opt_ == 0 ? V_ : b == 0 ? S1_ : S2_;
        B2N_CUDA(cudaMemcpyAsync(packed.data(), src.p, (size_t)n_packed_ * 4, cudaMemcpyDeviceToHost, stream_));
        B2N_CUDA(cudaStreamSynchronize(stream_));
        ckpt::put_u32(o, (uint32_t)params_.size());
        for (int i = 0; i < (int)params_.size(); ++i) put_tensor(packed, i);
    }
    ckpt::write_file(path + ".state", o, "save_network");
}

inline void Net::load(const std::string& path, bool with_state) {
    ckpt::Reader rd;
    rd.buf = ckpt::read_file(path, "load_network");
    if (rd.bytes(4) != "FNN1") throw Error(B2N_EFORMAT, "load_network: bad magic; expected FNN1");
    const uint32_t nl = rd.u32();
    if (nl != spec_kinds_.size())
        throw Error(B2N_EFORMAT, "load_network: checkpoint has " + std::to_string(nl) + " layers; network has " +
                                     std::to_string(spec_kinds_.size()));
    // parse everything before touching the device: a failed load leaves the parameters unchanged
    std::vector<float> packed((size_t)n_packed_), tmp;
    B2N_CUDA(cudaMemcpyAsync(packed.data(), P_.p, (size_t)n_packed_ * 4, cudaMemcpyDeviceToHost, stream_));
    B2N_CUDA(cudaStreamSynchronize(stream_));
    auto get_tensor = [&](ckpt::Reader& r, std::vector<float>& dst, int idx, const std::string& tag) {
        const ParamView& v = params_[idx];
        const uint32_t rank = r.u32();
        if (rank != v.dims.size())
            throw Error(B2N_EFORMAT, "load_network: tensor rank mismatch in layer '" + tag + "'");
        for (size_t d = 0; d < rank; ++d)
            if (r.u64() != (uint64_t)v.dims[d])
                throw Error(B2N_EFORMAT, "load_network: tensor extent mismatch in layer '" + tag + "'");
        tmp.resize((size_t)numel(v.dims));
        r.f32s(tmp.data(), tmp.size());
        scatter_params(dst, idx, tmp.data());
    };
    int pi = 0;
    for (int kind : spec_kinds_) {
        const uint32_t taglen = rd.u32();
        if (taglen > 64) throw Error(B2N_EFORMAT, "load_network: implausible tag length");
        const std::string tag = rd.bytes(taglen);
        const std::string want = ckpt::tag_of(kind);
        if (tag != want)
            throw Error(B2N_EFORMAT,
                        "load_network: layer tag mismatch; checkpoint '" + tag + "' vs network '" + want + "'");
        const uint32_t count = rd.u32();
        const uint32_t n = kind == B2N_DENSE || kind == B2N_CONV ? 2 : 0;
        if (count != n) throw Error(B2N_EFORMAT, "load_network: tensor count mismatch in layer '" + tag + "'");
        for (uint32_t t = 0; t < n; ++t) get_tensor(rd, packed, pi++, tag);
    }
    std::vector<std::vector<float>> bufs;
    float hp[3] = {lr_, mom_, wd_};
    uint64_t t = 0;
    if (with_state) {
        ckpt::Reader sr;
        sr.buf = ckpt::read_file(path + ".state", "load_network");
        if (sr.bytes(4) != "B2NS" || sr.u32() != 2) throw Error(B2N_EFORMAT, "load_network: bad state sidecar");
        if ((int)sr.u32() != opt_) throw Error(B2N_EFORMAT, "load_network: state sidecar is for another optimizer");
        t = sr.u64();
        sr.f32s(hp, 3);
        const uint32_t nbuf = sr.u32();
        if (nbuf != (opt_ == 0 || opt_ == OPT_ADAGRAD ? 1u : 2u))
            throw Error(B2N_EFORMAT, "load_network: state buffer count mismatch");
        for (uint32_t b = 0; b < nbuf; ++b) {
            if (sr.u32() != params_.size()) throw Error(B2N_EFORMAT, "load_network: state tensor count mismatch");
            bufs.emplace_back((size_t)n_packed_, 0.0f);
            for (int i = 0; i < (int)params_.size(); ++i) get_tensor(sr, bufs.back(), i, "state");
        }
    }
    B2N_CUDA(cudaMemcpyAsync(P_.p, packed.data(), (size_t)n_packed_ * 4, cudaMemcpyHostToDevice, stream_));
    if (with_state) {
        for (size_t b = 0; b < bufs.size(); ++b) {
            DevMem& dst = opt_ == 0 ? V_ : b == 0 ? S1_ : S2_;
            B2N_CUDA(cudaMemcpyAsync(dst.p, bufs[b].data(), (size_t)n_packed_ * 4, cudaMemcpyHostToDevice, stream_));
        }
        if (opt_cnt_.p) {
            const OptCounter oc{(long long)t, 0u};
            B2N_CUDA(cudaMemcpyAsync(opt_cnt_.p, &oc, sizeof(oc), cudaMemcpyHostToDevice, stream_));
            B2N_CUDA(cudaStreamSynchronize(stream_));
            opt_steps_ = (long long)t - 1;
            if (opt_ == OPT_ADAM) note_opt_step();  // table filled past t; opt_steps_ back to t
        }
        if (hp[0] != lr_ || hp[1] != mom_ || hp[2] != wd_) set_hparams(hp[0], hp[1], hp[2]);
    }
    B2N_CUDA(cudaStreamSynchronize(stream_));
}

// --------------------------------------------------------------------------- params
inline DevMem& Net::state_buffer(int which) {
    switch (which) {
        case B2N_VALUE: return P_;
        case B2N_GRAD: return G_;
        case B2N_VELOCITY: return V_;
        case B2N_OPT_STATE1:
            if (S1_.p) return S1_;
            break;
        case B2N_OPT_STATE2:
            if (S2_.p) return S2_;
            break;
    }
    throw Error(B2N_EBOUNDS, "parameter view " + std::to_string(which) + " does not exist for this optimizer");
}

inline void Net::get_param(int idx, int which, float* host) {
    if (idx < 0 || idx >= num_params()) throw Error(B2N_EBOUNDS, "param index out of range");
    const ParamView& v = params_[idx];
    const float* base = state_buffer(which).as<float>() + v.off;
    B2N_CUDA(cudaMemcpy2DAsync(host, v.cols * 4, base, v.pitch * 4, v.cols * 4, v.rows, cudaMemcpyDeviceToHost,
                               stream_));
    B2N_CUDA(cudaStreamSynchronize(stream_));
}

inline void Net::set_param(int idx, int which, const float* host) {
    if (idx < 0 || idx >= num_params()) throw Error(B2N_EBOUNDS, "param index out of range");
    const ParamView& v = params_[idx];
    float* base = state_buffer(which).as<float>() + v.off;
    B2N_CUDA(cudaMemcpy2DAsync(base, v.pitch * 4, host, v.cols * 4, v.cols * 4, v.rows, cudaMemcpyHostToDevice,
                               stream_));
    B2N_CUDA(cudaStreamSynchronize(stream_));
}

// The last forward's output of fused layer li (act + pool applied) for `batch` rows, NCHW per row
// (conv) or [batch][out] (dense), plus the pool argmax codes (window order (0,0) (0,1) (1,0) (1,1)) in
// the same NCHW order -- per-layer forward parity against the reference's conv_forward / pool_forward.
inline void Net::layer_output(int li, long long batch, float* host, uint8_t* codes_host) {
    if (li < 0 || li >= (int)layers_.size()) throw Error(B2N_EBOUNDS, "layer index out of range");
    if (batch < 1 || batch > cap_) throw Error(B2N_EBOUNDS, "batch exceeds the staged capacity");
    const Layer& L = layers_[li];
    B2N_CUDA(cudaStreamSynchronize(stream_));
    if (!L.Aout) throw Error(B2N_EPARAM, "the last layer keeps no activation buffer (use forward_batch)");
    if (L.kind == B2N_DENSE) {
        B2N_CUDA(cudaMemcpy2D(host, L.out * 4, L.Aout, L.ld_out * 4, L.out * 4, batch, cudaMemcpyDeviceToHost));
        return;
    }
    const long long k = L.out_shape[0], oh = L.out_shape[1], ow = L.out_shape[2], per = k * oh * ow;
    const long long kq = (k + 3) / 4;
    std::vector<float> raw((size_t)(batch * L.ld_out));
    B2N_CUDA(cudaMemcpy(raw.data(), L.Aout, raw.size() * 4, cudaMemcpyDeviceToHost));
    for (long long b = 0; b < batch; ++b)
        for (long long c = 0; c < k; ++c)
            for (long long y = 0; y < oh; ++y)
                for (long long x = 0; x < ow; ++x)
                    host[((b * k + c) * oh + y) * ow + x] =
                        L.blocked_out ? raw[(size_t)(b * L.ld_out + ((y * kq + c / 4) * ow + x) * 4 + c % 4)]
                                      : raw[(size_t)(b * L.ld_out + (c * oh + y) * ow + x)];
    if (codes_host && L.pool_after && L.arg) {
        std::vector<uint8_t> cr((size_t)(batch * L.codes_bstride));
        B2N_CUDA(cudaMemcpy(cr.data(), L.arg, cr.size(), cudaMemcpyDeviceToHost));
        for (long long b = 0; b < batch; ++b)
            for (long long c = 0; c < k; ++c)
                for (long long y = 0; y < oh; ++y)
                    for (long long x = 0; x < ow; ++x)
                        codes_host[((b * k + c) * oh + y) * ow + x] =
                            tconv_ ? cr[(size_t)(b * L.codes_bstride + ((y * kq + c / 4) * L.codes_pw + x) * 4 + c % 4)]
                                   : cr[(size_t)(b * L.codes_bstride + (c * oh + y) * ow + x)];
    }
    (void)per;
}

}  // namespace b2n
