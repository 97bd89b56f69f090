// ref_shim.cpp -- extern "C" access to the UNMODIFIED reference (TEST INFRASTRUCTURE ONLY).
//
// Compiled by oracle/Makefile against the reference headers where they lie
// (-I/root/reference/proj/include) into oracle/_ref/libfastnn_ref.so. Nothing from the reference
// is copied into this repository. Used for two things only:
//   1. generating / checking the golden vectors that pin oracle/fastnn_oracle.cpp
//      (tests/golden/make_golden.py), and
//   2. the CPU baseline ("cpu_baseline.kind = reference") timed by bench.py on the GPU box's host.
// For pad = 0 networks this drives the reference's own build_network / train_minibatch
// (network.hpp:284, :463) and cd_k_update (energy.hpp:131). The reference cannot build the
// ImageNet-shaped config (network.hpp:335 rejects 125x125 before a pool; LayerDesc has no pad;
// layers.hpp:159 rejects a padded backward), so pad > 0 networks run the SURVEY 8(c) composite of
// reference primitives: conv_forward with ConvShape.pad, dx = crop(conv_full(dy, kt)),
// gk += sum_img add_corr_map(pad_spatial(x), dy).
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "fastnn/energy.hpp"
#include "fastnn/network.hpp"

using namespace fastnn;

namespace {

struct orc_layer_c {
    int kind;
    long long in, out, k, kh, kw, pad;
    float p;
};

Tensor make_batch(const float* x, long long B, const std::vector<long long>& per) {
    std::vector<long long> dims{B};
    for (long long e : per) dims.push_back(e);
    Tensor t = make_tensor(dims);
    const std::size_t n = t.last_dim();
    for (std::size_t r = 0; r < t.rows_total(); ++r) std::memcpy(t.row_ptr(r), x + r * n, n * sizeof(float));
    return t;
}

void copy_out(const Tensor& t, float* out) {
    const std::size_t n = t.last_dim();
    for (std::size_t r = 0; r < t.rows_total(); ++r) std::memcpy(out + r * n, t.row_ptr(r), n * sizeof(float));
}

void copy_in(Tensor& t, const float* in) {
    const std::size_t n = t.last_dim();
    for (std::size_t r = 0; r < t.rows_total(); ++r) std::memcpy(t.row_ptr(r), in + r * n, n * sizeof(float));
}

Tensor one_hot(const int* labels, long long B, long long C) {
    Tensor y = make_tensor({B, C});
    for (long long r = 0; r < B; ++r) y.at(r, labels[r]) = 1.0f;
    return y;
}

// ----- composite padded conv node (reference primitives only) -----
class PaddedConvNode final : public NetLayer {
  public:
    explicit PaddedConvNode(const ConvShape& s) : layer_(s) {}
    Tensor forward(const Tensor& x, bool, std::mt19937&) override {
        x_ = x;
        return conv_forward(layer_, x);  // conv_valid with ConvShape.pad (conv.hpp:182-189, :230-235)
    }
    Tensor backward(const Tensor& dy) override {
        const ConvShape& s = layer_.shape;
        const std::size_t n = x_.dim(0), p = s.pad;
        const std::size_t oh = s.h + 2 * p - s.kh + 1, ow = s.w + 2 * p - s.kw + 1;
        Tensor kt = make_tensor({(long long)s.c_in, (long long)s.k, (long long)s.kh, (long long)s.kw});
        for (std::size_t f = 0; f < s.k; ++f)
            for (std::size_t c = 0; c < s.c_in; ++c)
                for (std::size_t di = 0; di < s.kh; ++di)
                    for (std::size_t dj = 0; dj < s.kw; ++dj) kt.at(c, f, di, dj) = layer_.kernels.at(f, c, di, dj);
        ConvShape sb;
        sb.n = n;
        sb.c_in = s.k;
        sb.k = s.c_in;
        sb.kh = s.kh;
        sb.kw = s.kw;
        sb.h = oh;
        sb.w = ow;
        Tensor full = conv_full(dy, kt, sb);  // (n, c_in, h+2p, w+2p)
        Tensor dx = make_tensor({(long long)n, (long long)s.c_in, (long long)s.h, (long long)s.w});
        for (std::size_t b = 0; b < n; ++b)
            for (std::size_t c = 0; c < s.c_in; ++c)
                for (std::size_t y = 0; y < s.h; ++y)
                    std::memcpy(&dx.at(b, c, y, 0), &full.at(b, c, y + p, p), s.w * sizeof(float));
        Tensor xp = detail::pad_spatial(x_, p, p);
        for (std::size_t f = 0; f < s.k; ++f)
            for (std::size_t c = 0; c < s.c_in; ++c) {
                float* dst = &layer_.gk.at(f, c, 0, 0);
                for (std::size_t img = 0; img < n; ++img)
                    detail::add_corr_map(dst, layer_.gk.stride_last(), &xp.at(img, c, 0, 0), xp.stride_last(),
                                         &dy.at(img, f, 0, 0), dy.stride_last(), oh, ow, s.kh, s.kw);
            }
        float* gb = layer_.gb.row_ptr(0);
        for (std::size_t img = 0; img < n; ++img)
            for (std::size_t f = 0; f < s.k; ++f)
                for (std::size_t oy = 0; oy < oh; ++oy) {
                    const float* q = &dy.at(img, f, oy, 0);
                    for (std::size_t ox = 0; ox < ow; ++ox) gb[f] += q[ox];
                }
        return dx;
    }
    std::string tag() const override { return "conv"; }
    std::vector<ParamRef> trainable() override { return {{&layer_.kernels, &layer_.gk}, {&layer_.b, &layer_.gb}}; }
    ConvLayer& impl() { return layer_; }

  private:
    ConvLayer layer_;
    Tensor x_;
};

class ActNodeC final : public NetLayer {
  public:
    explicit ActNodeC(Activation k) : kind_(k) {}
    Tensor forward(const Tensor& x, bool, std::mt19937&) override { return y_ = activation_apply(kind_, x); }
    Tensor backward(const Tensor& dy) override { return activation_gradient(kind_, y_, dy); }
    std::string tag() const override { return "act"; }

  private:
    Activation kind_;
    Tensor y_;
};

class PoolNodeC final : public NetLayer {
  public:
    Tensor forward(const Tensor& x, bool, std::mt19937&) override {
        PoolResult r = pool_forward(PoolMode::Max, x);
        arg_ = r.argmax;
        return r.y;
    }
    Tensor backward(const Tensor& dy) override { return pool_backward(PoolMode::Max, dy, arg_); }
    std::string tag() const override { return "maxpool"; }

  private:
    Tensor arg_;
};

class FlattenNodeC final : public NetLayer {
  public:
    FlattenNodeC(std::size_t c, std::size_t h, std::size_t w) : c_(c), h_(h), w_(w) {}
    Tensor forward(const Tensor& x, bool, std::mt19937&) override { return detail::flatten_batch(x); }
    Tensor backward(const Tensor& dy) override { return detail::unflatten_batch(dy, c_, h_, w_); }
    std::string tag() const override { return "flatten"; }

  private:
    std::size_t c_, h_, w_;
};

class DenseNodeC final : public NetLayer {
  public:
    DenseNodeC(std::size_t o, std::size_t i) : layer_(o, i) {}
    Tensor forward(const Tensor& x, bool, std::mt19937&) override {
        x_ = x;
        return dense_forward(layer_, x);
    }
    Tensor backward(const Tensor& dy) override { return dense_backward(layer_, x_, dy); }
    std::string tag() const override { return "dense"; }
    std::vector<ParamRef> trainable() override { return {{&layer_.w, &layer_.gw}, {&layer_.b, &layer_.gb}}; }
    DenseLayer& impl() { return layer_; }

  private:
    DenseLayer layer_;
    Tensor x_;
};

class SoftmaxNodeC final : public NetLayer {
  public:
    Tensor forward(const Tensor& x, bool, std::mt19937&) override { return softmax(x); }
    Tensor backward(const Tensor& dy) override { return dy.clone(); }
    std::string tag() const override { return "softmax"; }
};

struct RefNet {
    Network net;
    long long classes = 0;
    std::string err;
};

// the pad > 0 composite, built node by node with the same init order as build_network
bool build_composite(RefNet& rn, const std::vector<long long>& input, const orc_layer_c* d, int n, unsigned seed) {
    Network& net = rn.net;
    net.input = input;
    net.seed = seed;
    net.rng.seed(seed);
    std::vector<long long> cur = input;
    for (int i = 0; i < n; ++i) {
        switch (d[i].kind) {
            case 0:  // dense
                if (cur.size() == 3) {
                    net.layers.push_back(std::make_unique<FlattenNodeC>(cur[0], cur[1], cur[2]));
                    cur = {cur[0] * cur[1] * cur[2]};
                }
                net.layers.push_back(std::make_unique<DenseNodeC>(d[i].out, d[i].in));
                cur = {d[i].out};
                break;
            case 1: {
                ConvShape s;
                s.c_in = cur[0];
                s.k = d[i].k;
                s.kh = d[i].kh;
                s.kw = d[i].kw;
                s.h = cur[1];
                s.w = cur[2];
                s.pad = d[i].pad;
                net.layers.push_back(std::make_unique<PaddedConvNode>(s));
                cur = {d[i].k, cur[1] + 2 * d[i].pad - d[i].kh + 1, cur[2] + 2 * d[i].pad - d[i].kw + 1};
                break;
            }
            case 2:
                net.layers.push_back(std::make_unique<PoolNodeC>());
                cur = {cur[0], cur[1] / 2, cur[2] / 2};
                break;
            case 3: net.layers.push_back(std::make_unique<ActNodeC>(Activation::Sigmoid)); break;
            case 4: net.layers.push_back(std::make_unique<ActNodeC>(Activation::Relu)); break;
            case 5: net.layers.push_back(std::make_unique<SoftmaxNodeC>()); break;
            default: return false;
        }
    }
    rn.classes = cur[0];
    std::mt19937 init_rng(seed);
    for (auto& l : net.layers) {
        if (auto* dn = dynamic_cast<DenseNodeC*>(l.get())) dn->impl().init(init_rng);
        if (auto* cn = dynamic_cast<PaddedConvNode*>(l.get())) cn->impl().init(init_rng);
    }
    return true;
}

Dataset make_dataset(const RefNet& rn, const float* images, const int* labels, long long N) {
    Dataset ds;
    const std::vector<long long>& in = rn.net.input;
    std::vector<long long> dims{N};
    if (in.size() == 1) dims.insert(dims.end(), {1, 1, in[0]});
    else dims.insert(dims.end(), in.begin(), in.end());
    ds.images = make_tensor(dims);
    copy_in(ds.images, images);
    ds.labels.assign(labels, labels + N);
    ds.num_classes = (size_t)rn.classes;
    return ds;
}

}  // namespace

extern "C" {

void* ref_net_create(int input_rank, const long long* input, const orc_layer_c* descs, int n_layers, float lr,
                     float mom, float wd, unsigned seed, long long batch, char* err, int errlen) {
    auto rn = std::make_unique<RefNet>();
    bool padded = false;
    for (int i = 0; i < n_layers; ++i) padded |= descs[i].kind == 1 && descs[i].pad != 0;
    try {
        std::vector<long long> in(input, input + input_rank);
        if (padded) {
            if (!build_composite(*rn, in, descs, n_layers, seed)) throw SpecError("composite: unsupported layer");
        } else {
            NetworkSpec spec;
            spec.input = in;
            for (int i = 0; i < n_layers; ++i) {
                const orc_layer_c& d = descs[i];
                switch (d.kind) {
                    case 0: spec.layers.push_back(LayerDesc::dense(d.in, d.out)); break;
                    case 1: spec.layers.push_back(LayerDesc::conv(d.k, d.kh, d.kw)); break;
                    case 2: spec.layers.push_back(LayerDesc::maxpool()); break;
                    case 3: spec.layers.push_back(LayerDesc::sigmoid()); break;
                    case 4: spec.layers.push_back(LayerDesc::relu()); break;
                    case 5: spec.layers.push_back(LayerDesc::softmax()); break;
                    case 8: spec.layers.push_back(LayerDesc::flatten()); break;
                    default: throw SpecError("unsupported layer kind");
                }
            }
            spec.seed = seed;
            spec.batch_size = (std::size_t)batch;
            rn->net = build_network(spec);
            long long last = 0;
            for (int i = 0; i < n_layers; ++i)
                if (descs[i].kind == 0) last = descs[i].out;
            rn->classes = last;
        }
        rn->net.opt.lr = lr;
        rn->net.opt.momentum = mom;
        rn->net.opt.weight_decay = wd;
        rn->net.batch_size = (std::size_t)batch;
    } catch (const std::exception& e) {
        if (err && errlen > 0) {
            std::strncpy(err, e.what(), (size_t)errlen - 1);
            err[errlen - 1] = 0;
        }
        return nullptr;
    }
    return rn.release();
}

void ref_net_destroy(void* h) { delete static_cast<RefNet*>(h); }

int ref_net_num_params(void* h) { return (int)static_cast<RefNet*>(h)->net.trainable().size(); }

long long ref_net_param_size(void* h, int idx) {
    return (long long)static_cast<RefNet*>(h)->net.trainable()[idx].value->size();
}

// which: 0 value, 1 grad, 2 velocity, 3 acc (adagrad / adadelta) or m (adam), 4 acc_update or v
// (OptimizerState slot keyed by the parameter's storage, optim.hpp:23-34)
void ref_net_get(void* h, int idx, int which, float* out) {
    RefNet& rn = *static_cast<RefNet*>(h);
    ParamRef p = rn.net.trainable()[idx];
    if (which == 0) return copy_out(*p.value, out);
    if (which == 1) return copy_out(*p.grad, out);
    auto it = rn.net.opt.slots.find(p.value->data());
    if (it == rn.net.opt.slots.end() || !it->second.ready) {
        std::memset(out, 0, p.value->size() * sizeof(float));
        return;
    }
    const OptimizerState::Slot& sl = it->second;
    const bool adam = rn.net.opt.kind == OptimizerKind::Adam;
    copy_out(which == 2 ? sl.velocity : which == 3 ? (adam ? sl.m : sl.acc) : (adam ? sl.v : sl.acc_update), out);
}

void ref_net_set_optimizer(void* h, int kind) { static_cast<RefNet*>(h)->net.opt.kind = (OptimizerKind)kind; }

void ref_net_set(void* h, int idx, int which, const float* in) {
    RefNet& rn = *static_cast<RefNet*>(h);
    ParamRef p = rn.net.trainable()[idx];
    if (which == 0) copy_in(*p.value, in);
    if (which == 1) copy_in(*p.grad, in);
    if (which == 2) copy_in(rn.net.opt.slot_for(*p.value).velocity, in);
}

// the first half of train_minibatch (network.hpp:464-467): gradients left in place
double ref_net_forward_backward(void* h, const float* x, const int* labels, long long B, float* probs_out) {
    RefNet& rn = *static_cast<RefNet*>(h);
    Tensor xt = make_batch(x, B, rn.net.input);
    Tensor y = one_hot(labels, B, rn.classes);
    Tensor pred = net_forward(rn.net, xt, true);
    if (probs_out) copy_out(pred, probs_out);
    LossGrad lg = softmax_cross_entropy(pred, y);
    Tensor g = lg.dlogits;
    for (auto it = rn.net.layers.rbegin(); it != rn.net.layers.rend(); ++it) g = (*it)->backward(g);
    return lg.loss;
}

// the second half (network.hpp:468-470)
void ref_net_apply(void* h) {
    RefNet& rn = *static_cast<RefNet*>(h);
    if (rn.net.opt.lr != 0.0f)
        for (ParamRef p : rn.net.trainable()) optimizer_step(rn.net.opt, *p.value, *p.grad);
    rn.net.zero_grad();
}

// the whole reference step
double ref_net_train_minibatch(void* h, const float* x, const int* labels, long long B) {
    RefNet& rn = *static_cast<RefNet*>(h);
    Tensor xt = make_batch(x, B, rn.net.input);
    Tensor y = one_hot(labels, B, rn.classes);
    return train_minibatch(rn.net, xt, y);
}

// same, with the batch tensors already built (so a timing loop measures train_minibatch only)
void* ref_make_batch(void* h, const float* x, const int* labels, long long B) {
    RefNet& rn = *static_cast<RefNet*>(h);
    auto* pair = new std::pair<Tensor, Tensor>(make_batch(x, B, rn.net.input), one_hot(labels, B, rn.classes));
    return pair;
}
void ref_free_batch(void* b) { delete static_cast<std::pair<Tensor, Tensor>*>(b); }
double ref_net_train_prepared(void* h, void* batch) {
    auto* pair = static_cast<std::pair<Tensor, Tensor>*>(batch);
    return train_minibatch(static_cast<RefNet*>(h)->net, pair->first, pair->second);
}

// BatchIterator::order() after construction (epoch 0) and `epoch` reshuffles (data.hpp:224-238)
void ref_batch_order(long long N, unsigned seed, int epoch, long long* out) {
    Dataset ds;
    ds.images = make_tensor({N, 1, 1, 1});
    ds.labels.assign((size_t)N, 0);
    BatchIterator it(ds, 1, seed);
    for (int e = 1; e <= epoch; ++e) it.reshuffle(seed + (unsigned)e);
    for (size_t i = 0; i < it.order().size(); ++i) out[i] = (long long)it.order()[i];
}

// the reference's own fit (network.hpp:488-511) with the net's batch size / seed overridden
void ref_net_fit(void* h, const float* images, const int* labels, long long N, long long batch, unsigned seed,
                 int epochs, double* loss_out, double* acc_out) {
    RefNet& rn = *static_cast<RefNet*>(h);
    rn.net.batch_size = (size_t)batch;
    rn.net.seed = seed;
    Dataset ds = make_dataset(rn, images, labels, N);
    TrainReport rep = fit(rn.net, ds, (size_t)epochs);
    for (int e = 0; e < epochs; ++e) {
        loss_out[e] = rep.epochs[(size_t)e].loss;
        acc_out[e] = rep.epochs[(size_t)e].accuracy;
    }
}

double ref_net_evaluate(void* h, const float* images, const int* labels, long long N, long long batch) {
    RefNet& rn = *static_cast<RefNet*>(h);
    rn.net.batch_size = (size_t)batch;
    return evaluate(rn.net, make_dataset(rn, images, labels, N));
}

// the reference's own checkpoint I/O (network.hpp:552-607); returns 0 or the error text length
int ref_save_network(void* h, const char* path, char* err, int errlen) {
    try {
        save_network(static_cast<RefNet*>(h)->net, path);
    } catch (const std::exception& e) {
        std::strncpy(err, e.what(), (size_t)errlen - 1);
        err[errlen - 1] = 0;
        return 1;
    }
    return 0;
}
int ref_load_network(void* h, const char* path, char* err, int errlen) {
    try {
        load_network(static_cast<RefNet*>(h)->net, path);
    } catch (const std::exception& e) {
        std::strncpy(err, e.what(), (size_t)errlen - 1);
        err[errlen - 1] = 0;
        return 1;
    }
    return 0;
}

// the reference's dbn_pretrain (energy.hpp:208-240) over a stack of L binary RBMs, layer l being
// hid[l] x vis[l]; W/bv/bh hold every layer's parameters back to back (in: initial, out: trained);
// recon_out gets [layer][epoch]. Returns 0 or 1 with the exception text in err.
int ref_dbn_pretrain(int L, const long long* vis, const long long* hid, float* W, float* bv, float* bh,
                     const float* data, long long N, int epochs, float lr, long long batch, unsigned seed,
                     double* recon_out, char* err, int errlen) {
    try {
        std::vector<Rbm> stack;
        std::vector<long long> dims;
        size_t ow = 0, ov = 0, oh = 0;
        for (int l = 0; l < L; ++l) {
            dims = {vis[l], hid[l]};
            stack.emplace_back((size_t)hid[l], (size_t)vis[l]);
            copy_in(stack.back().w, W + ow);
            copy_in(stack.back().bv, bv + ov);
            copy_in(stack.back().bh, bh + oh);
            ow += (size_t)(vis[l] * hid[l]);
            ov += (size_t)vis[l];
            oh += (size_t)hid[l];
        }
        Tensor x = make_batch(data, N, {vis[0]});
        std::mt19937 rng(seed);
        DbnReport rep = dbn_pretrain(stack, x, (size_t)epochs, lr, (size_t)batch, rng);
        ow = ov = oh = 0;
        for (int l = 0; l < L; ++l) {
            copy_out(stack[l].w, W + ow);
            copy_out(stack[l].bv, bv + ov);
            copy_out(stack[l].bh, bh + oh);
            ow += (size_t)(vis[l] * hid[l]);
            ov += (size_t)vis[l];
            oh += (size_t)hid[l];
            for (int e = 0; e < epochs; ++e) recon_out[l * epochs + e] = rep.recon[(size_t)l][(size_t)e];
        }
    } catch (const std::exception& e) {
        std::strncpy(err, e.what(), (size_t)errlen - 1);
        err[errlen - 1] = 0;
        return 1;
    }
    return 0;
}

void ref_net_forward(void* h, const float* x, long long B, float* probs, int* argmax) {
    RefNet& rn = *static_cast<RefNet*>(h);
    Tensor pred = forward_batch(rn.net, make_batch(x, B, rn.net.input));
    if (probs) copy_out(pred, probs);
    if (argmax)
        for (long long r = 0; r < B; ++r) argmax[r] = (int)detail::argmax_row(pred, (std::size_t)r);
}

// cd_k_update (energy.hpp:131) with its own std::mt19937(rng_seed)
double ref_cd_k(long long H, long long V, float* W, float* bv, float* bh, const float* v0, long long B, int k, float lr,
                unsigned rng_seed) {
    Rbm rbm((std::size_t)H, (std::size_t)V);
    copy_in(rbm.w, W);
    copy_in(rbm.bv, bv);
    copy_in(rbm.bh, bh);
    Tensor v = make_batch(v0, B, {V});
    std::mt19937 rng(rng_seed);
    const double recon = cd_k_update(rbm, v, k, lr, rng);
    copy_out(rbm.w, W);
    copy_out(rbm.bv, bv);
    copy_out(rbm.bh, bh);
    return recon;
}

// persistent RBM for the CPU baseline timing loop
struct RefRbm {
    Rbm rbm;
    Tensor v;
    std::mt19937 rng;
};
void* ref_rbm_create(long long H, long long V, unsigned init_seed, const float* v0, long long B, unsigned rng_seed) {
    auto* r = new RefRbm{Rbm((std::size_t)H, (std::size_t)V), make_batch(v0, B, {V}), std::mt19937(rng_seed)};
    std::mt19937 init(init_seed);
    r->rbm.init(init);
    return r;
}
double ref_rbm_step(void* h, float lr) {
    RefRbm* r = static_cast<RefRbm*>(h);
    return cd_k_update(r->rbm, r->v, 1, lr, r->rng);
}
void ref_rbm_destroy(void* h) { delete static_cast<RefRbm*>(h); }

// crbm_cd_update (energy.hpp:333) with its own std::mt19937(rng_seed); kernels (k,c,kh,kw), bv (c), bh (k)
static ConvShape crbm_shape(long long C, long long Hh, long long Ww, long long K, long long KH, long long KW) {
    ConvShape s;
    s.c_in = (std::size_t)C;
    s.h = (std::size_t)Hh;
    s.w = (std::size_t)Ww;
    s.k = (std::size_t)K;
    s.kh = (std::size_t)KH;
    s.kw = (std::size_t)KW;
    return s;
}
double ref_crbm_cd(long long C, long long Hh, long long Ww, long long K, long long KH, long long KW, float* ker,
                   float* bv, float* bh, const float* v0, long long B, float lr, unsigned rng_seed) {
    Crbm m(crbm_shape(C, Hh, Ww, K, KH, KW));
    copy_in(m.kernels, ker);
    copy_in(m.bv, bv);
    copy_in(m.bh, bh);
    Tensor v = make_batch(v0, B, {C, Hh, Ww});
    std::mt19937 rng(rng_seed);
    const double recon = crbm_cd_update(m, v, lr, rng);
    copy_out(m.kernels, ker);
    copy_out(m.bv, bv);
    copy_out(m.bh, bh);
    return recon;
}
void ref_crbm_init(long long C, long long Hh, long long Ww, long long K, long long KH, long long KW, unsigned seed,
                   float* ker) {
    Crbm m(crbm_shape(C, Hh, Ww, K, KH, KW));
    std::mt19937 rng(seed);
    m.init(rng);
    copy_out(m.kernels, ker);
}
// persistent CRBM for the CPU baseline timing loop
struct RefCrbm {
    Crbm m;
    Tensor v;
    std::mt19937 rng;
};
void* ref_crbm_create(long long C, long long Hh, long long Ww, long long K, long long KH, long long KW,
                      unsigned init_seed, const float* v0, long long B, unsigned rng_seed) {
    auto* r = new RefCrbm{Crbm(crbm_shape(C, Hh, Ww, K, KH, KW)), make_batch(v0, B, {C, Hh, Ww}), std::mt19937(rng_seed)};
    std::mt19937 init(init_seed);
    r->m.init(init);
    return r;
}
double ref_crbm_step(void* h, float lr) {
    RefCrbm* r = static_cast<RefCrbm*>(h);
    return crbm_cd_update(r->m, r->v, lr, r->rng);
}
void ref_crbm_destroy(void* h) { delete static_cast<RefCrbm*>(h); }

void ref_rbm_init(long long H, long long V, unsigned seed, float* W) {
    Rbm rbm((std::size_t)H, (std::size_t)V);
    std::mt19937 rng(seed);
    rbm.init(rng);
    copy_out(rbm.w, W);
}

void ref_gemm(int ta, int tb, const float* A, const float* Bm, float* C, long long M, long long N, long long K) {
    Tensor a = ta ? make_tensor({K, M}) : make_tensor({M, K});
    Tensor b = tb ? make_tensor({N, K}) : make_tensor({K, N});
    copy_in(a, A);
    copy_in(b, Bm);
    copy_out(gemm(a, b, {.transpose_a = ta != 0, .transpose_b = tb != 0}), C);
}

void ref_sgd_momentum_step(float* p, float* v, const float* g, long long n, float lr, float mom, float wd) {
    OptimizerState st;
    st.lr = lr;
    st.momentum = mom;
    st.weight_decay = wd;
    Tensor pt = make_tensor({n}), gt = make_tensor({n});
    copy_in(pt, p);
    copy_in(gt, g);
    copy_in(st.slot_for(pt).velocity, v);
    sgd_momentum_step(st, pt, gt);
    copy_out(pt, p);
    copy_out(st.slot_for(pt).velocity, v);
}

// ----- the reference's op-level layer API (layers.hpp / network.hpp), for the b2n_op_* parity tests -----
void ref_conv_forward(long long n, long long c, long long h, long long w, long long k, long long kh, long long kw,
                      long long pad, const float* x, const float* ker, const float* bias, float* y) {
    ConvShape s;
    s.n = n, s.c_in = c, s.h = h, s.w = w, s.k = k, s.kh = kh, s.kw = kw, s.pad = pad;
    ConvLayer L(s);
    copy_in(L.kernels, ker);
    copy_in(L.b, bias);
    Tensor xt = make_tensor({n, c, h, w});
    copy_in(xt, x);
    copy_out(conv_forward(L, xt), y);
}
// dx = conv_backward(layer, x, dy); gk / gb accumulate from their incoming values
int ref_conv_backward(long long n, long long c, long long h, long long w, long long k, long long kh, long long kw,
                      long long pad, const float* x, const float* ker, const float* dy, float* gk, float* gb, float* dx,
                      char* err, int errlen) {
    try {
        ConvShape s;
        s.n = n, s.c_in = c, s.h = h, s.w = w, s.k = k, s.kh = kh, s.kw = kw, s.pad = pad;
        ConvLayer L(s);
        copy_in(L.kernels, ker);
        copy_in(L.gk, gk);
        copy_in(L.gb, gb);
        const long long oh = h + 2 * pad - kh + 1, ow = w + 2 * pad - kw + 1;
        Tensor xt = make_tensor({n, c, h, w}), dyt = make_tensor({n, k, oh, ow});
        copy_in(xt, x);
        copy_in(dyt, dy);
        copy_out(conv_backward(L, xt, dyt), dx);
        copy_out(L.gk, gk);
        copy_out(L.gb, gb);
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(err, (size_t)errlen, "%s", e.what());
        return 1;
    }
}
void ref_pool_forward(int mode, long long maps, long long h, long long w, const float* x, float* y, float* argmax) {
    Tensor xt = make_tensor({maps, h, w});
    copy_in(xt, x);
    PoolResult r = pool_forward(mode ? PoolMode::Avg : PoolMode::Max, xt);
    copy_out(r.y, y);
    if (!mode) copy_out(r.argmax, argmax);
}
void ref_pool_backward(int mode, long long maps, long long oh, long long ow, const float* dy, const float* argmax,
                       float* dx) {
    Tensor dyt = make_tensor({maps, oh, ow}), at = make_tensor({maps, oh, ow});
    copy_in(dyt, dy);
    if (!mode) copy_in(at, argmax);
    copy_out(pool_backward(mode ? PoolMode::Avg : PoolMode::Max, dyt, at), dx);
}
void ref_softmax(long long rows, long long cols, const float* x, float* y) {
    Tensor xt = make_tensor({rows, cols});
    copy_in(xt, x);
    copy_out(softmax(xt), y);
}
int ref_softmax_cross_entropy(long long rows, long long cols, const float* pred, const float* labels, float* dlogits,
                              double* loss, char* err, int errlen) {
    try {
        Tensor p = make_tensor({rows, cols}), l = make_tensor({rows, cols});
        copy_in(p, pred);
        copy_in(l, labels);
        LossGrad g = softmax_cross_entropy(p, l);
        copy_out(g.dlogits, dlogits);
        *loss = g.loss;
        return 0;
    } catch (const std::exception& e) {
        std::snprintf(err, (size_t)errlen, "%s", e.what());
        return 1;
    }
}
void ref_activation_apply(int kind, long long n, const float* x, float* y) {
    Tensor xt = make_tensor({n});
    copy_in(xt, x);
    copy_out(activation_apply(kind ? Activation::Relu : Activation::Sigmoid, xt), y);
}
void ref_activation_gradient(int kind, long long n, const float* y, const float* dy, float* dx) {
    Tensor yt = make_tensor({n}), gt = make_tensor({n});
    copy_in(yt, y);
    copy_in(gt, dy);
    copy_out(activation_gradient(kind ? Activation::Relu : Activation::Sigmoid, yt, gt), dx);
}

void ref_set_threads(int n) { set_thread_count(n); }
int ref_thread_count(void) { return thread_count(); }

}  // extern "C"
