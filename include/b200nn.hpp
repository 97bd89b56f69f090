// b200nn.hpp -- header-only C++ host API over the C ABI (b200nn.h), mirroring the reference's
// hot-path API (fastnn, /root/reference/proj/include/fastnn) name for name:
//
//   fastnn                                   b200nn
//   LayerDesc / NetworkSpec (network.hpp:194-234)   LayerDesc / NetworkSpec (+ conv pad)
//   build_network (network.hpp:284)          build_network          -> device-resident Network
//   train_minibatch (network.hpp:463)        train_minibatch        -> loss, params updated in HBM
//   forward_batch / evaluate (:402, :474)    forward_batch / evaluate
//   Rbm / cd_k_update (energy.hpp:16, :131)  Rbm / cd_k_update      (rng's Bernoulli stream drawn on the GPU)
//   Error, ShapeError, ... (config.hpp:11-57) the same exception types, thrown from C ABI statuses
//
// Tensors: any type with fastnn::Tensor's accessors (rank(), dim(i), rows_total(), last_dim(),
// row_ptr(r)) -- pass fastnn::Tensor itself for a drop-in swap; rows are packed (lane padding
// stripped, tensor.hpp:16-18) before the host->device copy.
#pragma once
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <random>
#include <stdexcept>
#include <type_traits>
#include <cstdint>
#include <string>
#include <vector>

#include "b200nn.h"

namespace b200nn {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ShapeError : Error {
    using Error::Error;
};
struct ParamError : Error {
    using Error::Error;
};
struct LabelError : Error {
    using Error::Error;
};
struct SpecError : Error {
    using Error::Error;
};
struct BoundsError : Error {
    using Error::Error;
};
struct CudaError : Error {
    using Error::Error;
};
struct NcclError : Error {
    using Error::Error;
};
struct FormatError : Error {
    using Error::Error;
};
struct LengthError : Error {
    using Error::Error;
};
struct DataMissingError : Error {
    using Error::Error;
};
struct ConsistencyError : Error {
    using Error::Error;
};
struct DataError : Error {
    using Error::Error;
};

inline void check(int status) {
    if (status == B2N_OK) return;
    const std::string msg = b2n_last_error();
    switch (status) {
        case B2N_ESHAPE: throw ShapeError(msg);
        case B2N_EPARAM: throw ParamError(msg);
        case B2N_ELABEL: throw LabelError(msg);
        case B2N_ESPEC: throw SpecError(msg);
        case B2N_EBOUNDS: throw BoundsError(msg);
        case B2N_ECUDA: throw CudaError(msg);
        case B2N_ENCCL: throw NcclError(msg);
        case B2N_EFORMAT: throw FormatError(msg);
        case B2N_ELENGTH: throw LengthError(msg);
        case B2N_EIO: throw DataMissingError(msg);
        case B2N_ECONSISTENCY: throw ConsistencyError(msg);
        case B2N_EDATA: throw DataError(msg);
        default: throw Error(msg);
    }
}

struct LayerDesc {
    enum class Kind { Dense, Conv, MaxPool, Sigmoid, Relu, Softmax, Dropout, BatchNorm, Flatten };
    Kind kind = Kind::Dense;
    long long in = 0, out = 0;
    long long k = 0, kh = 0, kw = 0, pad = 0;
    float p = 0.0f;
    static LayerDesc dense(long long in, long long out) { return {Kind::Dense, in, out}; }
    static LayerDesc conv(long long k, long long kh, long long kw, long long pad = 0) {
        LayerDesc d;
        d.kind = Kind::Conv;
        d.k = k, d.kh = kh, d.kw = kw, d.pad = pad;
        return d;
    }
    static LayerDesc maxpool() { return LayerDesc{Kind::MaxPool}; }
    static LayerDesc sigmoid() { return LayerDesc{Kind::Sigmoid}; }
    static LayerDesc relu() { return LayerDesc{Kind::Relu}; }
    static LayerDesc softmax() { return LayerDesc{Kind::Softmax}; }
    static LayerDesc flatten() { return LayerDesc{Kind::Flatten}; }
};

struct NetworkSpec {
    std::vector<long long> input;
    std::vector<LayerDesc> layers;
    int optimizer = 0;  // SgdMomentum
    float lr = 0.1f, momentum = 0.9f, weight_decay = 0.0f;
    std::size_t batch_size = 100;
    unsigned seed = 42;
};

namespace detail {
template <class T>
std::vector<float> pack_rows(const T& t) {  // logical elements, lane padding stripped
    const std::size_t rows = t.rows_total(), n = t.last_dim();
    std::vector<float> out(rows * n);
    for (std::size_t r = 0; r < rows; ++r) std::memcpy(out.data() + r * n, t.row_ptr(r), n * sizeof(float));
    return out;
}
}  // namespace detail

class Network {
  public:
    Network(const NetworkSpec& spec, int device = 0, int precision = B2N_TF32X3) {
        std::vector<b2n_layer_desc> ld;
        for (const LayerDesc& d : spec.layers)
            ld.push_back({(int)d.kind, d.in, d.out, d.k, d.kh, d.kw, d.pad, d.p});
        b2n_network_spec s{};
        s.input_rank = (int)spec.input.size();
        for (std::size_t i = 0; i < spec.input.size() && i < 3; ++i) s.input[i] = spec.input[i];
        s.layers = ld.data();
        s.n_layers = (int)ld.size();
        s.optimizer = spec.optimizer;
        s.lr = spec.lr, s.momentum = spec.momentum, s.weight_decay = spec.weight_decay;
        s.batch_size = (long long)spec.batch_size;
        s.seed = spec.seed;
        b2n_net* h = nullptr;
        check(b2n_build_network(&s, device, precision, &h));
        h_.reset(h);
        input_ = spec.input;
        batch_size = spec.batch_size;
        for (const LayerDesc& d : spec.layers)
            if (d.kind == LayerDesc::Kind::Dense) classes_ = d.out;
    }
    b2n_net* handle() const { return h_.get(); }
    std::size_t batch_size = 100;
    long long classes() const { return classes_; }
    long long input_size() const {
        long long n = 1;
        for (long long e : input_) n *= e;
        return n;
    }

    // Network::trainable() (network.hpp:244-249): w then b per layer
    int num_params() const {
        int n = 0;
        check(b2n_net_num_params(h_.get(), &n));
        return n;
    }
    std::vector<long long> param_dims(int idx) const {
        int rank = 0;
        long long dims[4];
        check(b2n_net_param_shape(h_.get(), idx, &rank, dims));
        return std::vector<long long>(dims, dims + rank);
    }
    std::vector<float> param(int idx, int which = B2N_VALUE) const {
        long long n = 1;
        for (long long d : param_dims(idx)) n *= d;
        std::vector<float> out((std::size_t)n);
        check(b2n_net_get_param(h_.get(), idx, which, out.data()));
        return out;
    }
    void set_param(int idx, const std::vector<float>& v, int which = B2N_VALUE) {
        check(b2n_net_set_param(h_.get(), idx, which, v.data()));
    }

  private:
    struct Del {
        void operator()(b2n_net* n) const { b2n_net_destroy(n); }
    };
    std::unique_ptr<b2n_net, Del> h_;
    std::vector<long long> input_;
    long long classes_ = 0;
};

inline Network build_network(const NetworkSpec& spec, int device = 0) { return Network(spec, device); }

// train_minibatch (network.hpp:463-472): x (batch, ...) and y one-hot (batch, classes)
template <class T>
double train_minibatch(Network& net, const T& x, const T& y) {
    if (x.rank() < 2 || (long long)(x.rows_total() * x.last_dim() / x.dim(0)) != net.input_size())
        throw ShapeError("network input expects (batch, " + std::to_string(net.input_size()) + ")");
    if (y.rank() != 2 || y.dim(0) != x.dim(0) || (long long)y.dim(1) != net.classes())
        throw ShapeError("softmax_cross_entropy: predictions and labels must both be (batch, classes)");
    const std::vector<float> xs = detail::pack_rows(x), ys = detail::pack_rows(y);
    double loss = 0.0;
    check(b2n_train_minibatch(net.handle(), xs.data(), ys.data(), (long long)x.dim(0), &loss));
    return loss;
}

// forward_batch (network.hpp:402): probabilities, plus argmax_row ids (first maximum wins)
template <class T>
std::vector<float> forward_batch(Network& net, const T& x, std::vector<int>* argmax = nullptr) {
    const std::vector<float> xs = detail::pack_rows(x);
    const long long B = (long long)x.dim(0);
    std::vector<float> probs((std::size_t)(B * net.classes()));
    std::vector<int> am((std::size_t)B);
    check(b2n_forward_batch(net.handle(), xs.data(), B, probs.data(), am.data()));
    if (argmax) *argmax = std::move(am);
    return probs;
}

// The reference's training loop -- one train_minibatch per batch -- over `steps` consecutive host
// batches of packed samples (rows [i*batch, (i+1)*batch) of images / labels), each step's
// host->device copy overlapped with the previous step. Returns every step's loss.
inline std::vector<double> train_stream(Network& net, const float* images, const int* labels, std::size_t steps,
                                        std::size_t batch) {
    std::vector<double> loss(steps);
    check(b2n_net_train_stream(net.handle(), images, labels, (long long)steps, (long long)batch, loss.data()));
    return loss;
}

// evaluate (network.hpp:474-484) over a dataset of `n` packed samples and int labels, held in
// device memory for the pass
inline double evaluate(Network& net, const float* images, const int* labels, std::size_t n) {
    double acc = 0.0;
    check(b2n_net_evaluate(net.handle(), images, labels, (long long)n, &acc));
    return acc;
}

// EpochStats / TrainReport / fit (network.hpp:255-265, :488-511): BatchIterator order from the
// net's seed, dataset resident in device memory, batches gathered on the device
struct EpochStats {
    double loss = 0.0, accuracy = 0.0, seconds = 0.0;
};
struct TrainReport {
    std::vector<EpochStats> epochs;
    double test_accuracy = -1.0;
    std::size_t total_batches = 0;
};
inline TrainReport fit(Network& net, const float* images, const int* labels, std::size_t n, std::size_t epochs) {
    std::vector<double> loss(epochs), acc(epochs), sec(epochs);
    check(b2n_net_fit(net.handle(), images, labels, (long long)n, (int)epochs, loss.data(), acc.data(), sec.data()));
    TrainReport r;
    for (std::size_t e = 0; e < epochs; ++e) r.epochs.push_back({loss[e], acc[e], sec[e]});
    r.total_batches = epochs * ((n + net.batch_size - 1) / net.batch_size);
    return r;
}

// save_network / load_network (network.hpp:552-607): the reference's FNN1 file; with_state adds
// the `<path>.state` sidecar (velocities, hyper-parameters) for an exact resume
inline void save_network(Network& net, const std::string& path, bool with_state = false) {
    check(b2n_save_network(net.handle(), path.c_str(), with_state ? 1 : 0));
}
inline void load_network(Network& net, const std::string& path, bool with_state = false) {
    check(b2n_load_network(net.handle(), path.c_str(), with_state ? 1 : 0));
}

// Rbm (energy.hpp:16-32), binary units
class Rbm {
  public:
    Rbm(std::size_t hidden, std::size_t visible, int device = 0, int precision = B2N_TF32X3)
        : hidden_(hidden), visible_(visible) {
        b2n_rbm* h = nullptr;
        check(b2n_rbm_create((long long)hidden, (long long)visible, device, precision, &h));
        h_.reset(h);
    }
    // Rbm::init (energy.hpp:31): glorot_fill(w, visible, hidden) drawn from the caller's generator,
    // exactly as the reference consumes it (uniform_real_distribution<float>, layers.hpp:40-48)
    void init(std::mt19937& rng) {
        const float limit = std::sqrt(6.0f / static_cast<float>(visible_ + hidden_));
        std::vector<float> w(hidden_ * visible_), bv(visible_, 0.0f), bh(hidden_, 0.0f);
        for (float& x : w) {
            const float u = std::generate_canonical<float, std::numeric_limits<float>::digits>(rng);
            x = std::fma(u, limit - (-limit), -limit);
        }
        set(w, bv, bh);
    }
    void init_seed(unsigned seed) { check(b2n_rbm_init(h_.get(), seed)); }
    void set(const std::vector<float>& w, const std::vector<float>& bv, const std::vector<float>& bh) {
        check(b2n_rbm_set(h_.get(), w.data(), bv.data(), bh.data()));
    }
    void get(std::vector<float>& w, std::vector<float>& bv, std::vector<float>& bh) const {
        w.resize(hidden_ * visible_);
        bv.resize(visible_);
        bh.resize(hidden_);
        check(b2n_rbm_get(h_.get(), w.data(), bv.data(), bh.data()));
    }
    std::size_t hidden_units() const { return hidden_; }
    std::size_t visible_units() const { return visible_; }
    b2n_rbm* handle() const { return h_.get(); }

  private:
    struct Del {
        void operator()(b2n_rbm* r) const { b2n_rbm_destroy(r); }
    };
    std::unique_ptr<b2n_rbm, Del> h_;
    std::size_t hidden_, visible_;
};

namespace detail {
#if defined(__GLIBCXX__)
// The caller's std::mt19937 as the C ABI's 625-word state (libstdc++: _M_x[624], _M_p -- the same
// numbers `os << rng` prints). The Bernoulli draws then run on the device from this state
// (b2n_mt19937_draw) and the advanced state is written back, so `rng` ends exactly where the
// reference's cd_k_update would have left it.
constexpr bool kDeviceDraws = true;
struct MtRaw {
    std::uint_fast32_t x[624];
    std::size_t p;
};
static_assert(sizeof(std::mt19937) == sizeof(MtRaw) && std::is_trivially_copyable<std::mt19937>::value,
              "libstdc++ mersenne_twister_engine layout");
inline void mt_export(const std::mt19937& g, unsigned s[625]) {
    MtRaw r;
    std::memcpy(&r, &g, sizeof r);
    for (int i = 0; i < 624; ++i) s[i] = (unsigned)r.x[i];
    s[624] = (unsigned)r.p;
}
inline void mt_import(std::mt19937& g, const unsigned s[625]) {
    MtRaw r;
    for (int i = 0; i < 624; ++i) r.x[i] = s[i];
    r.p = s[624];
    std::memcpy(static_cast<void*>(&g), &r, sizeof r);
}
#else
constexpr bool kDeviceDraws = false;  // another standard library: draw on the host and supply them
inline void mt_export(const std::mt19937&, unsigned*) {}
inline void mt_import(std::mt19937&, const unsigned*) {}
#endif
inline std::vector<double> host_draws(std::mt19937& rng, std::size_t n) {
    std::vector<double> u(n);
    for (double& d : u) d = std::generate_canonical<double, 53>(rng);
    return u;
}
}  // namespace detail

// cd_k_update (energy.hpp:131-171). The reference draws its Bernoulli samples from `rng`; here the
// same stream (generate_canonical<double,53>, what std::bernoulli_distribution consumes) is
// generated on the GPU from rng's state and rng is advanced past it, so sampling stays bit-exact.
template <class T>
double cd_k_update(Rbm& rbm, const T& v0, int k, float lr, std::mt19937& rng) {
    if (k < 1) throw ParamError("cd_k_update: k must be >= 1, got " + std::to_string(k));
    if (v0.rank() != 2) throw ShapeError("cd_k_update: expected a rank-2 tensor, got rank " + std::to_string(v0.rank()));
    if (v0.dim(1) != rbm.visible_units()) throw ShapeError("cd_k_update: visible extent mismatch");
    const std::vector<float> vs = detail::pack_rows(v0);
    const std::size_t B = v0.dim(0);
    double recon = 0.0;
    if (detail::kDeviceDraws) {
        unsigned st[625];
        detail::mt_export(rng, st);
        check(b2n_rbm_set_rng(rbm.handle(), st));
        check(b2n_cd_k_update(rbm.handle(), vs.data(), (long long)B, k, lr, nullptr, (long long)B, &recon));
        check(b2n_rbm_get_rng(rbm.handle(), st));
        detail::mt_import(rng, st);
        return recon;
    }
    const std::vector<double> u = detail::host_draws(rng, (std::size_t)k * B * rbm.hidden_units());
    check(b2n_cd_k_update(rbm.handle(), vs.data(), (long long)B, k, lr, u.data(), (long long)B, &recon));
    return recon;
}

// Crbm (energy.hpp:245-262): kernels (k, c_in, kh, kw), bv (c_in), bh (k), binary units. Takes the
// reference's ConvShape-style extents (c_in, h, w, k, kh, kw); same ShapeError for kh > h / kw > w.
class Crbm {
  public:
    Crbm(std::size_t c_in, std::size_t h, std::size_t w, std::size_t k, std::size_t kh, std::size_t kw,
         int device = 0, int precision = B2N_TF32X3)
        : c_(c_in), h_(h), w_(w), k_(k), kh_(kh), kw_(kw) {
        b2n_crbm* p = nullptr;
        check(b2n_crbm_create((int)c_in, (int)h, (int)w, (int)k, (int)kh, (int)kw, device, precision, &p));
        p_.reset(p);
    }
    // Crbm::init (energy.hpp:261): glorot_fill(kernels, c_in*kh*kw, k*kh*kw) from the caller's generator
    void init(std::mt19937& rng) {
        const float limit = std::sqrt(6.0f / static_cast<float>(c_ * kh_ * kw_ + k_ * kh_ * kw_));
        std::vector<float> ker(k_ * c_ * kh_ * kw_), bv(c_, 0.0f), bh(k_, 0.0f);
        for (float& x : ker) {
            const float u = std::generate_canonical<float, std::numeric_limits<float>::digits>(rng);
            x = std::fma(u, limit - (-limit), -limit);
        }
        set(ker, bv, bh);
    }
    void set(const std::vector<float>& kernels, const std::vector<float>& bv, const std::vector<float>& bh) {
        check(b2n_crbm_set(p_.get(), kernels.data(), bv.data(), bh.data()));
    }
    void get(std::vector<float>& kernels, std::vector<float>& bv, std::vector<float>& bh) const {
        kernels.resize(k_ * c_ * kh_ * kw_);
        bv.resize(c_);
        bh.resize(k_);
        check(b2n_crbm_get(p_.get(), kernels.data(), bv.data(), bh.data()));
    }
    std::size_t c_in() const { return c_; }
    std::size_t height() const { return h_; }
    std::size_t width() const { return w_; }
    std::size_t hidden_maps() const { return k_; }
    std::size_t hidden_pixels() const { return k_ * (h_ - kh_ + 1) * (w_ - kw_ + 1); }
    b2n_crbm* handle() const { return p_.get(); }

  private:
    struct Del {
        void operator()(b2n_crbm* r) const { b2n_crbm_destroy(r); }
    };
    std::unique_ptr<b2n_crbm, Del> p_;
    std::size_t c_, h_, w_, k_, kh_, kw_;
};

// crbm_cd_update (energy.hpp:333-376): the reference's Bernoulli draws (unit_sample_inplace over
// the n x k x oh x ow hidden tensor, energy.hpp:53-71) are taken from `rng` on the host in the same
// order and supplied, so sampling stays bit-exact given the same probabilities.
template <class T>
double crbm_cd_update(Crbm& m, const T& v0, float lr, std::mt19937& rng) {
    if (v0.rank() != 4 || v0.dim(1) != m.c_in() || v0.dim(2) != m.height() || v0.dim(3) != m.width())
        throw ShapeError("crbm_cd_update: input does not match the model's visible shape");
    const std::vector<float> vs = detail::pack_rows(v0);
    const std::size_t B = v0.dim(0);
    double recon = 0.0;
    if (detail::kDeviceDraws) {  // the draws generated on the GPU from rng's state (see cd_k_update)
        unsigned st[625];
        detail::mt_export(rng, st);
        check(b2n_crbm_set_rng(m.handle(), st));
        check(b2n_crbm_cd_update(m.handle(), vs.data(), (long long)B, lr, nullptr, (long long)B, &recon));
        check(b2n_crbm_get_rng(m.handle(), st));
        detail::mt_import(rng, st);
        return recon;
    }
    const std::vector<double> u = detail::host_draws(rng, B * m.hidden_pixels());
    check(b2n_crbm_cd_update(m.handle(), vs.data(), (long long)B, lr, u.data(), (long long)B, &recon));
    return recon;
}

// `steps` cd_k_update(rbm, batch_i, 1, lr, rng) calls over consecutive host batches of v0 (rows
// [i*batch, (i+1)*batch), pitch visible): the Bernoulli draws are taken from `rng` in the
// reference's order (step by step, row-major), and each step's copies overlap the previous step.
// Returns every step's reconstruction error.
inline std::vector<double> cd1_stream(Rbm& rbm, const float* v0, std::size_t steps, std::size_t batch, float lr,
                                      std::mt19937& rng) {
    std::vector<double> recon(steps);
    if (detail::kDeviceDraws) {  // each step's draws generated on the GPU ahead of the step
        unsigned st[625];
        detail::mt_export(rng, st);
        check(b2n_rbm_set_rng(rbm.handle(), st));
        check(b2n_rbm_train_stream(rbm.handle(), v0, nullptr, (long long)steps, (long long)batch, lr, recon.data()));
        check(b2n_rbm_get_rng(rbm.handle(), st));
        detail::mt_import(rng, st);
        return recon;
    }
    const std::vector<double> u = detail::host_draws(rng, steps * batch * rbm.hidden_units());
    check(b2n_rbm_train_stream(rbm.handle(), v0, u.data(), (long long)steps, (long long)batch, lr, recon.data()));
    return recon;
}

// dbn_pretrain (energy.hpp:208-240) with the reference's signature: the stack trains on the device
// (data uploaded once, hidden means passed up on the device); `rng` supplies the Bernoulli
// uniforms in the reference's order, drawn on this thread while the GPU runs the previous step.
struct DbnReport {
    std::vector<std::vector<double>> recon;  // [layer][epoch]
};
template <class T>
DbnReport dbn_pretrain(std::vector<Rbm>& stack, const T& data, std::size_t epochs, float lr, std::size_t batch_size,
                       std::mt19937& rng) {
    if (data.rank() != 2) throw ShapeError("dbn_pretrain: data must be (rows, visible)");
    const std::vector<float> xs = detail::pack_rows(data);
    std::vector<b2n_rbm*> hs;
    for (Rbm& r : stack) hs.push_back(r.handle());
    std::vector<double> rec(std::max<std::size_t>(stack.size() * epochs, 1));
    auto fill = [](void* ctx, double* out, long long count) {
        std::mt19937& g = *static_cast<std::mt19937*>(ctx);
        for (long long i = 0; i < count; ++i) out[i] = std::generate_canonical<double, 53>(g);
    };
    if (detail::kDeviceDraws) {  // the draws generated on the GPU from rng's state, rng advanced
        unsigned st[625];
        detail::mt_export(rng, st);
        check(b2n_dbn_pretrain(hs.data(), (int)hs.size(), xs.data(), (long long)data.dim(0), (int)epochs, lr,
                               (long long)batch_size, nullptr, st, rec.data()));
        detail::mt_import(rng, st);
    } else {
        check(b2n_dbn_pretrain(hs.data(), (int)hs.size(), xs.data(), (long long)data.dim(0), (int)epochs, lr,
                               (long long)batch_size, fill, &rng, rec.data()));
    }
    DbnReport r;
    for (std::size_t l = 0; l < stack.size(); ++l)
        r.recon.emplace_back(rec.begin() + (long)(l * epochs), rec.begin() + (long)((l + 1) * epochs));
    return r;
}

}  // namespace b200nn
