// b200nn.cu -- the C ABI (include/b200nn.h): status codes + thread-local messages around the
// device runtime (network.cuh, rbm.cuh, conv.cuh, gemm_tc.cuh). Built by
// paper_1804_04512_b200/build.py into paper_1804_04512_b200/_build/libb200nn.so for sm_100a.
#include <cstdio>
#include <new>

#include "../../include/b200nn.h"
#include "network.cuh"
#include "crbm.cuh"
#include "rbm.cuh"
#include "runtime.cuh"

struct b2n_net {
    b2n::Net impl;
    template <class... A>
    explicit b2n_net(A&&... a) : impl(std::forward<A>(a)...) {}
};
struct b2n_rbm {
    b2n::Rbm impl;
    template <class... A>
    explicit b2n_rbm(A&&... a) : impl(std::forward<A>(a)...) {}
};

struct b2n_crbm {
    b2n::Crbm impl;
    template <class... A>
    explicit b2n_crbm(A&&... a) : impl(std::forward<A>(a)...) {}
};

namespace {
thread_local std::string g_last_error;

template <class F>
int guard(F&& f) {
    try {
        f();
        g_last_error.clear();
        return B2N_OK;
    } catch (const b2n::Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return B2N_EOOM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return B2N_EINTERNAL;
    }
}

#define B2N_REQUIRE(cond, code, msg) \
    do {                             \
        if (!(cond)) throw b2n::Error(code, msg); \
    } while (0)

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }
}  // namespace

namespace b2n {
void set_last_error(const char* msg) { g_last_error = msg; }  // ops.cu's guard
}

extern "C" {

const char* b2n_last_error(void) { return g_last_error.c_str(); }
int b2n_version(void) { return 1; }
int b2n_device_count(int* n) {
    return guard([&] { B2N_CUDA(cudaGetDeviceCount(n)); });
}

// ------------------------------------------------------------------ network
int b2n_build_network(const b2n_network_spec* spec, int device, int precision, b2n_net** out) {
    return guard([&] {
        B2N_REQUIRE(spec && out, B2N_EPARAM, "null argument");
        *out = new b2n_net(*spec, device, precision);
    });
}
int b2n_net_destroy(b2n_net* net) {
    return guard([&] { delete net; });
}
int b2n_net_num_params(b2n_net* net, int* n) {
    return guard([&] { *n = net->impl.num_params(); });
}
int b2n_net_param_shape(b2n_net* net, int idx, int* rank, long long dims[4]) {
    return guard([&] {
        B2N_REQUIRE(idx >= 0 && idx < net->impl.num_params(), B2N_EBOUNDS, "param index out of range");
        const auto& v = net->impl.param(idx);
        *rank = (int)v.dims.size();
        for (size_t i = 0; i < v.dims.size(); ++i) dims[i] = v.dims[i];
    });
}
int b2n_net_get_param(b2n_net* net, int idx, int which, float* host) {
    return guard([&] { net->impl.get_param(idx, which, host); });
}
int b2n_net_set_param(b2n_net* net, int idx, int which, const float* host) {
    return guard([&] { net->impl.set_param(idx, which, host); });
}
int b2n_net_set_hparams(b2n_net* net, float lr, float momentum, float weight_decay) {
    return guard([&] { net->impl.set_hparams(lr, momentum, weight_decay); });
}

int b2n_train_minibatch(b2n_net* net, const float* x, const float* y_onehot, long long batch, double* loss) {
    return guard([&] {
        // one-hot contract of softmax_cross_entropy (network.hpp:423-432) checked on the host
        long long C = 0;
        int rank;
        long long dims[4];
        int np = net->impl.num_params();
        b2n_net_param_shape(net, np - 1, &rank, dims);
        C = dims[0];
        std::vector<int> labels((size_t)batch);
        for (long long r = 0; r < batch; ++r) {
            long long ones = 0, truth = 0;
            for (long long j = 0; j < C; ++j) {
                const float y = y_onehot[r * C + j];
                if (y == 1.0f) {
                    ++ones;
                    truth = j;
                } else if (y != 0.0f) {
                    throw b2n::Error(B2N_ELABEL, "softmax_cross_entropy: labels must be one-hot; row " + std::to_string(r));
                }
            }
            if (ones != 1)
                throw b2n::Error(B2N_ELABEL, "softmax_cross_entropy: labels must be one-hot; row " + std::to_string(r));
            labels[(size_t)r] = (int)truth;
        }
        *loss = net->impl.train(x, labels.data(), batch);
    });
}
int b2n_net_train_stream(b2n_net* net, const float* x, const int* labels, long long steps, long long batch,
                         double* loss_out) {
    return guard([&] { net->impl.train_stream(x, labels, steps, batch, loss_out); });
}
int b2n_train_minibatch_labels(b2n_net* net, const float* x, const int* labels, long long batch, double* loss) {
    return guard([&] { *loss = net->impl.train(x, labels, batch); });
}
int b2n_forward_batch(b2n_net* net, const float* x, long long batch, float* probs, int* argmax) {
    return guard([&] { net->impl.forward(x, batch, probs, argmax); });
}
int b2n_net_forward_backward(b2n_net* net, const float* x, const int* labels, long long batch, long long batch_global,
                             double* loss_share) {
    return guard([&] { *loss_share = net->impl.forward_backward(x, labels, batch, batch_global); });
}
int b2n_net_num_layers(b2n_net* net, long long* n) {
    return guard([&] { *n = net->impl.num_layers(); });
}
int b2n_net_layer_output(b2n_net* net, int layer, long long batch, float* out, unsigned char* codes) {
    return guard([&] { net->impl.layer_output(layer, batch, out, codes); });
}
int b2n_net_apply_update(b2n_net* net) {
    return guard([&] { net->impl.apply_update(); });
}
int b2n_net_grad_buffer(b2n_net* net, float** dev_ptr, long long* n) {
    return guard([&] {
        *dev_ptr = net->impl.grad_buffer();
        *n = net->impl.packed_floats();
    });
}
int b2n_nccl_unique_id(char id_out[128]) {
    return guard([&] {
        ncclUniqueId uid;
        b2n::nccl_check(b2n::nccl().getUniqueId(&uid), "ncclGetUniqueId");
        std::memcpy(id_out, uid.internal, 128);
    });
}
int b2n_net_dp_init(b2n_net* net, const char id[128], int rank, int world) {
    return guard([&] { net->impl.dp_init(id, rank, world); });
}
int b2n_net_stage(b2n_net* net, const float* x, const int* labels, long long batch) {
    return guard([&] { net->impl.stage(x, labels, batch); });
}
int b2n_net_run_staged(b2n_net* net, int steps, long long batch_global) {
    return guard([&] { net->impl.run_staged(steps, batch_global); });
}
int b2n_net_fit(b2n_net* net, const float* images, const int* labels, long long n, int epochs, double* loss_out,
                double* accuracy_out, double* seconds_out) {
    return guard([&] {
        auto st = net->impl.fit(images, labels, n, epochs);
        for (size_t e = 0; e < st.size(); ++e) {
            if (loss_out) loss_out[e] = st[e].loss;
            if (accuracy_out) accuracy_out[e] = st[e].accuracy;
            if (seconds_out) seconds_out[e] = st[e].seconds;
        }
    });
}
int b2n_net_evaluate(b2n_net* net, const float* images, const int* labels, long long n, double* accuracy) {
    return guard([&] { *accuracy = net->impl.evaluate(images, labels, n); });
}
int b2n_save_network(b2n_net* net, const char* path, int with_state) {
    return guard([&] {
        if (!path) throw b2n::Error(B2N_EIO, "save_network: cannot open (null path)");
        net->impl.save(path, with_state != 0);
    });
}
int b2n_load_network(b2n_net* net, const char* path, int with_state) {
    return guard([&] {
        if (!path) throw b2n::Error(B2N_EIO, "load_network: cannot open (null path)");
        net->impl.load(path, with_state != 0);
    });
}
int b2n_dbn_pretrain(b2n_rbm* const* stack, int layers, const float* data, long long n, int epochs, float lr,
                     long long batch, b2n_uniform_fn fill, void* ctx, double* recon_out) {
    return guard([&] {
        if (layers < 1 || !stack) throw b2n::Error(B2N_EPARAM, "dbn_pretrain: empty stack");
        if (batch < 1) throw b2n::Error(B2N_EPARAM, "dbn_pretrain: batch_size must be >= 1");
        if (epochs < 0) throw b2n::Error(B2N_EPARAM, "dbn_pretrain: epochs must be >= 0");
        // fill == null: ctx is the caller's std::mt19937 state (625 words), advanced on the device
        if (!fill && !ctx) throw b2n::Error(B2N_EPARAM, "dbn_pretrain: no uniform source");
        uint32_t* mt = fill ? nullptr : static_cast<uint32_t*>(ctx);
        long long in = stack[0]->impl.visible();
        for (int l = 0; l < layers; ++l) {  // energy.hpp:216-224
            const long long v = stack[l]->impl.visible();
            if (v != in)
                throw b2n::Error(B2N_ESHAPE, "dbn_pretrain: layer " + std::to_string(l) + " expects " + std::to_string(v) +
                                                 " visible units but layer " + std::to_string(l ? l - 1 : 0) +
                                                 (l ? " provides " : "'s input provides ") + std::to_string(in));
            in = stack[l]->impl.hidden();
        }
        if (n < 1) throw b2n::Error(B2N_EDATA, "dbn_pretrain: empty dataset");
        b2n::Rbm& r0 = stack[0]->impl;
        const long long V0 = r0.visible();
        b2n::DevMem cur, next;
        cur.alloc((size_t)(n * r0.ld_visible() * 4));
        B2N_CUDA(cudaMemcpy2DAsync(cur.p, r0.ld_visible() * 4, data, V0 * 4, V0 * 4, n, cudaMemcpyHostToDevice,
                                   r0.stream()));
        B2N_CUDA(cudaStreamSynchronize(r0.stream()));
        for (int l = 0; l < layers; ++l) {
            b2n::Rbm& r = stack[l]->impl;
            if (mt) r.set_rng(mt);
            for (int e = 0; e < epochs; ++e) {
                const double rc = r.train_epoch(cur.as<float>(), n, batch, lr, fill, ctx);
                if (recon_out) recon_out[(size_t)l * epochs + e] = rc;
            }
            if (mt) r.get_rng(mt);
            if (l + 1 < layers) {
                next.alloc((size_t)(n * stack[l + 1]->impl.ld_visible() * 4));
                r.transform_up(cur.as<float>(), n, next.as<float>());
                B2N_CUDA(cudaStreamSynchronize(r.stream()));
                std::swap(cur.p, next.p);  // DevMem is not movable: swap the owned pointers
                std::swap(cur.bytes, next.bytes);
            }
        }
    });
}
int b2n_batch_order(long long n, unsigned seed, int epoch, long long* order_out) {
    return guard([&] {
        if (n < 1) throw b2n::Error(B2N_EPARAM, "batch_iterator: empty dataset");
        std::vector<long long> o;
        b2n::batch_order(o, n, seed, epoch);
        std::copy(o.begin(), o.end(), order_out);
    });
}
int b2n_net_loss(b2n_net* net, double* loss) {
    return guard([&] { *loss = net->impl.loss(); });
}
int b2n_net_stream(b2n_net* net, void** s) {
    return guard([&] { *s = net->impl.stream(); });
}
int b2n_net_kernels_per_step(b2n_net* net, long long batch, int* n) {
    return guard([&] { *n = net->impl.kernels_per_step(batch); });
}

namespace {
void export_stats(const std::vector<b2n::OpStats>& st, int max_ops, double* stats, char* names, int names_len,
                  int* n_ops) {
    *n_ops = (int)st.size();
    std::string joined;
    for (size_t i = 0; i < st.size() && (int)i < max_ops; ++i) {
        stats[i * 4 + 0] = st[i].ms;
        stats[i * 4 + 1] = st[i].flops;
        stats[i * 4 + 2] = st[i].bytes;
        stats[i * 4 + 3] = st[i].kernels;
        joined += st[i].name;
        joined.push_back('\n');
    }
    if (names && names_len > 0) {
        std::strncpy(names, joined.c_str(), (size_t)names_len - 1);
        names[names_len - 1] = 0;
    }
}
}  // namespace

int b2n_net_profile(b2n_net* net, long long batch, int steps, int max_ops, double* stats, char* names, int names_len,
                    int* n_ops) {
    return guard([&] { export_stats(net->impl.profile(batch, steps), max_ops, stats, names, names_len, n_ops); });
}

// ------------------------------------------------------------------ RBM
int b2n_rbm_create(long long hidden, long long visible, int device, int precision, b2n_rbm** out) {
    return guard([&] { *out = new b2n_rbm(hidden, visible, device, precision); });
}
int b2n_rbm_destroy(b2n_rbm* r) {
    return guard([&] { delete r; });
}
int b2n_rbm_init(b2n_rbm* r, unsigned seed) {
    return guard([&] { r->impl.init(seed); });
}
int b2n_rbm_set(b2n_rbm* r, const float* w, const float* bv, const float* bh) {
    return guard([&] { r->impl.set(w, bv, bh); });
}
int b2n_rbm_get(b2n_rbm* r, float* w, float* bv, float* bh) {
    return guard([&] { r->impl.get(w, bv, bh); });
}
int b2n_cd_k_update(b2n_rbm* r, const float* v0, long long batch, int k, float lr, const double* u,
                    long long batch_global, double* recon) {
    return guard([&] { *recon = r->impl.cd_k(v0, batch, k, lr, u, batch_global ? batch_global : batch); });
}
int b2n_rbm_last_states(b2n_rbm* r, float* h0, float* hs, float* v1, float* h1) {
    return guard([&] { r->impl.last_states(h0, hs, v1, h1); });
}
int b2n_rbm_dp_init(b2n_rbm* r, const char id[128], int rank, int world) {
    return guard([&] { r->impl.dp_init(id, rank, world); });
}
int b2n_rbm_stage(b2n_rbm* r, const float* v0, const double* u, long long batch) {
    return guard([&] { r->impl.stage(v0, u, batch, 1); });
}
int b2n_rbm_run_staged(b2n_rbm* r, int steps, float lr, long long batch_global) {
    return guard([&] { r->impl.run_staged(steps, lr, batch_global); });
}
int b2n_rbm_train_stream(b2n_rbm* r, const float* v0, const double* u, long long steps, long long batch, float lr,
                         double* recon_out) {
    return guard([&] { r->impl.train_stream(v0, u, steps, batch, lr, recon_out); });
}
int b2n_rbm_set_rng(b2n_rbm* r, const unsigned state[625]) {
    return guard([&] { r->impl.set_rng(state); });
}
int b2n_rbm_get_rng(b2n_rbm* r, unsigned state[625]) {
    return guard([&] { r->impl.get_rng(state); });
}
int b2n_crbm_set_rng(b2n_crbm* m, const unsigned state[625]) {
    return guard([&] { m->impl.set_rng(state); });
}
int b2n_crbm_get_rng(b2n_crbm* m, unsigned state[625]) {
    return guard([&] { m->impl.get_rng(state); });
}
int b2n_mt19937_draw(int device, unsigned state[625], double* out_host, long long n) {
    return guard([&] {
        B2N_REQUIRE(state && (out_host || n == 0) && n >= 0, B2N_EPARAM, "mt19937_draw: bad arguments");
        B2N_CUDA(cudaSetDevice(device));
        cudaStream_t st;
        B2N_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        try {
            b2n::DevRng g;
            g.load(state, st);
            b2n::DevMem out;
            out.alloc((size_t)std::max<long long>(n, 1) * 8);
            g.draw(out.as<double>(), n, st);
            B2N_CUDA(cudaMemcpyAsync(out_host, out.p, (size_t)n * 8, cudaMemcpyDeviceToHost, st));
            g.store(state, st);
        } catch (...) {
            cudaStreamDestroy(st);
            throw;
        }
        B2N_CUDA(cudaStreamDestroy(st));
    });
}
int b2n_rbm_set_grad_only(b2n_rbm* r, int on) {
    return guard([&] { r->impl.set_grad_only(on != 0); });
}
int b2n_rbm_get_grad(b2n_rbm* r, float* w, float* bv, float* bh) {
    return guard([&] { r->impl.get_grad(w, bv, bh); });
}
int b2n_rbm_set_grad(b2n_rbm* r, const float* w, const float* bv, const float* bh) {
    return guard([&] { r->impl.set_grad(w, bv, bh); });
}
int b2n_rbm_apply_update(b2n_rbm* r, float lr, long long batch_global) {
    return guard([&] { r->impl.apply_update(lr, batch_global); });
}
int b2n_rbm_recon(b2n_rbm* r, double* recon) {
    return guard([&] { *recon = r->impl.recon(); });
}
int b2n_rbm_profile(b2n_rbm* r, int steps, float lr, long long batch_global, int max_ops, double* stats, char* names,
                    int names_len, int* n_ops) {
    return guard([&] { export_stats(r->impl.profile(steps, lr, batch_global), max_ops, stats, names, names_len, n_ops); });
}
int b2n_rbm_kernels_per_step(b2n_rbm* r, int* n) {
    return guard([&] { *n = r->impl.kernels_per_step(); });
}
int b2n_rbm_stream(b2n_rbm* r, void** s) {
    return guard([&] { *s = r->impl.stream(); });
}

// ------------------------------------------------------------------ convolutional RBM
int b2n_crbm_create(int c_in, int h, int w, int k, int kh, int kw, int device, int precision, b2n_crbm** out) {
    return guard([&] { *out = new b2n_crbm(c_in, h, w, k, kh, kw, device, precision); });
}
int b2n_crbm_destroy(b2n_crbm* m) {
    return guard([&] { delete m; });
}
int b2n_crbm_init(b2n_crbm* m, unsigned seed) {
    return guard([&] { m->impl.init(seed); });
}
int b2n_crbm_set(b2n_crbm* m, const float* kernels, const float* bv, const float* bh) {
    return guard([&] { m->impl.set(kernels, bv, bh); });
}
int b2n_crbm_get(b2n_crbm* m, float* kernels, float* bv, float* bh) {
    return guard([&] { m->impl.get(kernels, bv, bh); });
}
int b2n_crbm_cd_update(b2n_crbm* m, const float* v0, long long batch, float lr, const double* u,
                       long long batch_global, double* recon) {
    return guard([&] {
        B2N_REQUIRE(batch >= 1 && (batch_global == 0 || batch_global >= batch), B2N_ESHAPE,
                    "crbm_cd_update: need 1 <= batch <= batch_global");
        *recon = m->impl.cd_update(v0, batch, lr, u, batch_global ? batch_global : batch);
    });
}
int b2n_crbm_train_stream(b2n_crbm* m, const float* v0, const double* u, long long steps, long long batch, float lr,
                          double* recon_out) {
    return guard([&] { m->impl.train_stream(v0, u, steps, batch, lr, recon_out); });
}
int b2n_crbm_last_states(b2n_crbm* m, float* h0, float* hs, float* v1, float* h1) {
    return guard([&] { m->impl.last_states(h0, hs, v1, h1); });
}
int b2n_crbm_dp_init(b2n_crbm* m, const char id[128], int rank, int world) {
    return guard([&] { m->impl.dp_init(id, rank, world); });
}
int b2n_crbm_keep_states(b2n_crbm* m, int on) {
    return guard([&] { m->impl.keep_states(on != 0); });
}
int b2n_crbm_stage(b2n_crbm* m, const float* v0, const double* u, long long batch) {
    return guard([&] { m->impl.stage(v0, u, batch); });
}
int b2n_crbm_run_staged(b2n_crbm* m, int steps, float lr, long long batch_global) {
    return guard([&] { m->impl.run_staged(steps, lr, batch_global); });
}
int b2n_crbm_recon(b2n_crbm* m, double* recon) {
    return guard([&] { *recon = m->impl.recon(); });
}
int b2n_crbm_kernels_per_step(b2n_crbm* m, int* n) {
    return guard([&] { *n = m->impl.kernels_per_step(); });
}
int b2n_crbm_stream(b2n_crbm* m, void** s) {
    return guard([&] { *s = m->impl.stream(); });
}
int b2n_crbm_profile(b2n_crbm* m, int steps, float lr, long long batch_global, int max_ops, double* stats, char* names,
                     int names_len, int* n_ops) {
    return guard([&] { export_stats(m->impl.profile(steps, lr, batch_global), max_ops, stats, names, names_len, n_ops); });
}

// ------------------------------------------------------------------ op level
int b2n_gemm(const float* A, long long lda, int ta, const float* B, long long ldb, int tb, float* C, long long ldc,
             long long M, long long N, long long K, int precision, void* stream) {
    return guard([&] {
        B2N_REQUIRE(M > 0 && N > 0 && K > 0, B2N_ESHAPE, "gemm extents must be positive");
        b2n::EpiParams e = b2n::epi_default();
        e.C = C;
        e.ldc = ldc;
        // op(A) = A (K-major rows of M) or A^T (A stored K x M: MN-major)
        // op(B) = B^T (B stored N x K: K-major) or B (stored K x N: MN-major)
        b2n::GemmLaunch g = b2n::plan_gemm((int)M, (int)N, (int)K, {A, lda, ta != 0}, {B, ldb, tb == 0}, b2n::EPI_STORE,
                                           e, precision == B2N_TF32X3);
        g.run(as_stream(stream));
    });
}

int b2n_sgd_momentum_step(float* p, float* v, const float* g, long long n, float lr, float momentum, float wd,
                          void* stream) {
    return guard([&] {
        B2N_REQUIRE(n % 4 == 0, B2N_ESHAPE, "sgd: n must be a multiple of 4");
        B2N_REQUIRE(lr > 0.0f, B2N_EPARAM, "optimizer step: lr must be > 0");
        B2N_REQUIRE(momentum >= 0.0f && momentum < 1.0f, B2N_EPARAM, "optimizer step: momentum must be in [0, 1)");
        b2n::sgd_packed_kernel<<<b2n::grid_for(n / 4), 256, 0, as_stream(stream)>>>(
            reinterpret_cast<float4*>(p), reinterpret_cast<float4*>(v), reinterpret_cast<const float4*>(g), n / 4, lr,
            momentum, wd);
        B2N_CUDA(cudaGetLastError());
    });
}

// bring-up: time one GEMM with a per-CTA %globaltimer trace (trace: grid * 64 u64)
int b2n_debug_gemm_trace(const float* A, long long lda, int ta, const float* B, long long ldb, int tb, float* C,
                         long long ldc, long long M, long long N, long long K, int precision, int bn,
                         unsigned long long* trace, int* grid_out) {
    return guard([&] {
        b2n::EpiParams e = b2n::epi_default();
        e.C = C;
        e.ldc = ldc;
        b2n::GemmLaunch g = b2n::plan_gemm((int)M, (int)N, (int)K, {A, lda, ta != 0}, {B, ldb, tb == 0}, b2n::EPI_STORE,
                                           e, precision == B2N_TF32X3, bn);
        g.p.trace = trace;
        g.run(nullptr);
        B2N_CUDA(cudaDeviceSynchronize());
        *grid_out = (int)(g.grid.x * g.grid.y * g.grid.z);
    });
}

// bring-up: copy the B2N_TRACE=1 registry (regions x 512 CTAs x 64 u64 stamps); returns regions used
int b2n_debug_rbm_trace(b2n_rbm* r, unsigned long long* host) {
    return guard([&] { r->impl.read_trace(host); });
}
int b2n_debug_trace_read(unsigned long long* host, long long max_u64, int* regions) {
    return guard([&] {
        auto& r = b2n::TraceRegistry::get();
        *regions = r.used;
        if (!r.buf.p) return;
        const size_t n = std::min<size_t>((size_t)max_u64, r.buf.bytes / 8);
        B2N_CUDA(cudaDeviceSynchronize());
        B2N_CUDA(cudaMemcpy(host, r.buf.p, n * 8, cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"
