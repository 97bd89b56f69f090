/* b200nn.h -- C ABI of the B200-native training step (libb200nn.so).
 *
 * The drop-in boundary for the reference's hot path. The reference (fastnn) is header-only C++
 * with no C ABI; each entry point below replaces the reference interface cited beside it, with
 * plain pointers and sizes (no C++ or torch types). Host-side C++ mirroring fastnn's API
 * (include/b200nn.hpp) and the Python binding (paper_1804_04512_b200/_lib.py) sit on top.
 *
 * Conventions
 *  - Every call returns a status; 0 = B2N_OK. On failure b2n_last_error() gives the message
 *    (thread-local). Status codes map one-to-one onto fastnn's typed exceptions
 *    (config.hpp:11-57), which the C++ wrapper rethrows.
 *  - "host" pointers are ordinary (ideally pinned) CPU memory; "dev" pointers are CUDA device
 *    memory on the object's device. Dense row-major layouts, fastnn logical order
 *    (NCHW for images, (out, in) for dense weights, (k, c, kh, kw) for conv kernels).
 *  - Objects are single-thread affine (fastnn layers are not re-entrant).
 */
#ifndef B200NN_H
#define B200NN_H

#ifdef __cplusplus
extern "C" {
#endif

/* status codes == fastnn error types */
enum {
    B2N_OK = 0,
    B2N_ESHAPE = 1,  /* ShapeError   */
    B2N_EPARAM = 2,  /* ParamError   */
    B2N_ELABEL = 3,  /* LabelError   */
    B2N_ECUDA = 4,   /* CUDA runtime / driver failure */
    B2N_ENCCL = 5,   /* NCCL failure */
    B2N_EOOM = 6,    /* device allocation failure */
    B2N_ESPEC = 7,   /* SpecError    */
    B2N_EBOUNDS = 8, /* BoundsError  */
    B2N_EINTERNAL = 9,
    B2N_EFORMAT = 10, /* FormatError: malformed / mismatched checkpoint */
    B2N_ELENGTH = 11, /* LengthError: checkpoint truncated */
    B2N_EIO = 12,     /* DataMissingError: file cannot be opened / written */
    B2N_ECONSISTENCY = 13, /* ConsistencyError: e.g. a dataset label outside [0, classes) */
    B2N_EDATA = 14         /* DataError: e.g. an empty dataset */
};

/* fastnn::LayerDesc::Kind numbering (network.hpp:195) */
enum {
    B2N_DENSE = 0,
    B2N_CONV = 1,
    B2N_MAXPOOL = 2,
    B2N_SIGMOID = 3,
    B2N_RELU = 4,
    B2N_SOFTMAX = 5,
    B2N_DROPOUT = 6,
    B2N_BATCHNORM = 7,
    B2N_FLATTEN = 8
};

/* tensor-core precision policy: 3xTF32 (split hi/lo, ~fp32; default) or 1xTF32 (fast) */
enum { B2N_TF32X3 = 0, B2N_TF32 = 1 };

/* parameter views for get/set */
enum {
    B2N_VALUE = 0,
    B2N_GRAD = 1,
    B2N_VELOCITY = 2,    /* SGD-momentum velocity */
    B2N_OPT_STATE1 = 3,  /* Adagrad / Adadelta acc, Adam m (optim.hpp:25-26) */
    B2N_OPT_STATE2 = 4   /* Adadelta acc_update, Adam v */
};

/* == fastnn::LayerDesc (network.hpp:194-223) plus a conv zero-padding field (`pad`) that the
 *    reference's ConvShape has (conv.hpp:21) but its LayerDesc cannot set. */
typedef struct b2n_layer_desc {
    int kind;
    long long in, out;    /* dense extents */
    long long k, kh, kw;  /* conv extents */
    long long pad;        /* conv zero padding */
    float p;              /* dropout probability (dropout is outside the hot path: ESPEC) */
} b2n_layer_desc;

/* == fastnn::NetworkSpec (network.hpp:225-234) */
typedef struct b2n_network_spec {
    int input_rank; /* 1: {features}, 3: {c, h, w} */
    long long input[3];
    const b2n_layer_desc* layers;
    int n_layers;
    int optimizer; /* OptimizerKind (optim.hpp:11): 0 SgdMomentum, 1 Adagrad, 2 Adadelta, 3 Adam */
    float lr, momentum, weight_decay;
    long long batch_size;
    unsigned seed;
} b2n_network_spec;

typedef struct b2n_net b2n_net;
typedef struct b2n_rbm b2n_rbm;
typedef struct b2n_crbm b2n_crbm;

const char* b2n_last_error(void);
int b2n_version(void);
int b2n_device_count(int* n);

/* ---- network: replaces build_network / train_minibatch / forward_batch (network.hpp:284-484) ---- */

/* build_network (network.hpp:284-375): same validation (ESPEC), same seeded Glorot init
 * (layers.hpp:40-48, identical std::mt19937 draws), parameters resident on `device`. */
int b2n_build_network(const b2n_network_spec* spec, int device, int precision, b2n_net** out);
int b2n_net_destroy(b2n_net* net);

/* Network::trainable() order (network.hpp:244-249): w then b per dense / conv layer */
int b2n_net_num_params(b2n_net* net, int* n);
int b2n_net_param_shape(b2n_net* net, int idx, int* rank, long long dims[4]);
int b2n_net_get_param(b2n_net* net, int idx, int which, float* host);
int b2n_net_set_param(b2n_net* net, int idx, int which, const float* host);
int b2n_net_set_hparams(b2n_net* net, float lr, float momentum, float weight_decay);

/* train_minibatch (network.hpp:463-472): forward, softmax-xent, backward, SGD-momentum step
 * (skipped when lr == 0), gradients cleared. y_onehot is validated like network.hpp:423-432
 * (ELABEL). Host buffers; returns the mean loss. */
int b2n_train_minibatch(b2n_net* net, const float* x_host, const float* y_onehot_host, long long batch,
                        double* loss);
/* same with int class ids (the shim's one-hot -> id conversion skipped) */
int b2n_train_minibatch_labels(b2n_net* net, const float* x_host, const int* labels_host, long long batch,
                               double* loss);
/* forward_batch + argmax_row (network.hpp:66-72, :402): probs (batch x classes) and first-max ids */
/* `steps` train_minibatch_labels calls over consecutive host batches: step i uses rows
 * [i*batch, (i+1)*batch) of x_host / labels_host; the host->device copy of step i+1 overlaps
 * step i (double-buffered staging on a copy stream). loss_out[i] = step i's loss. */
int b2n_net_train_stream(b2n_net* net, const float* x_host, const int* labels_host, long long steps, long long batch,
                         double* loss_out);
int b2n_forward_batch(b2n_net* net, const float* x_host, long long batch, float* probs_host, int* argmax_host);

/* Data-parallel pieces. forward_backward leaves the full-batch-scaled gradient
 * (dlogits / batch_global) in the packed gradient buffer without touching parameters;
 * apply_update runs the SGD-momentum kernel over the packed buffers. With b2n_net_dp_init the
 * step allreduces the gradient over NCCL between the two. */
int b2n_net_forward_backward(b2n_net* net, const float* x_host, const int* labels_host, long long batch,
                             long long batch_global, double* loss_share);
int b2n_net_apply_update(b2n_net* net);
/* Inspection of the last forward (per-layer parity; no reference counterpart -- fastnn keeps its node
 * outputs in Network::forward's locals, network.hpp:58-64): the output of fused layer `layer` (conv +
 * act + 2x2 pool, or dense + act) for `batch` rows, NCHW per row, and the pool argmax codes in the
 * same order (codes may be NULL). */
int b2n_net_num_layers(b2n_net* net, long long* n);
int b2n_net_layer_output(b2n_net* net, int layer, long long batch, float* out_host, unsigned char* codes_host);
int b2n_net_grad_buffer(b2n_net* net, float** dev_ptr, long long* n_floats);
int b2n_nccl_unique_id(char id_out[128]);
int b2n_net_dp_init(b2n_net* net, const char id[128], int rank, int world);

/* Device-resident stepping (throughput measurement): stage a batch into the net's device input
 * buffers once, then run `steps` whole training steps as CUDA-graph launches on the net's
 * stream without host synchronisation. b2n_net_loss waits and returns the last step's loss. */
int b2n_net_stage(b2n_net* net, const float* x_host, const int* labels_host, long long batch);
int b2n_net_run_staged(b2n_net* net, int steps, long long batch_global);
int b2n_net_loss(b2n_net* net, double* loss);
int b2n_net_stream(b2n_net* net, void** cuda_stream);
int b2n_net_kernels_per_step(b2n_net* net, long long batch, int* n);
/* fit (network.hpp:488-511) over a dataset held in device memory: images (n x prod(input)),
 * int class ids (validated like data.hpp:257-260, ECONSISTENCY; empty dataset EDATA). Batches follow BatchIterator's order
 * (data.hpp:224-238: std::shuffle with mt19937(net seed), reshuffled with seed + epoch) and are
 * gathered on the device; one host synchronisation per epoch. Per epoch: loss (mean row loss),
 * accuracy (evaluate over the training set) and the batch-loop wall time. Arrays hold `epochs`
 * entries. */
int b2n_net_fit(b2n_net* net, const float* images_host, const int* labels_host, long long n, int epochs,
                double* loss_out, double* accuracy_out, double* seconds_out);
/* evaluate (network.hpp:474-484): fraction of rows whose first-max class equals the label,
 * forward_batch in net.batch_size chunks in dataset order */
int b2n_net_evaluate(b2n_net* net, const float* images_host, const int* labels_host, long long n,
                     double* accuracy);
/* BatchIterator's sample order for epoch `epoch` (0 = construction shuffle) */
int b2n_batch_order(long long n, unsigned seed, int epoch, long long* order_out);
/* save_network / load_network (network.hpp:552-607): the reference's FNN1 byte format, written
 * from / read into the device-resident parameters (one packed D2H / H2D copy). with_state != 0
 * also writes / reads the sidecar `<path>.state` holding momentum velocities and hyper-parameters
 * for an exact resume (the reference has no such file). Errors: EIO (cannot open), ELENGTH
 * (truncated), EFORMAT (magic, layer count, tag, tensor count / rank / extent mismatch). */
int b2n_save_network(b2n_net* net, const char* path, int with_state);
int b2n_load_network(b2n_net* net, const char* path, int with_state);
/* Per-op device time of the planned step (un-graphed launches, CUDA events between ops), averaged
 * over `steps`: stats[i*4 + {0,1,2,3}] = {ms, algorithmic FLOPs, algorithmic HBM bytes, kernels};
 * names gets the op names, newline-separated. */
int b2n_net_profile(b2n_net* net, long long batch, int steps, int max_ops, double* stats, char* names, int names_len,
                    int* n_ops);

/* A source of Bernoulli uniforms: writes the next `count` draws of the caller's stream
 * (std::generate_canonical<double,53> over its std::mt19937 -- what std::bernoulli_distribution
 * consumes) to `out`. Called on the calling thread, in step order. */
typedef void (*b2n_uniform_fn)(void* ctx, double* out, long long count);

/* The reference's generator on the device. A std::mt19937 is passed as its libstdc++ state: the
 * 624 state words then the position (_M_x[0..623], _M_p -- the 625 numbers `os << rng` prints).
 * Every entry point below that takes uniforms_host also accepts NULL: the draws then come from the
 * object's device copy of the caller's generator (set with *_set_rng, read back with *_get_rng),
 * generated on the GPU bit-exactly as std::bernoulli_distribution would have drawn them
 * (generate_canonical<double,53>, energy.hpp:53-71) -- no host draws, no uniforms over PCIe.
 * b2n_mt19937_draw: the next n generate_canonical<double,53> draws of `state` (advanced in place). */
int b2n_mt19937_draw(int device, unsigned state[625], double* out_host, long long n);

/* ---- RBM: replaces Rbm (energy.hpp:16-32) and cd_k_update (energy.hpp:131-171) ---- */
int b2n_rbm_create(long long hidden, long long visible, int device, int precision, b2n_rbm** out);
int b2n_rbm_destroy(b2n_rbm* rbm);
/* Rbm::init (energy.hpp:31): Glorot on w with std::mt19937(seed), zero biases */
int b2n_rbm_init(b2n_rbm* rbm, unsigned seed);
int b2n_rbm_set(b2n_rbm* rbm, const float* w_host, const float* bv_host, const float* bh_host);
int b2n_rbm_get(b2n_rbm* rbm, float* w_host, float* bv_host, float* bh_host);
/* cd_k_update for binary units. uniforms_host holds the k*batch*hidden draws
 * std::bernoulli_distribution would consume (generate_canonical<double,53>, row-major per Gibbs
 * step): h = (u < p) is then bit-exact with the reference's sampling given the same p.
 * batch_global > batch makes this a data-parallel shard (lr / batch_global scaling). */
int b2n_cd_k_update(b2n_rbm* rbm, const float* v0_host, long long batch, int k, float lr,
                    const double* uniforms_host, long long batch_global, double* recon);
/* the chain states of the last update (h0 mean, h sample, v1 mean, h1 mean), batch-major */
int b2n_rbm_last_states(b2n_rbm* rbm, float* h0, float* hs, float* v1, float* h1);
int b2n_rbm_dp_init(b2n_rbm* rbm, const char id[128], int rank, int world);
/* Data parallelism driven by the caller (no NCCL; e.g. a gloo / MPI allreduce): with grad_only on,
 * b2n_cd_k_update(..., batch_global) leaves the parameters alone and keeps this shard's raw sums
 * dW = h0^T v0 - h1^T v1, dbh = sum(h0 - h1), dbv = sum(v0 - v1) (energy.hpp:148-169 before the
 * lr / batch scale); get_grad / set_grad move them (w: hidden x visible), apply_update adds
 * lr / batch_global * (the summed sums) -- the same arithmetic the NCCL mode runs in its step. */
int b2n_rbm_set_grad_only(b2n_rbm* rbm, int on);
/* the device generator behind uniforms_host == NULL (see b2n_mt19937_draw) */
int b2n_rbm_set_rng(b2n_rbm* rbm, const unsigned state[625]);
int b2n_rbm_get_rng(b2n_rbm* rbm, unsigned state[625]);
int b2n_rbm_get_grad(b2n_rbm* rbm, float* w_host, float* bv_host, float* bh_host);
int b2n_rbm_set_grad(b2n_rbm* rbm, const float* w_host, const float* bv_host, const float* bh_host);
int b2n_rbm_apply_update(b2n_rbm* rbm, float lr, long long batch_global);
int b2n_rbm_stage(b2n_rbm* rbm, const float* v0_host, const double* uniforms_host, long long batch);
int b2n_rbm_run_staged(b2n_rbm* rbm, int steps, float lr, long long batch_global);
int b2n_rbm_recon(b2n_rbm* rbm, double* recon);
/* `steps` CD-1 updates (k = 1) over consecutive host batches -- the reference's loop of
 * cd_k_update calls: step i uses rows [i*batch, (i+1)*batch) of v0_host (steps*batch x visible)
 * and of uniforms_host (steps*batch x hidden). The host->device copy of step i+1 overlaps step i
 * (staged up to 4 steps ahead on a copy stream); recon_out[i] = step i's reconstruction error.
 * v0_host / uniforms_host may also be device pointers (device-resident batches). */
int b2n_rbm_train_stream(b2n_rbm* rbm, const float* v0_host, const double* uniforms_host, long long steps,
                         long long batch, float lr, double* recon_out);
int b2n_rbm_stream(b2n_rbm* rbm, void** cuda_stream);
/* dbn_pretrain (energy.hpp:208-240): greedy CD-1 training of a stack of `layers` RBMs (layer l's
 * visible extent == layer l-1's hidden extent; all on one device). `data` (n x visible(0), host)
 * is uploaded once; each layer trains `epochs` passes of CD-1 over its input in file order,
 * `batch` rows per step, then its hidden means (rbm_transform_up, energy.hpp:122-126) become the
 * next layer's input -- on the device. Uniforms: B x H per step from `fill`, layer by layer,
 * epoch by epoch, batch by batch (the reference's single rng stream). recon_out[layer*epochs + e]
 * = mean per-step reconstruction error. Errors: EPARAM (empty stack, batch < 1, epochs < 0),
 * ESHAPE (extent chain, the reference's message). fill == NULL: ctx is the caller's generator
 * state (unsigned[625], see b2n_mt19937_draw), drawn from and advanced on the device. */
int b2n_dbn_pretrain(b2n_rbm* const* stack, int layers, const float* data_host, long long n, int epochs, float lr,
                     long long batch, b2n_uniform_fn fill, void* ctx, double* recon_out);
int b2n_rbm_kernels_per_step(b2n_rbm* rbm, int* n);
int b2n_rbm_profile(b2n_rbm* rbm, int steps, float lr, long long batch_global, int max_ops, double* stats, char* names,
                    int names_len, int* n_ops);

/* ---- convolutional RBM: replaces Crbm (energy.hpp:245-262) and crbm_cd_update
 * (energy.hpp:333-376), binary units, non-pooled formulation, valid convolutions ----
 * kernels (k, c_in, kh, kw), bv (c_in), bh (k); visible batches NCHW (batch, c_in, h, w).
 * Errors: ESHAPE for kh > h or kw > w (the reference's "crbm: kernel extents exceed visible
 * extents") and outside the tensor-core conv envelope (k, c_in <= 32, c_in*kh*kw <= 320,
 * k*kh*kw <= 320). */
int b2n_crbm_create(int c_in, int h, int w, int k, int kh, int kw, int device, int precision, b2n_crbm** out);
int b2n_crbm_destroy(b2n_crbm* crbm);
/* Crbm::init (energy.hpp:261): Glorot(c_in*kh*kw, k*kh*kw) on the kernels, std::mt19937(seed) */
int b2n_crbm_init(b2n_crbm* crbm, unsigned seed);
int b2n_crbm_set(b2n_crbm* crbm, const float* kernels_host, const float* bv_host, const float* bh_host);
int b2n_crbm_get(b2n_crbm* crbm, float* kernels_host, float* bv_host, float* bh_host);
/* crbm_cd_update: uniforms_host holds the batch*k*oh*ow draws unit_sample_inplace consumes
 * (generate_canonical<double,53>, NCHW order); recon = sum (v0 - v1)^2 / batch_global. */
int b2n_crbm_cd_update(b2n_crbm* crbm, const float* v0_host, long long batch, float lr,
                       const double* uniforms_host, long long batch_global, double* recon);
/* the chain states of the last update (h0 mean, h sample, v1 mean, h1 mean), NCHW; the fused
 * one-launch step keeps them in shared memory unless keep_states was enabled before the step
 * (EPARAM otherwise) */
int b2n_crbm_keep_states(b2n_crbm* crbm, int on);
/* data-parallel CRBM (one process per GPU): each rank steps its shard with batch_global = the
 * global batch; the shards' parameter and reconstruction sums are allreduced (NCCL) before the
 * identical update on every rank. Needs the one-launch step's shape envelope (EPARAM otherwise). */
int b2n_crbm_dp_init(b2n_crbm* crbm, const char id[128], int rank, int world);
int b2n_crbm_last_states(b2n_crbm* crbm, float* h0, float* hs, float* v1, float* h1);
/* `steps` crbm_cd_update calls over consecutive host batches of v0_host (steps*batch images, NCHW):
 * uniforms_host (steps*batch*k*oh*ow) or NULL (the device generator, several steps generated
 * concurrently by jump-ahead); the next steps' copies overlap the current one; recon_out[i] = step i's
 * reconstruction error. v0_host / uniforms_host may be device pointers. */
int b2n_crbm_train_stream(b2n_crbm* crbm, const float* v0_host, const double* uniforms_host, long long steps,
                          long long batch, float lr, double* recon_out);
int b2n_crbm_set_rng(b2n_crbm* crbm, const unsigned state[625]);
int b2n_crbm_get_rng(b2n_crbm* crbm, unsigned state[625]);
int b2n_crbm_stage(b2n_crbm* crbm, const float* v0_host, const double* uniforms_host, long long batch);
int b2n_crbm_run_staged(b2n_crbm* crbm, int steps, float lr, long long batch_global);
int b2n_crbm_recon(b2n_crbm* crbm, double* recon);
int b2n_crbm_kernels_per_step(b2n_crbm* crbm, int* n);
int b2n_crbm_stream(b2n_crbm* crbm, void** cuda_stream);
int b2n_crbm_profile(b2n_crbm* crbm, int steps, float lr, long long batch_global, int max_ops, double* stats,
                     char* names, int names_len, int* n_ops);

/* ---- op level (device pointers, async on `stream`; NULL = default stream) ---- */
/* gemm (gemm.hpp:225-229): C = op(A) . op(B); lda/ldb/ldc are row pitches in floats (multiples
 * of 4, 16-byte aligned bases -- every fastnn tensor satisfies this, tensor.hpp:142) */
int b2n_gemm(const float* A, long long lda, int transpose_a, const float* B, long long ldb, int transpose_b,
             float* C, long long ldc, long long M, long long N, long long K, int precision, void* stream);
/* ---- the reference's op-level layer API (layers.hpp:124-320, network.hpp:410-437) on host tensors,
 * bit-identical to fastnn's (each op computes in the reference's own order; ops.cu). For programs that
 * call the layer functions directly; the training step itself runs the fused kernels above. ---- */
typedef struct b2n_conv_shape {  /* fastnn::ConvShape (conv.hpp:20) */
    long long n, c_in, k, kh, kw, h, w, pad;
} b2n_conv_shape;
/* conv_forward (layers.hpp:132): y (n, k, oh, ow) = valid conv of x (n, c_in, h, w) padded by pad with
 * kernels (k, c_in, kh, kw), + bias (k) */
int b2n_op_conv_forward(int device, const b2n_conv_shape* shape, const float* x, const float* kernels,
                        const float* bias, float* y);
/* conv_backward (layers.hpp:152): dx (n, c_in, h, w); gk (k, c_in, kh, kw) and gb (k) ACCUMULATE into
 * their incoming values, as the layer's gradient tensors do. ESHAPE for pad != 0 (the reference's
 * "padded forward has no backward pass"); EPARAM for kernels above 5x5 (the reference's FFT backend). */
int b2n_op_conv_backward(int device, const b2n_conv_shape* shape, const float* x, const float* kernels,
                         const float* dy, float* gk, float* gb, float* dx);
/* pool_forward / pool_backward (layers.hpp:205, :240): mode 0 = max (argmax = in-window index 0..3 as
 * float, ties keep the first), 1 = avg; maps = product of the leading extents */
int b2n_op_pool_forward(int device, int mode, long long maps, long long h, long long w, const float* x, float* y,
                        float* argmax);
int b2n_op_pool_backward(int device, int mode, long long maps, long long oh, long long ow, const float* dy,
                         const float* argmax, float* dx);
/* activation_apply / activation_gradient (layers.hpp:278-299): kind 0 = sigmoid, 1 = relu; the gradient
 * takes the forward output y */
int b2n_op_activation_apply(int device, int kind, long long n, const float* x, float* y);
int b2n_op_activation_gradient(int device, int kind, long long n, const float* y, const float* dy, float* dx);
/* softmax (layers.hpp:301), softmax_cross_entropy (network.hpp:410): LABEL for labels that are not
 * one-hot (the reference's message) */
int b2n_op_softmax(int device, long long rows, long long cols, const float* x, float* y);
int b2n_op_softmax_cross_entropy(int device, long long rows, long long cols, const float* predictions,
                                 const float* labels, float* dlogits, double* loss);

/* sgd_momentum_step (optim.hpp:69-80) over n contiguous floats (n % 4 == 0, 16-byte aligned) */
int b2n_sgd_momentum_step(float* p, float* v, const float* g, long long n, float lr, float momentum,
                          float weight_decay, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* B200NN_H */
