// ops.cu -- the reference's op-level layer API on the GPU (layers.hpp:124-320, network.hpp:410-437):
// conv_forward, conv_backward, pool_forward / pool_backward, activation_apply / _gradient, softmax
// and softmax_cross_entropy as standalone C-ABI calls on host tensors (b2n_op_*, include/b200nn.h),
// for a fastnn program that calls the layer functions directly instead of train_minibatch.
//
// These are the drop-in for the reference's per-op entry points, not the training hot path (the step
// kernels fuse the same arithmetic: network.cuh / convx.cuh / convt.cuh). Every one of them computes
// in the reference's own order so its results are bit-identical to fastnn's:
//   conv_forward   one fp32 fma chain per output over (c, di, dj) from 0, padding contributing exact
//                  zeros, then + bias (conv.hpp:62-119 add_corr_map / :215-273 im2col, layers.hpp:132-148)
//   conv_backward  dx: the padded-valid full conv (conv.hpp:337-345, kernels <= 5x5), one chain per
//                  input pixel over (kernel f, di, dj) of the flipped, channel-transposed taps;
//                  gk: per (f, c, tap) one chain over the images and the dy pixels in row-major order,
//                  continuing from the incoming gk (layers.hpp:176-184); gb: sequential sums (:185-191)
//   pool           2x2 windows, first-index max (layers.hpp:205-271)
//   softmax        max, expf(x - max), sequential sum, divide (layers.hpp:301-320); expf is glibc's own
//                  algorithm (ptx.cuh glibc_expf), bit for bit
//   softmax_cross_entropy  the one-hot check on the host (LabelError), dlogits = (p - y) / (float)b on
//                  the device, the loss as the reference's ordered sum of per-row double logs
#include <cstring>
#include <string>
#include <vector>

#include "../../include/b200nn.h"
#include "runtime.cuh"

namespace b2n {
namespace {

__device__ __forceinline__ float expf_rn(float v) { return glibc_expf(v); }  // libm's expf, bit for bit

__global__ void op_conv_fwd_kernel(const float* __restrict__ x, const float* __restrict__ ker,
                                   const float* __restrict__ bias, float* __restrict__ y, long long n, int C, int H,
                                   int W, int K, int KH, int KW, int pad, int OH, int OW) {
    const long long total = n * K * OH * OW;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int ox = (int)(i % OW), oy = (int)((i / OW) % OH), k = (int)((i / ((long long)OW * OH)) % K);
        const long long img = i / ((long long)OW * OH * K);
        float acc = 0.0f;
        for (int c = 0; c < C; ++c) {
            const float* xc = x + ((img * C + c) * H) * (long long)W;
            const float* kc = ker + ((long long)k * C + c) * KH * KW;
            for (int di = 0; di < KH; ++di) {
                const int iy = oy + di - pad;
                for (int dj = 0; dj < KW; ++dj) {
                    const int ix = ox + dj - pad;
                    const float v = (iy >= 0 && iy < H && ix >= 0 && ix < W) ? xc[(long long)iy * W + ix] : 0.0f;
                    acc = fmaf(kc[di * KW + dj], v, acc);
                }
            }
        }
        y[i] = acc + bias[k];
    }
}

// dx[img][c][y][x] = sum_f sum_di sum_dj dy_pad[img][f][y + di][x + dj] * ker[f][c][KH-1-di][KW-1-dj]
__global__ void op_conv_dx_kernel(const float* __restrict__ dy, const float* __restrict__ ker, float* __restrict__ dx,
                                  long long n, int C, int H, int W, int K, int KH, int KW, int OH, int OW) {
    const long long total = n * C * H * W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int xx = (int)(i % W), yy = (int)((i / W) % H), c = (int)((i / ((long long)W * H)) % C);
        const long long img = i / ((long long)W * H * C);
        float acc = 0.0f;
        for (int f = 0; f < K; ++f) {
            const float* d = dy + ((img * K + f) * OH) * (long long)OW;
            const float* kf = ker + ((long long)f * C + c) * KH * KW;
            for (int di = 0; di < KH; ++di) {
                const int sy = yy + di - (KH - 1);
                for (int dj = 0; dj < KW; ++dj) {
                    const int sx = xx + dj - (KW - 1);
                    const float v = (sy >= 0 && sy < OH && sx >= 0 && sx < OW) ? d[(long long)sy * OW + sx] : 0.0f;
                    acc = fmaf(kf[(KH - 1 - di) * KW + (KW - 1 - dj)], v, acc);
                }
            }
        }
        dx[i] = acc;
    }
}

// gk[f][c][di][dj] continues its chain over images, then dy pixels row-major; gb[f] likewise (adds)
__global__ void op_conv_gk_kernel(const float* __restrict__ x, const float* __restrict__ dy, float* gk, float* gb,
                                  long long n, int C, int H, int W, int K, int KH, int KW, int OH, int OW) {
    const int total = K * C * KH * KW;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < total) {
        const int dj = i % KW, di = (i / KW) % KH, c = (i / (KW * KH)) % C, f = i / (KW * KH * C);
        float acc = gk[i];
        for (long long img = 0; img < n; ++img) {
            const float* xc = x + ((img * C + c) * H) * (long long)W;
            const float* d = dy + ((img * K + f) * OH) * (long long)OW;
            for (int oy = 0; oy < OH; ++oy)
                for (int ox = 0; ox < OW; ++ox) acc = fmaf(d[oy * OW + ox], xc[(long long)(oy + di) * W + ox + dj], acc);
        }
        gk[i] = acc;
    } else if (i < total + K) {
        const int f = i - total;
        float acc = gb[f];
        for (long long img = 0; img < n; ++img) {
            const float* d = dy + ((img * K + f) * OH) * (long long)OW;
            for (int p = 0; p < OH * OW; ++p) acc += d[p];
        }
        gb[f] = acc;
    }
}

__global__ void op_pool_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, float* __restrict__ arg,
                                   long long maps, int H, int W, int avg) {
    const int oh = H / 2, ow = W / 2;
    const long long total = maps * oh * ow;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int ox = (int)(i % ow), oy = (int)((i / ow) % oh);
        const long long m = i / ((long long)ow * oh);
        const float* r0 = x + (m * H + 2 * oy) * (long long)W;
        const float* r1 = r0 + W;
        const float v[4] = {r0[2 * ox], r0[2 * ox + 1], r1[2 * ox], r1[2 * ox + 1]};
        if (avg) {
            y[i] = (v[0] + v[1] + v[2] + v[3]) / 4.0f;
        } else {
            int best = 0;
            for (int j = 1; j < 4; ++j)
                if (v[j] > v[best]) best = j;  // ties keep the first index
            y[i] = v[best];
            arg[i] = (float)best;
        }
    }
}

__global__ void op_pool_bwd_kernel(const float* __restrict__ dy, const float* __restrict__ arg, float* __restrict__ dx,
                                   long long maps, int oh, int ow, int avg) {
    const long long total = maps * oh * ow;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int ox = (int)(i % ow), oy = (int)((i / ow) % oh);
        const long long m = i / ((long long)ow * oh);
        float* r0 = dx + (m * 2 * oh + 2 * oy) * (long long)(2 * ow);
        float* r1 = r0 + 2 * ow;
        const float g = dy[i];
        if (avg) {
            const float v = g / 4.0f;
            r0[2 * ox] = r0[2 * ox + 1] = r1[2 * ox] = r1[2 * ox + 1] = v;
        } else {
            const int best = (int)arg[i];
            r0[2 * ox] = r0[2 * ox + 1] = r1[2 * ox] = r1[2 * ox + 1] = 0.0f;
            (best < 2 ? r0 : r1)[2 * ox + best % 2] = g;
        }
    }
}

__global__ void op_act_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out,
                              long long n, int kind, int grad) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float v = a[i];
        if (!grad)
            out[i] = kind == 0 ? 1.0f / (1.0f + expf_rn(-v)) : (v > 0.0f ? v : 0.0f);
        else  // a = y (forward output), b = dy
            out[i] = kind == 0 ? b[i] * v * (1.0f - v) : (v > 0.0f ? b[i] : 0.0f);
    }
}

// one thread per row, the reference's sequential order
__global__ void op_softmax_kernel(const float* __restrict__ x, float* __restrict__ y, long long rows, int cols) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows; r += (long long)gridDim.x * blockDim.x) {
        const float* p = x + r * cols;
        float* q = y + r * cols;
        float m = p[0];
        for (int j = 1; j < cols; ++j) m = fmaxf(m, p[j]);
        float sum = 0.0f;
        for (int j = 0; j < cols; ++j) {
            q[j] = expf_rn(p[j] - m);
            sum += q[j];
        }
        for (int j = 0; j < cols; ++j) q[j] /= sum;
    }
}

__global__ void op_xent_kernel(const float* __restrict__ p, const float* __restrict__ yl, const int* __restrict__ truth,
                               float* __restrict__ g, double* __restrict__ rowlog, long long rows, int cols) {
    const long long total = rows * cols;
    const float fb = (float)rows;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        g[i] = (p[i] - yl[i]) / fb;
        if (i % cols == 0) {
            const long long r = i / cols;
            rowlog[r] = log(fmax((double)p[r * cols + truth[r]], 1e-300));
        }
    }
}

// device copies of a call's host tensors, freed in stream order
struct OpMem {
    cudaStream_t st = nullptr;
    std::vector<void*> ptrs;
    explicit OpMem(int device) {
        B2N_CUDA(cudaSetDevice(device));
        B2N_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    }
    ~OpMem() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
    template <class T>
    T* up(const T* h, long long n) {
        T* d = alloc<T>(n);
        if (n) B2N_CUDA(cudaMemcpyAsync(d, h, (size_t)n * sizeof(T), cudaMemcpyHostToDevice, st));
        return d;
    }
    template <class T>
    T* alloc(long long n) {
        void* d = nullptr;
        B2N_CUDA(cudaMallocAsync(&d, (size_t)std::max<long long>(n, 1) * sizeof(T), st));
        ptrs.push_back(d);
        return static_cast<T*>(d);
    }
    template <class T>
    void down(T* h, const T* d, long long n) {
        if (n) B2N_CUDA(cudaMemcpyAsync(h, d, (size_t)n * sizeof(T), cudaMemcpyDeviceToHost, st));
    }
    void sync() {
        B2N_CUDA(cudaGetLastError());
        B2N_CUDA(cudaStreamSynchronize(st));
    }
};

int grid_of(long long n) { return (int)std::min<long long>((n + 255) / 256, 148LL * 16); }

}  // namespace
}  // namespace b2n

namespace b2n {
void set_last_error(const char* msg);  // b200nn.cu: the thread's b2n_last_error() text
}
namespace {
template <class F>
int op_guard(F&& f) {
    try {
        f();
        b2n::set_last_error("");
        return B2N_OK;
    } catch (const b2n::Error& e) {
        b2n::set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        b2n::set_last_error("host allocation failed");
        return B2N_EOOM;
    } catch (const std::exception& e) {
        b2n::set_last_error(e.what());
        return B2N_EINTERNAL;
    }
}
void check_conv(const b2n_conv_shape* s) {
    if (!s || s->n < 1 || s->c_in < 1 || s->k < 1 || s->kh < 1 || s->kw < 1 || s->h < 1 || s->w < 1 || s->pad < 0)
        throw b2n::Error(B2N_ESHAPE, "conv: extents must be positive");
    if (s->kh > s->h + 2 * s->pad || s->kw > s->w + 2 * s->pad)
        throw b2n::Error(B2N_ESHAPE, "conv: kernel extents exceed the padded input");
}
}  // namespace

extern "C" {

int b2n_op_conv_forward(int device, const b2n_conv_shape* s, const float* x, const float* kernels, const float* bias,
                        float* y) {
    return op_guard([&] {
        check_conv(s);
        const long long n = s->n, C = s->c_in, H = s->h, W = s->w, K = s->k, KH = s->kh, KW = s->kw, pad = s->pad;
        const long long OH = H + 2 * pad - KH + 1, OW = W + 2 * pad - KW + 1;
        b2n::OpMem m(device);
        const float* dx = m.up(x, n * C * H * W);
        const float* dk = m.up(kernels, K * C * KH * KW);
        const float* db = m.up(bias, K);
        float* dy = m.alloc<float>(n * K * OH * OW);
        b2n::op_conv_fwd_kernel<<<b2n::grid_of(n * K * OH * OW), 256, 0, m.st>>>(
            dx, dk, db, dy, n, (int)C, (int)H, (int)W, (int)K, (int)KH, (int)KW, (int)pad, (int)OH, (int)OW);
        m.down(y, (const float*)dy, n * K * OH * OW);
        m.sync();
    });
}

int b2n_op_conv_backward(int device, const b2n_conv_shape* s, const float* x, const float* kernels, const float* dy,
                         float* gk, float* gb, float* dx) {
    return op_guard([&] {
        check_conv(s);
        if (s->pad != 0) throw b2n::Error(B2N_ESHAPE, "conv_backward: padded forward has no backward pass");
        if (s->kh * s->kw > 25)
            throw b2n::Error(B2N_EPARAM, "conv_backward: kernels above 5x5 (the reference's FFT backend) are not offered");
        const long long n = s->n, C = s->c_in, H = s->h, W = s->w, K = s->k, KH = s->kh, KW = s->kw;
        const long long OH = H - KH + 1, OW = W - KW + 1;
        b2n::OpMem m(device);
        const float* d_x = m.up(x, n * C * H * W);
        const float* d_k = m.up(kernels, K * C * KH * KW);
        const float* d_dy = m.up(dy, n * K * OH * OW);
        float* d_gk = m.up(gk, K * C * KH * KW);
        float* d_gb = m.up(gb, K);
        float* d_dx = m.alloc<float>(n * C * H * W);
        b2n::op_conv_dx_kernel<<<b2n::grid_of(n * C * H * W), 256, 0, m.st>>>(d_dy, d_k, d_dx, n, (int)C, (int)H, (int)W,
                                                                             (int)K, (int)KH, (int)KW, (int)OH, (int)OW);
        const long long ng = K * C * KH * KW + K;
        b2n::op_conv_gk_kernel<<<(int)((ng + 127) / 128), 128, 0, m.st>>>(d_x, d_dy, d_gk, d_gb, n, (int)C, (int)H,
                                                                          (int)W, (int)K, (int)KH, (int)KW, (int)OH,
                                                                          (int)OW);
        m.down(dx, (const float*)d_dx, n * C * H * W);
        m.down(gk, (const float*)d_gk, K * C * KH * KW);
        m.down(gb, (const float*)d_gb, K);
        m.sync();
    });
}

int b2n_op_pool_forward(int device, int mode, long long maps, long long h, long long w, const float* x, float* y,
                        float* argmax) {
    return op_guard([&] {
        if (maps < 1 || h < 1 || w < 1) throw b2n::Error(B2N_ESHAPE, "pool_forward: expected rank >= 2");
        if (h % 2 || w % 2)
            throw b2n::Error(B2N_ESHAPE, "pool_forward: spatial extents must be even, got " + std::to_string(h) + "x" +
                                             std::to_string(w));
        if (mode == 0 && !argmax) throw b2n::Error(B2N_EPARAM, "pool_forward: max mode needs an argmax output");
        b2n::OpMem m(device);
        const float* d_x = m.up(x, maps * h * w);
        const long long no = maps * (h / 2) * (w / 2);
        float* d_y = m.alloc<float>(no);
        float* d_a = m.alloc<float>(no);
        b2n::op_pool_fwd_kernel<<<b2n::grid_of(no), 256, 0, m.st>>>(d_x, d_y, d_a, maps, (int)h, (int)w, mode != 0);
        m.down(y, (const float*)d_y, no);
        if (mode == 0) m.down(argmax, (const float*)d_a, no);
        m.sync();
    });
}

int b2n_op_pool_backward(int device, int mode, long long maps, long long oh, long long ow, const float* dy,
                         const float* argmax, float* dx) {
    return op_guard([&] {
        if (maps < 1 || oh < 1 || ow < 1) throw b2n::Error(B2N_ESHAPE, "pool_backward: expected rank >= 2");
        if (mode == 0 && !argmax) throw b2n::Error(B2N_ESHAPE, "pool_backward: dy/argmax shape mismatch");
        b2n::OpMem m(device);
        const long long no = maps * oh * ow;
        const float* d_dy = m.up(dy, no);
        const float* d_a = mode == 0 ? m.up(argmax, no) : nullptr;
        float* d_dx = m.alloc<float>(4 * no);
        b2n::op_pool_bwd_kernel<<<b2n::grid_of(no), 256, 0, m.st>>>(d_dy, d_a, d_dx, maps, (int)oh, (int)ow, mode != 0);
        m.down(dx, (const float*)d_dx, 4 * no);
        m.sync();
    });
}

int b2n_op_activation_apply(int device, int kind, long long n, const float* x, float* y) {
    return op_guard([&] {
        if (kind != 0 && kind != 1) throw b2n::Error(B2N_EPARAM, "activation: kind is 0 (sigmoid) or 1 (relu)");
        b2n::OpMem m(device);
        const float* d_x = m.up(x, n);
        float* d_y = m.alloc<float>(n);
        b2n::op_act_kernel<<<b2n::grid_of(n), 256, 0, m.st>>>(d_x, nullptr, d_y, n, kind, 0);
        m.down(y, (const float*)d_y, n);
        m.sync();
    });
}

int b2n_op_activation_gradient(int device, int kind, long long n, const float* y, const float* dy, float* dx) {
    return op_guard([&] {
        if (kind != 0 && kind != 1) throw b2n::Error(B2N_EPARAM, "activation: kind is 0 (sigmoid) or 1 (relu)");
        b2n::OpMem m(device);
        const float* d_y = m.up(y, n);
        const float* d_g = m.up(dy, n);
        float* d_x = m.alloc<float>(n);
        b2n::op_act_kernel<<<b2n::grid_of(n), 256, 0, m.st>>>(d_y, d_g, d_x, n, kind, 1);
        m.down(dx, (const float*)d_x, n);
        m.sync();
    });
}

int b2n_op_softmax(int device, long long rows, long long cols, const float* x, float* y) {
    return op_guard([&] {
        if (rows < 1 || cols < 1) throw b2n::Error(B2N_ESHAPE, "softmax: expected a rank-2 tensor");
        b2n::OpMem m(device);
        const float* d_x = m.up(x, rows * cols);
        float* d_y = m.alloc<float>(rows * cols);
        b2n::op_softmax_kernel<<<b2n::grid_of(rows), 256, 0, m.st>>>(d_x, d_y, rows, (int)cols);
        m.down(y, (const float*)d_y, rows * cols);
        m.sync();
    });
}

int b2n_op_softmax_cross_entropy(int device, long long rows, long long cols, const float* predictions,
                                 const float* labels, float* dlogits, double* loss) {
    return op_guard([&] {
        if (rows < 1 || cols < 1)
            throw b2n::Error(B2N_ESHAPE, "softmax_cross_entropy: predictions and labels must both be (batch, classes)");
        std::vector<int> truth((size_t)rows);
        for (long long r = 0; r < rows; ++r) {  // the one-hot contract (network.hpp:423-432)
            long long ones = 0;
            for (long long j = 0; j < cols; ++j) {
                const float v = labels[r * cols + j];
                if (v == 1.0f) {
                    ++ones;
                    truth[(size_t)r] = (int)j;
                } else if (v != 0.0f) {
                    throw b2n::Error(B2N_ELABEL, "softmax_cross_entropy: labels must be one-hot; row " + std::to_string(r));
                }
            }
            if (ones != 1)
                throw b2n::Error(B2N_ELABEL, "softmax_cross_entropy: labels must be one-hot; row " + std::to_string(r));
        }
        b2n::OpMem m(device);
        const float* d_p = m.up(predictions, rows * cols);
        const float* d_l = m.up(labels, rows * cols);
        const int* d_t = m.up(truth.data(), rows);
        float* d_g = m.alloc<float>(rows * cols);
        double* d_r = m.alloc<double>(rows);
        b2n::op_xent_kernel<<<b2n::grid_of(rows * cols), 256, 0, m.st>>>(d_p, d_l, d_t, d_g, d_r, rows, (int)cols);
        std::vector<double> rl((size_t)rows);
        m.down(dlogits, (const float*)d_g, rows * cols);
        m.down(rl.data(), (const double*)d_r, rows);
        m.sync();
        double acc = 0.0;
        for (long long r = 0; r < rows; ++r) acc -= rl[(size_t)r];  // the reference's order (network.hpp:433)
        *loss = acc / (double)rows;
    });
}

}  // extern "C"
