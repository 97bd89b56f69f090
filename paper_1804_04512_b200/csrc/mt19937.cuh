// mt19937.cuh -- the reference's Bernoulli draw stream on the device, bit-exact.
//
// The reference samples every binary unit with std::bernoulli_distribution(p)(rng) on a
// std::mt19937 (energy.hpp:53-71, drawn in row-major order from cd_k_update's rng, :137-144, and
// crbm_cd_update's, :330-376). libstdc++ evaluates that draw as
//     u = generate_canonical<double, 53>(rng)  =  rn(w0 + w1 * 2^32) * 2^-64   (w0, w1: two tempered
//         32-bit outputs; u >= 1 -> nextafter(1, 0))              (bits/random.tcc:3349-3381)
//     sample = u < (double)p                                     (bits/random.h bernoulli_distribution)
// so one draw consumes two generator words. Here the caller's generator state (the 624 state
// words + the position libstdc++ keeps, i.e. what `os << rng` prints) lives in device memory and is
// advanced on the device: the step kernels read the same doubles the reference would have drawn,
// the host never runs the generator and nothing of the stream crosses PCIe.
//
// The generator is sequential, so the words are produced by ONE CTA as a wavefront over the
// unrolled sequence X[n] (X[0..623] = the current state array, the k-th output is temper(X[p+k])):
//     X[n] = X[n-227] ^ F(X[n-624], X[n-623])                      (the libstdc++ block twist)
// F is linear over GF(2) in its two words, so expanding X[n-227] twice gives
//     X[n] = X[n-681] ^ F(X[n-624] ^ X[n-851] ^ X[n-1078], X[n-623] ^ X[n-850] ^ X[n-1077])
// whose nearest dependency is 623 words back: 620 words per barrier (4 per thread, 16-byte smem
// vectors) instead of 227 (three bootstrap stages of the plain recurrence cover n < 1080). The raw
// words go to a scratch buffer; a grid-wide second kernel tempers and converts them (two words -> one
// double). The generator always completes whole 624-word blocks, so the final state equals
// libstdc++'s (_M_x, _M_p) after the same draws. One CTA is issue/latency bound at ~1 barrier per
// 620 words; the step kernels never wait for it where it runs on the copy stream ahead of them.
#pragma once
#include "runtime.cuh"

namespace b2n {

constexpr int kMtN = 624;

__device__ __forceinline__ uint32_t mt_twist(uint32_t a, uint32_t b) {
    return (((a & 0x80000000u) | (b & 0x7fffffffu)) >> 1) ^ ((b & 1u) ? 0x9908b0dfu : 0u);
}
__host__ __device__ __forceinline__ uint32_t mt_temper(uint32_t z) {
    z ^= z >> 11;
    z ^= (z << 7) & 0x9d2c5680u;
    z ^= (z << 15) & 0xefc60000u;
    z ^= z >> 18;
    return z;
}
// generate_canonical<double, 53> of two consecutive tempered words
__host__ __device__ __forceinline__ double mt_canonical(uint32_t w0, uint32_t w1) {
    const double s = (double)w1 * 4294967296.0 + (double)w0;  // the product is exact: one rounding, fma or not
    const double u = s * 5.42101086242752217003726400434970855712890625e-20;  // 2^-64, exact
    return u >= 1.0 ? 0.99999999999999988897769753748434595763683319091796875 : u;
}

// st = [624 state words, position p]. Writes the raw (untempered) words X[0 .. end) of the unrolled
// sequence to wbuf (end = the last whole block the draws reach), p to meta[0], and leaves st at
// libstdc++'s state after 2n draws. Four consecutive words per thread (all smem traffic 16-byte
// vectors): the ring is mapped twice (slot s and s + R hold the same word) so every read of a
// 4-word group is an immediate offset from one register, never a wrapped index.
constexpr int kMtR = 2048;         // ring words (> 1080 behind + 620 ahead)
constexpr int kMtW = 620;          // main-wavefront width: 155 threads x 4 words, <= 623
static __global__ void __launch_bounds__(256, 1) mt_words_kernel(uint32_t* st, uint32_t* __restrict__ wbuf,
                                                                 long long* meta, long long n) {
    pdl_wait();
    __shared__ __align__(16) uint32_t ring[2 * kMtR];
    constexpr int M = kMtR - 1;
    const int t = threadIdx.x;
    const long long p = st[kMtN];
    const long long E = p + 2 * n;
    const long long blk = n > 0 ? (E - 1) / kMtN : 0;
    const long long end = kMtN * (blk + 1);
    for (int i = t; i < kMtN; i += blockDim.x) {
        const uint32_t x = st[i];
        ring[i] = x;
        ring[i + kMtR] = x;
        wbuf[i] = x;
    }
    if (t == 0) meta[0] = p;
    __syncthreads();
    // bootstrap with the plain recurrence X[q] = X[q-227] ^ T(X[q-624], X[q-623]): [624, 851),
    // [851, 1078), [1078, 1080) -- after which the main wavefront starts 4-word aligned
    const int bs[4] = {624, 851, 1078, 1080};
    for (int k = 0; k < 3; ++k) {
        const int q = bs[k] + t;
        if (q < bs[k + 1] && q < end) {
            const uint32_t v = ring[(q - 227) & M] ^ mt_twist(ring[(q - 624) & M], ring[(q - 623) & M]);
            ring[q & M] = v;
            ring[(q & M) + kMtR] = v;
            wbuf[q] = v;
        }
        __syncthreads();
    }
    // X[q] = X[q-681] ^ T(c[q-624], c[q-623]),  c[j] = X[j] ^ X[j-227] ^ X[j-454]
    // The loop is bound by shared-memory bandwidth + one barrier round trip per chunk (measured
    // ~200 clk for load -> compute -> store -> barrier alone): each group is read with the narrowest
    // aligned vectors that cover exactly its words, and X[q-620] is this thread's own word of the
    // previous chunk (a register).
    if (t < 160) {  // 5 warps: lanes 0..154 carry the wavefront, all 160 take the named barrier
        uint4* wb = reinterpret_cast<uint4*>(wbuf);
        int A = (1080 + 4 * t) & M;  // ring slot of this thread's first word
        uint32_t own0 = t < kMtW / 4 ? ring[(1080 + 4 * t - 620) & M] : 0u;  // X[q - 620] (lanes that compute)
        for (long long s = 1080; s < end; s += kMtW) {
            const long long q = s + 4 * t;
            if (t < kMtW / 4 && q < end) {
                const uint32_t* r = ring + A + kMtR;  // r[-d] = X[q - d]
                const uint4 a0 = *reinterpret_cast<const uint4*>(r - 624);        // X[q-624 .. q-621]
                const uint32_t b0 = r[-851];                                     // X[q-851]
                const uint2 b1 = *reinterpret_cast<const uint2*>(r - 850);        // X[q-850], X[q-849]
                const uint2 b2 = *reinterpret_cast<const uint2*>(r - 848);        // X[q-848], X[q-847]
                const uint2 d0 = *reinterpret_cast<const uint2*>(r - 1078);       // X[q-1078], X[q-1077]
                const uint2 d1 = *reinterpret_cast<const uint2*>(r - 1076);       // X[q-1076], X[q-1075]
                const uint32_t d2 = r[-1074];                                    // X[q-1074]
                const uint32_t e0 = r[-681];                                     // X[q-681]
                const uint2 e1 = *reinterpret_cast<const uint2*>(r - 680);        // X[q-680], X[q-679]
                const uint32_t e2 = r[-678];                                     // X[q-678]
                const uint32_t c0 = a0.x ^ b0 ^ d0.x, c1 = a0.y ^ b1.x ^ d0.y, c2 = a0.z ^ b1.y ^ d1.x,
                               c3 = a0.w ^ b2.x ^ d1.y, c4 = own0 ^ b2.y ^ d2;
                uint4 v;
                v.x = e0 ^ mt_twist(c0, c1);
                v.y = e1.x ^ mt_twist(c1, c2);
                v.z = e1.y ^ mt_twist(c2, c3);
                v.w = e2 ^ mt_twist(c3, c4);
                own0 = v.x;
                *reinterpret_cast<uint4*>(ring + A) = v;
                *reinterpret_cast<uint4*>(ring + A + kMtR) = v;
                wb[q >> 2] = v;
            }
            A = (A + kMtW) & M;
            asm volatile("bar.sync 1, 160;" ::: "memory");
        }
    }
    __syncthreads();
    for (int i = t; i < kMtN; i += blockDim.x) st[i] = ring[(kMtN * blk + i) & M];
    if (t == 0) st[kMtN] = (uint32_t)(E - kMtN * blk);
}

// out[j] = generate_canonical<double, 53> of the words X[p + 2j], X[p + 2j + 1]
static __global__ void __launch_bounds__(256) mt_canonical_kernel(const uint32_t* __restrict__ wbuf,
                                                                  const long long* __restrict__ meta,
                                                                  double* __restrict__ out, long long n) {
    pdl_wait();
    const uint32_t* w = wbuf + meta[0];
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x)
        out[j] = mt_canonical(mt_temper(w[2 * j]), mt_temper(w[2 * j + 1]));
}

// A std::mt19937 whose state lives on the device. load() takes the caller's state (625 words:
// _M_x[624], _M_p) -- uploaded only when it differs from the last state this object handed back,
// so a caller that threads one generator through consecutive steps pays no copy; draw() appends
// n doubles of the stream to a device buffer; store() returns the advanced state to the caller.
class DevRng {
  public:
    void load(const uint32_t* s, cudaStream_t st) {
        if (!st_.p) {
            st_.alloc(kMtN * 4 + 64);
            host_.alloc(kMtN * 4 + 64);
        }
        if (valid_ && !dirty_ && std::memcmp(s, shadow_, sizeof(shadow_)) == 0) return;
        if (s[kMtN] > (uint32_t)kMtN) throw Error(B2N_EPARAM, "mt19937 state: position must be <= 624");
        std::memcpy(host_.p, s, sizeof(shadow_));
        B2N_CUDA(cudaMemcpyAsync(st_.p, host_.p, sizeof(shadow_), cudaMemcpyHostToDevice, st));
        B2N_CUDA(cudaStreamSynchronize(st));  // host_ is reused by store()
        std::memcpy(shadow_, s, sizeof(shadow_));
        valid_ = true;
    }
    void draw(double* out, long long n, cudaStream_t st) {
        if (!valid_) throw Error(B2N_EPARAM, "device generator used before its state was set");
        if (n <= 0) return;
        const size_t words = (size_t)(2 * n + 2 * kMtN + 16);  // >= the whole blocks the draws reach
        if (wbuf_.bytes < words * 4) {
            B2N_CUDA(cudaStreamSynchronize(st));  // a pending draw may still read the old buffer
            wbuf_.alloc(words * 4);
        }
        launch_ex(mt_words_kernel, dim3(1), dim3(256), 0, st, 1u, st_.as<uint32_t>(), wbuf_.as<uint32_t>(),
                  reinterpret_cast<long long*>(st_.as<uint8_t>() + kMtN * 4 + 16), n);
        const int g = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
        launch_ex(mt_canonical_kernel, dim3(g), dim3(256), 0, st, 1u, (const uint32_t*)wbuf_.as<uint32_t>(),
                  (const long long*)(st_.as<uint8_t>() + kMtN * 4 + 16), out, n);
        dirty_ = true;
    }
    // copy the device state back (synchronises st); s may be null to just refresh the shadow
    void store(uint32_t* s, cudaStream_t st) {
        if (!valid_) throw Error(B2N_EPARAM, "device generator read before its state was set");
        if (dirty_) {
            B2N_CUDA(cudaMemcpyAsync(host_.p, st_.p, sizeof(shadow_), cudaMemcpyDeviceToHost, st));
            spin_sync(st);
            std::memcpy(shadow_, host_.p, sizeof(shadow_));
            dirty_ = false;
        }
        if (s) std::memcpy(s, shadow_, sizeof(shadow_));
    }
    bool valid() const { return valid_; }

  private:
    DevMem st_;    // [624 words, p] + the draw's starting position (read by the canonical kernel)
    DevMem wbuf_;  // the raw words of the draw in flight
    HostPinned host_;
    uint32_t shadow_[kMtN + 1];
    bool valid_ = false;
    bool dirty_ = false;
};

}  // namespace b2n
