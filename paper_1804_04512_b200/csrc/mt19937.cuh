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
#include "mt_jump.cuh"
#include "runtime.cuh"

namespace b2n {


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
// st_in -> st_out may alias (all of st_in is read first); st_out null: the state is not written back.
// prefix != 0: just the first kMtPrefix words of the sequence from st_in's block (for mt_jump.cuh).
static __global__ void __launch_bounds__(256, 1) mt_words_kernel(const uint32_t* st_in, uint32_t* st_out,
                                                                 uint32_t* __restrict__ wbuf, long long* meta,
                                                                 long long n, int prefix) {
    pdl_wait();
    __shared__ __align__(16) uint32_t ring[2 * kMtR];
    constexpr int M = kMtR - 1;
    const int t = threadIdx.x;
    const long long p = prefix ? 0 : st_in[kMtN];
    const long long E = prefix ? kMtPrefix : p + 2 * n;
    const long long blk = E > p ? (E - 1) / kMtN : 0;
    const long long end = kMtN * (blk + 1);
    for (int i = t; i < kMtN; i += blockDim.x) {
        const uint32_t x = st_in[i];
        ring[i] = x;
        ring[i + kMtR] = x;
        wbuf[i] = x;
    }
    if (t == 0 && !prefix) meta[0] = p;
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
    if (!st_out) return;
    for (int i = t; i < kMtN; i += blockDim.x) st_out[i] = ring[(kMtN * blk + i) & M];
    if (t == 0) st_out[kMtN] = (uint32_t)(E - kMtN * blk);
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
        host_pending_ = false;
        B2N_CUDA(cudaMemcpyAsync(st_.p, host_.p, sizeof(shadow_), cudaMemcpyHostToDevice, st));
        B2N_CUDA(cudaStreamSynchronize(st));  // host_ is reused by store()
        std::memcpy(shadow_, s, sizeof(shadow_));
        valid_ = true;
        p_ = s[kMtN];
    }
    void draw(double* out, long long n, cudaStream_t st) {
        if (!valid_) throw Error(B2N_EPARAM, "device generator used before its state was set");
        if (n <= 0) return;
        const size_t words = (size_t)(2 * n + 2 * kMtN + 16);  // >= the whole blocks the draws reach
        if (wbuf_.bytes < words * 4) {
            B2N_CUDA(cudaStreamSynchronize(st));  // a pending draw may still read the old buffer
            wbuf_.alloc(words * 4);
        }
        launch_ex(mt_words_kernel, dim3(1), dim3(256), 0, st, 1u, (const uint32_t*)st_.as<uint32_t>(), st_.as<uint32_t>(),
                  wbuf_.as<uint32_t>(), reinterpret_cast<long long*>(st_.as<uint8_t>() + kMtN * 4 + 16), n, 0);
        const int g = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
        launch_ex(mt_canonical_kernel, dim3(g), dim3(256), 0, st, 1u, (const uint32_t*)wbuf_.as<uint32_t>(),
                  (const long long*)(st_.as<uint8_t>() + kMtN * 4 + 16), out, n);
        dirty_ = true;
        host_pending_ = false;  // host_ (if a stream left it) is older than this draw
        p_ = advance(p_, n);
    }

    // ---- consecutive draws of n doubles each, pipelined (train_stream): a chain stream computes every
    // step's starting state by jump-ahead (prefix words -> XOR of windows -> block), kGen generator
    // streams produce the steps' draws concurrently. Bit-identical to draw() called step after step.
    void stream_begin(long long n, cudaStream_t base, int gens = 3) {
        if (!valid_) throw Error(B2N_EPARAM, "device generator used before its state was set");
        host_pending_ = false;
        if (!sm_.slots.p) {
            sm_.slots.alloc((size_t)kSlots * kSlotBytes);
            sm_.prefix.alloc((size_t)(kMtN * 34) * 4);
            sm_.part.alloc((size_t)kMtJumpCtas * kMtN * 4);
            for (int g = 0; g < kGen; ++g) {
                sm_.gmeta[g].alloc(64);
                B2N_CUDA(cudaStreamCreateWithFlags(&sm_.gen[g], cudaStreamNonBlocking));
            }  // (one generator CTA per stream; kGen streams exist, sm_.ngen of them are used)
            B2N_CUDA(cudaStreamCreateWithFlags(&sm_.chain, cudaStreamNonBlocking));
            for (int k = 0; k < kSlots; ++k) {
                B2N_CUDA(cudaEventCreateWithFlags(&sm_.ev_state[k], cudaEventDisableTiming));
                B2N_CUDA(cudaEventCreateWithFlags(&sm_.ev_gen[k], cudaEventDisableTiming));
            }
            B2N_CUDA(cudaEventCreateWithFlags(&sm_.ev_base, cudaEventDisableTiming));
        }
        sm_.ngen = std::max(1, std::min(gens, kGen));
        const size_t words = (size_t)(2 * n + 2 * kMtN + 16);
        for (int g = 0; g < sm_.ngen; ++g)
            if (sm_.gwbuf[g].bytes < words * 4) {
                B2N_CUDA(cudaDeviceSynchronize());
                sm_.gwbuf[g].alloc(words * 4);
            }
        sm_.n = n;
        sm_.p.assign(1, p_);
        // every jump distance this step size can need (a step starting at position p covers
        // (p + 2n - 1) / 624 blocks: two or three values over p in [0, 624]), prepared here so no
        // later step of this or a following stream stops for the host-side polynomial work
        if (n > 0)
            for (long long blk = (2 * n - 1) / kMtN; blk <= (2 * n + kMtN - 1) / kMtN; ++blk)
                if (blk > 0) jump_poly(kMtN * blk - 1);
        B2N_CUDA(cudaEventRecord(sm_.ev_base, base));
        B2N_CUDA(cudaStreamWaitEvent(sm_.chain, sm_.ev_base, 0));
        for (int g = 0; g < sm_.ngen; ++g) B2N_CUDA(cudaStreamWaitEvent(sm_.gen[g], sm_.ev_base, 0));
        B2N_CUDA(cudaMemcpyAsync(slot(0), st_.p, (kMtN + 1) * 4, cudaMemcpyDeviceToDevice, sm_.chain));
        B2N_CUDA(cudaEventRecord(sm_.ev_state[0], sm_.chain));
        for (int k = 0; k < kSlots; ++k) B2N_CUDA(cudaEventRecord(sm_.ev_gen[k], sm_.chain));
    }
    // step i of `steps`: its draws into out once `out_free` has fired; `out_ready` is recorded after them
    void stream_step(int i, int steps, double* out, cudaEvent_t out_free, cudaEvent_t out_ready) {
        const long long n = sm_.n;
        const int si = i % kSlots, g = i % sm_.ngen;
        cudaStream_t gs = sm_.gen[g];
        B2N_CUDA(cudaStreamWaitEvent(gs, sm_.ev_state[si], 0));
        B2N_CUDA(cudaStreamWaitEvent(gs, out_free, 0));
        uint32_t* fin = i == steps - 1 ? st_.as<uint32_t>() : nullptr;  // the last step hands the state back
        long long* meta = sm_.gmeta[g].as<long long>();
        launch_ex(mt_words_kernel, dim3(1), dim3(256), 0, gs, 1u, (const uint32_t*)slot(si), fin,
                  sm_.gwbuf[g].as<uint32_t>(), meta, n, 0);
        const int grid = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
        launch_ex(mt_canonical_kernel, dim3(grid), dim3(256), 0, gs, 1u, (const uint32_t*)sm_.gwbuf[g].as<uint32_t>(),
                  (const long long*)meta, out, n);
        B2N_CUDA(cudaEventRecord(out_ready, gs));
        B2N_CUDA(cudaEventRecord(sm_.ev_gen[si], gs));
        const long long pi = sm_.p.back(), E = pi + 2 * n, blk = (E - 1) / kMtN;
        sm_.p.push_back(E - kMtN * blk);
        sm_.p_host[(size_t)(i + 1) % kSlots] = (unsigned)sm_.p.back();
        if (i + 1 >= steps) return;
        // the next step's block: jump blk blocks ahead from this step's block (slot free once its last
        // generator is done)
        const int sn = (i + 1) % kSlots;
        B2N_CUDA(cudaStreamWaitEvent(sm_.chain, sm_.ev_gen[sn], 0));
        if (blk == 0) {  // the draws stayed inside the block: same block, new position
            B2N_CUDA(cudaMemcpyAsync(slot(sn), slot(si), kMtN * 4, cudaMemcpyDeviceToDevice, sm_.chain));
            B2N_CUDA(cudaMemcpyAsync(slot(sn) + kMtN, &sm_.p_host[(size_t)(i + 1) % kSlots], 4, cudaMemcpyHostToDevice,
                                     sm_.chain));
            B2N_CUDA(cudaEventRecord(sm_.ev_state[sn], sm_.chain));
            return;
        }
        const JumpPoly& jp = jump_poly(kMtN * blk - 1);
        launch_ex(mt_words_kernel, dim3(1), dim3(256), 0, sm_.chain, 1u, (const uint32_t*)slot(si), (uint32_t*)nullptr,
                  sm_.prefix.as<uint32_t>(), (long long*)nullptr, 0LL, 1);
        launch_ex(mt_jump_kernel, dim3(kMtJumpCtas), dim3(640), 0, sm_.chain, 1u, (const uint32_t*)sm_.prefix.as<uint32_t>(),
                  (const int*)jp.terms.as<int>(), (const int*)jp.off.as<int>(), sm_.part.as<uint32_t>());
        launch_ex(mt_jump_finish_kernel, dim3(1), dim3(640), 0, sm_.chain, 1u, (const uint32_t*)sm_.part.as<uint32_t>(),
                  slot(sn), (unsigned)sm_.p.back());
        B2N_CUDA(cudaEventRecord(sm_.ev_state[sn], sm_.chain));
    }
    // base waits for the whole stream; the generator state is the last step's
    void stream_end(int steps, cudaStream_t base) {
        B2N_CUDA(cudaEventRecord(sm_.ev_base, sm_.chain));
        B2N_CUDA(cudaStreamWaitEvent(base, sm_.ev_base, 0));
        for (int g = 0; g < sm_.ngen; ++g) {
            B2N_CUDA(cudaEventRecord(sm_.ev_base, sm_.gen[g]));
            B2N_CUDA(cudaStreamWaitEvent(base, sm_.ev_base, 0));
        }
        if (steps > 0) {
            dirty_ = true;
            p_ = sm_.p[(size_t)steps];
            // the advanced state comes back with the stream (the caller's sync covers it): store() then
            // needs no round trip of its own
            B2N_CUDA(cudaMemcpyAsync(host_.p, st_.p, sizeof(shadow_), cudaMemcpyDeviceToHost, base));
            host_pending_ = true;
        }
    }
    // copy the device state back (synchronises st); s may be null to just refresh the shadow
    void store(uint32_t* s, cudaStream_t st) {
        if (!valid_) throw Error(B2N_EPARAM, "device generator read before its state was set");
        if (dirty_) {
            if (!host_pending_) B2N_CUDA(cudaMemcpyAsync(host_.p, st_.p, sizeof(shadow_), cudaMemcpyDeviceToHost, st));
            spin_sync(st);
            host_pending_ = false;
            std::memcpy(shadow_, host_.p, sizeof(shadow_));
            dirty_ = false;
            if (shadow_[kMtN] != (uint32_t)p_) throw Error(B2N_EINTERNAL, "device generator position out of sync");
        }
        if (s) std::memcpy(s, shadow_, sizeof(shadow_));
    }
    bool valid() const { return valid_; }

    ~DevRng() {
        if (sm_.chain) cudaStreamDestroy(sm_.chain);
        for (int g = 0; g < kGen; ++g)
            if (sm_.gen[g]) cudaStreamDestroy(sm_.gen[g]);
        for (int k = 0; k < kSlots; ++k) {
            if (sm_.ev_state[k]) cudaEventDestroy(sm_.ev_state[k]);
            if (sm_.ev_gen[k]) cudaEventDestroy(sm_.ev_gen[k]);
        }
        if (sm_.ev_base) cudaEventDestroy(sm_.ev_base);
    }

  private:
    static constexpr int kSlots = 40, kGen = 32, kSlotBytes = 4096;
    struct JumpPoly {
        DevMem terms, off;
    };
    // x^m mod phi as per-CTA term lists (host Berlekamp-Massey / powmod once per m, mt_jump.cuh)
    const JumpPoly& jump_poly(long long m) {
        auto it = jumps_.find(m);
        if (it != jumps_.end()) return *it->second;
        const std::vector<int> t = mtpoly::jump_terms(m);
        std::vector<int> off(kMtJumpCtas + 1, 0);
        for (int v : t) ++off[(size_t)(v / 623 + 1)];
        for (int c = 0; c < kMtJumpCtas; ++c) off[(size_t)c + 1] += off[(size_t)c];
        auto jp = std::make_unique<JumpPoly>();
        jp->terms.alloc(std::max<size_t>(t.size(), 1) * 4);
        jp->off.alloc(off.size() * 4);
        B2N_CUDA(cudaMemcpy(jp->terms.p, t.data(), t.size() * 4, cudaMemcpyHostToDevice));
        B2N_CUDA(cudaMemcpy(jp->off.p, off.data(), off.size() * 4, cudaMemcpyHostToDevice));
        return *(jumps_[m] = std::move(jp));
    }
    uint32_t* slot(int k) { return reinterpret_cast<uint32_t*>(sm_.slots.as<uint8_t>() + (size_t)k * kSlotBytes); }
    static long long advance(long long p, long long n) {
        const long long E = p + 2 * n, blk = n > 0 ? (E - 1) / kMtN : 0;
        return E - kMtN * blk;
    }
    struct StreamRes {
        DevMem slots, prefix, part, gwbuf[kGen], gmeta[kGen];
        cudaStream_t chain = nullptr, gen[kGen] = {};
        cudaEvent_t ev_state[kSlots] = {}, ev_gen[kSlots] = {}, ev_base = nullptr;
        long long n = 0;
        int ngen = 3;
        std::vector<long long> p;  // position before each step of the stream in flight
        unsigned p_host[kSlots] = {};  // pinned-free staging of a position for the blk == 0 copy
    } sm_;
    std::map<long long, std::unique_ptr<JumpPoly>> jumps_;
    long long p_ = 0;  // the state's position, tracked on the host
    DevMem st_;    // [624 words, p] + the draw's starting position (read by the canonical kernel)
    DevMem wbuf_;  // the raw words of the draw in flight
    HostPinned host_;
    uint32_t shadow_[kMtN + 1];
    bool valid_ = false;
    bool dirty_ = false;
    bool host_pending_ = false;  // host_ receives the state at the end of a stream (stream_end)
};

}  // namespace b2n
