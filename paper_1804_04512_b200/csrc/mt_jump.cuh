// mt_jump.cuh -- jump-ahead for the device std::mt19937 (mt19937.cuh), so consecutive steps' draws are
// generated concurrently instead of one after the other.
//
// The generator's 624-word window W_i = (X[i], .., X[i+623]) of the unrolled sequence evolves linearly
// over GF(2): W_{i+1} = A W_i. Its characteristic polynomial phi (degree 19937) is found once by
// Berlekamp-Massey on one bit of the output; then A^m W_0 = g(A) W_0 with g = x^m mod phi, i.e. the
// XOR of the windows W_t for the t where g has a 1 -- windows of the first 20,560 words of the
// sequence, which a short "prefix" run of the generator produces. This is exact on every bit that
// influences the future (the low 31 bits of a window's first word never do, since the twist reads
// only that word's top bit), so the jump lands one word early, m = J - 1, and the block X[J .. J+623]
// follows exactly: its first 623 words are W_{J-1}[1..623] and its last is one recurrence step.
// (Checked on the host against direct generation before this was written; tests/test_gpu_rng.py
// checks every streamed draw and the final state against the host generator.)
#pragma once
#include <map>
#include <vector>

#include "runtime.cuh"

namespace b2n {

constexpr int kMtN = 624;                         // std::mt19937 state words
constexpr int kMtL = 19937;                       // degree of the characteristic polynomial
constexpr int kMtPrefix = 20560;                  // words of the sequence the jump XORs windows of
constexpr int kMtJumpCtas = (kMtL + 622) / 623;   // 33: CTA c owns the terms t in [623 c, 623 c + 623)

namespace mtpoly {
using Bits = std::vector<uint64_t>;
inline int bit(const Bits& a, long i) { return (int)((a[(size_t)(i >> 6)] >> (i & 63)) & 1ull); }
inline void flip(Bits& a, long i) { a[(size_t)(i >> 6)] ^= 1ull << (i & 63); }
// a ^= b << sh (bit shift), a sized to hold the result
inline void xor_shifted(Bits& a, const Bits& b, long sh) {
    const long ws = sh >> 6, bs = sh & 63;
    for (size_t i = 0; i < b.size(); ++i) {
        if (!b[i]) continue;
        const size_t j = i + (size_t)ws;
        if (j < a.size()) a[j] ^= b[i] << bs;
        if (bs && j + 1 < a.size()) a[j + 1] ^= b[i] >> (64 - bs);
    }
}

// phi(x), bit i = coefficient of x^i (degree kMtL): Berlekamp-Massey over bit 5 of the raw words of
// the sequence from std::mt19937's default seed (any non-degenerate bit / seed gives the same phi)
inline const Bits& charpoly() {
    static const Bits phi = [] {
        const long N = 2L * kMtL + 128;
        std::vector<uint32_t> X((size_t)(N + kMtN));
        X[0] = 5489u;
        for (int i = 1; i < kMtN; ++i) X[(size_t)i] = 1812433253u * (X[(size_t)i - 1] ^ (X[(size_t)i - 1] >> 30)) + (uint32_t)i;
        for (size_t n = kMtN; n < X.size(); ++n) {
            const uint32_t y = (X[n - 624] & 0x80000000u) | (X[n - 623] & 0x7fffffffu);
            X[n] = X[n - 227] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        const size_t W = (size_t)(N / 64 + 2);
        Bits rev(W, 0);  // rev bit k = s[N - 1 - k], s[n] = bit 5 of X[n + 624]
        for (long n = 0; n < N; ++n)
            if ((X[(size_t)(n + kMtN)] >> 5) & 1u) flip(rev, N - 1 - n);
        auto rev_word = [&](long pos) -> uint64_t {  // bits rev[pos .. pos + 64)
            const size_t w = (size_t)(pos >> 6);
            const int b = (int)(pos & 63);
            uint64_t lo = w < W ? rev[w] : 0, hi = w + 1 < W ? rev[w + 1] : 0;
            return b ? (lo >> b) | (hi << (64 - b)) : lo;
        };
        Bits C(W, 0), B(W, 0), T;
        C[0] = B[0] = 1;
        long L = 0, m = 1;
        for (long n = 0; n < N; ++n) {
            // d = s[n] + sum_{i=1..L} C_i s[n-i];  s[n-i] = rev[N-1-n+i]
            uint64_t acc = (uint64_t)bit(rev, N - 1 - n);
            const long base = N - 1 - n;
            for (long i = 0; i <= L; i += 64) {
                uint64_t c = C[(size_t)(i >> 6)];
                if (i == 0) c &= ~1ull;  // C_0 is s[n] itself, counted above
                const long hi = L - i;   // keep bits i .. L
                if (hi < 63) c &= (hi < 0) ? 0 : ((2ull << hi) - 1);
                acc ^= c & rev_word(base + i);
            }
            if (!(__builtin_popcountll(acc) & 1)) {
                ++m;
                continue;
            }
            T = C;
            xor_shifted(C, B, m);
            if (2 * L <= n) {
                L = n + 1 - L;
                B = T;
                m = 1;
            } else {
                ++m;
            }
        }
        if (L != kMtL) throw Error(B2N_EINTERNAL, "mt19937 jump: characteristic polynomial degree " + std::to_string(L));
        Bits phi((size_t)(kMtL / 64 + 1), 0);  // reciprocal of the connection polynomial
        for (long i = 0; i <= L; ++i)
            if (bit(C, i)) flip(phi, L - i);
        return phi;
    }();
    return phi;
}

// the sorted exponents t (< kMtL) where x^m mod phi has a 1
inline std::vector<int> jump_terms(long long m) {
    const Bits& phi = charpoly();
    const size_t W2 = (size_t)(2 * kMtL / 64 + 2);
    Bits g(W2, 0), t;
    g[0] = 1;
    auto reduce = [&](Bits& a) {
        for (long i = 2L * kMtL; i >= kMtL; --i)
            if ((size_t)(i >> 6) < a.size() && bit(a, i)) xor_shifted(a, phi, i - kMtL);
    };
    int top = 62;
    while (top >= 0 && !((m >> top) & 1)) --top;
    for (int b = top; b >= 0; --b) {
        t.assign(W2, 0);  // square: spread the bits
        for (long i = 0; i < kMtL; ++i)
            if (bit(g, i)) flip(t, 2 * i);
        g.swap(t);
        if ((m >> b) & 1) {  // times x
            t.assign(W2, 0);
            xor_shifted(t, g, 1);
            g.swap(t);
        }
        reduce(g);
    }
    std::vector<int> terms;
    for (long i = 0; i < kMtL; ++i)
        if (bit(g, i)) terms.push_back((int)i);
    return terms;
}
}  // namespace mtpoly

// CTA c: partial window = XOR over its terms t of X[t .. t + 623] (the prefix staged in smem)
static __global__ void __launch_bounds__(640) mt_jump_kernel(const uint32_t* __restrict__ X, const int* __restrict__ terms,
                                                            const int* __restrict__ off, uint32_t* __restrict__ part) {
    pdl_wait();
    __shared__ uint32_t sx[2 * 624];
    const int c = blockIdx.x, base = 623 * c;
    for (int i = threadIdx.x; i < 2 * 624; i += blockDim.x) sx[i] = base + i < kMtPrefix ? X[base + i] : 0u;
    __syncthreads();
    if (threadIdx.x < kMtN) {
        uint32_t acc = 0;
        for (int e = off[c]; e < off[c + 1]; ++e) acc ^= sx[terms[e] - base + threadIdx.x];
        part[c * kMtN + threadIdx.x] = acc;
    }
}

// W = XOR of the partial windows = (X[J-1] top bit, X[J .. J+622]); the block X[J .. J+623] + position
static __global__ void __launch_bounds__(640) mt_jump_finish_kernel(const uint32_t* __restrict__ part, uint32_t* st_next,
                                                                   unsigned p_next) {
    pdl_wait();
    __shared__ uint32_t w[kMtN];
    if (threadIdx.x < kMtN) {
        uint32_t acc = 0;
        for (int c = 0; c < kMtJumpCtas; ++c) acc ^= part[c * kMtN + threadIdx.x];
        w[threadIdx.x] = acc;
    }
    __syncthreads();
    if (threadIdx.x < kMtN - 1) st_next[threadIdx.x] = w[threadIdx.x + 1];
    if (threadIdx.x == 0) {
        const uint32_t y = (w[0] & 0x80000000u) | (w[1] & 0x7fffffffu);  // X[J+623] = X[J+396] ^ T(X[J-1], X[J])
        st_next[kMtN - 1] = w[397] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        st_next[kMtN] = p_next;
    }
}

}  // namespace b2n
