// rbm_fused.cuh -- one CD-1 step of a binary RBM (cd_k_update, energy.hpp:131-171) as ONE persistent
// kernel: the four dependent products of the step are separated by grid barriers instead of kernel
// boundaries, and every CTA keeps a fixed piece of the problem.
//
// 64 CTAs = 8 hidden tiles j (64 units) x 8 visible slices s (128 units), clusters of the 8 slices of
// a hidden tile (a B200 holds 15 co-resident clusters of 8 at this shared-memory size, measured). W_aug is (H+1) x ldw with bh in column V and bv in row H (rbm.cuh).
//   phase 1  h0 = sigmoid(v0 W^T + bh), hs = (u < h0)   CTA (j,s): v0[:, s] . W[j, s]^T over its 128
//            visible units (K), partials of the 8 slices summed through distributed shared memory
//   phase 2  v1 = sigmoid(hs W + bv), recon rows        CTA (j,s): hs[:, j] . W[j, s] (K = 32 hidden);
//            the 8 hidden-tile partials meet in an L2 workspace, each CTA finishes 16 batch rows of its
//            slice: sigmoid, (v0 - v1)^2 row partials
//   phase 3  -h1 = -sigmoid(v1 W^T + bh)                 as phase 1
//   phase 4  W_aug[j, s] += lr/B * (Hcat^T Vcat)^T       K = 2B over [h0; -h1] x [v0; v1] with the +-1 /
//            ones columns: dW, dbh and dbv of energy.hpp:148-169 in one product, written by the owner
// 3xTF32 everywhere (tcgen05.mma kind::tf32; the TMA-landed tile is the hi part, lo split by all threads).
// Reductions are in fixed order (deterministic); the grid barrier is a generation counter in global
// memory (all 128 CTAs are co-resident: one per SM).
#pragma once
#include "gemm_tc.cuh"
#include "runtime.cuh"

namespace b2n {

constexpr int kRfThreads = 256;
constexpr int kRfSlices = 8;                  // visible slices = cluster size
constexpr int kRfSliceW = 128;                // visible units per slice
constexpr int kRfTileH = 64;                  // hidden units per tile
constexpr int kRfStage = 64 * 1024;           // operand stage: A hi | B hi | A lo | B lo
constexpr int kRfStages = 3;
constexpr int kRfTileP = 66;                  // padded pitch of the [128][64] reduction tile (8 B aligned rows)
constexpr int kRfSmem = kRfStages * kRfStage + 128 * kRfTileP * 4 + 1024 + 512;

struct RbmFusedParams {
    int B, H, V;
    long long ldw, ldv, ldh, ldhs;
    float* W;          // W_aug
    float* Vcat;       // [v0; v1] (+ ones column V)
    float* Hcat;       // [h0; -h1] (+ +-1 column H)
    float* HS;         // samples
    const double* u;   // uniforms [B][H]
    double* row_part;  // recon partials [slice][cap]
    long long cap;
    float* ws2;        // phase-2 partials [jt tiles][128 rows][8*128 cols]
    float* ws1;        // phase-1/3 partials [jt tiles][8 slices][128 rows][64]
    unsigned* gbar;    // slice barriers: a 64-bit arrival counter per slice, 128 B apart
    unsigned long long* trace;  // bring-up: phase timestamps (clock64) of CTA (0,0) and (7,7), null normally
    float alpha;       // lr / B_global
    int jt;            // hidden tiles
    double* recon_out;  // host-mapped: the step's reconstruction error, written by the last CTA (or null)
    unsigned* done;     // CTAs finished (last-CTA election for recon_out)
    double bg;          // batch_global (the recon divisor, energy.hpp:144)
    // zero-copy inputs (or null): v0 rows (pitch ld_src floats) and the uniforms [B][H] read straight
    // from device-accessible host memory (pinned user buffers) -- no staging copies before the step
    const float* v0_src;
    long long ld_src;
    const double* u_src;
    // train_stream: the staging buffer holding v0_src / u_src is complete once *ready >= ready_val
    // (written by the copy stream after its copies); null otherwise
    const unsigned* ready;
    unsigned ready_val;
    // data-parallel shard / gradient-only step: phase 4 stores the raw sums (Hcat^T Vcat)^T of this
    // shard into G (W_aug layout) and leaves W alone; the update W += lr / B_global * sum_ranks G
    // follows the allreduce (NCCL inside the step graph, or the caller's for b2n_rbm_set_grad_only)
    float* G;
    int grad_only;
    // tf32 lo parts (x - trunc_tf32(x)) of W_aug, Vcat and Hcat, same layouts: written next to every
    // store of the operand, read by TMA as the 3xTF32 correction terms (the 0/1 samples need none)
    float* Wlo;
    float* Vlo;
    float* Hlo;
    const unsigned* v0_inexact;  // per visible slice: nonzero when some v0 of the slice has a tf32 lo part
};

// the step's TMA maps (hi operand, lo companion): K-major operands of phases 1-3, MN-major ones of
// phases 2 and 4
struct alignas(64) RbmMaps {
    CUtensorMap vk, wk, hsk, wmn, vmn, hmn;
    CUtensorMap vk_lo, wk_lo, wmn_lo, vmn_lo, hmn_lo;
};

// slice barrier counters: one monotonically increasing 64-bit arrival count per slice, 128 B apart
__device__ __forceinline__ unsigned long long* sbar_of(const RbmFusedParams& p, int s) {
    return reinterpret_cast<unsigned long long*>(p.gbar) + 16 * s;
}

// barrier over the nblocks CTAs that share the arrival counter: one release-add (cumulative over the
// CTA's writes, ordered by the preceding bar.sync), then acquire-polls until the count reaches the end
// of this barrier instance -- (old / nblocks + 1) * nblocks, so no generation word has to be read
// first and no reset is needed between launches. Generic-proxy writes are fenced for the async proxy
// (later TMA reads) on both sides.
__device__ __forceinline__ void rf_grid_sync(unsigned long long* ctr, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        unsigned long long old, v;
        asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(ctr) : "memory");
        const unsigned long long target = (old / nblocks + 1) * nblocks;
        unsigned long long spins = 0;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
            if (v >= target) break;
            // all CTAs are co-resident (checked on the host); the watchdog turns a broken invariant into
            // a launch error instead of a hung GPU
            if (++spins > 64) __nanosleep(32);
            if (spins > (1ull << 26)) __trap();
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();
}

// one 3xTF32 product of this phase into TMEM columns [0, N): nkb K-blocks of 32, operands by TMA into a
// ring of ns stages carved for this phase, with this phase's own full / empty barriers (fresh parity).
// Every operand arrives PRE-SPLIT: its tf32 lo part (x - trunc_tf32(x)) lives in a companion array
// written by the producer of the operand (the phase epilogues, the v0 staging, the W update), so the
// loop is a pure TMA -> MMA pipeline: thread 0 streams the K-blocks as slots drain, warp 1 issues the
// MMAs, nobody else touches the ring (no per-block split pass, no per-block CTA barrier).
// load(kb, a_hi, b_hi, b_lo, a_lo, bar) issues the boxes of K-block kb (a_lo == null for the K-blocks
// before lo_from, whose A is exact in tf32: the 0/1 samples, binary v0); tph = running TMEM-barrier phase.
template <class Load>
__device__ __forceinline__ void rf_product(uint8_t* ring, uint64_t* full, uint64_t* empty, uint64_t* tbar, int& tph,
                                           int ns, int nkb, int a_bytes, int b_bytes, int lo_from, bool a_mn,
                                           bool b_mn, uint32_t idesc, uint32_t idesc2, Load load) {
    // stage = A hi | B hi | B lo | A lo: B hi and B lo are adjacent along N, so ONE MMA with N doubled
    // (idesc2) computes a_hi.b_hi into columns [0, N) and a_hi.b_lo into [N, 2N); a second MMA adds
    // a_lo.b_hi into [0, N). rf_tmem_to_smem folds the halves.
    const int warp = threadIdx.x >> 5;
    const int sb = 2 * (a_bytes + b_bytes);
    auto slot = [&](int g) { return ring + (g % ns) * sb; };
    if (threadIdx.x == 0) {
        for (int i = 0; i < nkb; ++i) {
            const int st = i % ns;
            if (i >= ns) mbar_wait(&empty[st], ((i / ns) - 1) & 1);
            uint8_t* d = slot(i);
            const bool lo = i >= lo_from;
            mbar_arrive_expect_tx(&full[st], (uint32_t)(a_bytes + 2 * b_bytes + (lo ? a_bytes : 0)));
            load(i, d, d + a_bytes, d + a_bytes + b_bytes, lo ? d + a_bytes + 2 * b_bytes : nullptr, &full[st]);
        }
    } else if (warp == 1) {
        const uint64_t a_lo_off = (uint64_t)((a_bytes + 2 * b_bytes) >> 4);
        for (int i = 0; i < nkb; ++i) {
            const int st = i % ns;
            mbar_wait(&full[st], (i / ns) & 1);
            tc_fence_after();
            const uint32_t a0 = smem_u32(slot(i)), b0 = a0 + (uint32_t)a_bytes;
            uint64_t da = a_mn ? desc_mnmajor(a0, 0) : desc_kmajor(a0, 0);
            uint64_t db = b_mn ? desc_mnmajor(b0, 0) : desc_kmajor(b0, 0);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk, da += a_mn ? 64 : 2, db += b_mn ? 64 : 2) {
                mma_tf32_warp(0u, da, db, idesc2, (i | kk) != 0);
                if (i >= lo_from) mma_tf32_warp(0u, da + a_lo_off, db, idesc, 1);
            }
            mma_commit_warp(&empty[st]);
            if (i == nkb - 1) mma_commit_warp(tbar);
        }
    }
    mbar_wait(tbar, tph & 1);
    ++tph;
    tc_fence_after();
}


// TMEM [128 lanes][2*ncols] -> smem tile (pitch tp floats) as cols[c] + cols[c + ncols] (the hi.lo half);
// warps w and w+4 share lane quadrant w%4
__device__ __forceinline__ void rf_tmem_to_smem(float* tile, int tp, int ncols) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, half = warp >> 2;
    const int row = 32 * q + lane;
    const int per = ncols / 2;
    for (int c = half * per; c < (half + 1) * per; c += 16) {
        float v[16], w[16];
        tmem_ld16(((uint32_t)(32 * q) << 16) + (uint32_t)c, v);
        tmem_ld16(((uint32_t)(32 * q) << 16) + (uint32_t)(c + ncols), w);
#pragma unroll
        for (int i = 0; i < 16; ++i) tile[row * tp + c + i] = v[i] + w[i];
    }
    tc_fence_before();
}

__global__ void __cluster_dims__(kRfSlices, 1, 1) __launch_bounds__(kRfThreads, 1)
    rbm_cd1_fused_kernel(const __grid_constant__ RbmMaps m, const RbmFusedParams p) {
    extern __shared__ uint8_t smem_raw[];
    if (p.trace && threadIdx.x == 0) {  // bring-up: entry time of every CTA (globaltimer, ns)
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        p.trace[64 + blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
    // 1 KB-aligned ring by offsetting the __shared__ array itself (not via an integer round trip), so
    // every pointer derived from it stays in the shared address space (LDS/STS, not generic LD/ST)
    uint8_t* ring = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw));
    float* tile = reinterpret_cast<float*>(ring + kRfStages * kRfStage);  // [128][kRfTileP]
    uint64_t* full = reinterpret_cast<uint64_t*>(tile + 128 * kRfTileP);  // [phase][4]
    uint64_t* empty = full + 16;
    uint64_t* tbar = empty + 16;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tbar + 1);

    const int s = blockIdx.x, j = blockIdx.y;  // visible slice (= cluster rank), hidden tile
    const int warp = threadIdx.x >> 5;
    const int B = p.B, H = p.H, V = p.V;
    const int v0c = s * kRfSliceW, h0c = j * kRfTileH;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 16; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tbar, 1);
        fence_barrier_init();
        tma_prefetch(&m.vk);
        tma_prefetch(&m.wk);
        tma_prefetch(&m.hsk);
        tma_prefetch(&m.wmn);
        tma_prefetch(&m.vmn);
        tma_prefetch(&m.hmn);
        tma_prefetch(&m.vk_lo);
        tma_prefetch(&m.wk_lo);
        tma_prefetch(&m.wmn_lo);
        tma_prefetch(&m.vmn_lo);
        tma_prefetch(&m.hmn_lo);
    }
    if (warp == 1) tmem_alloc(tslot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (*tslot != 0u) __trap();  // TMEM base column 0 (one CTA per SM)
    pdl_wait();
    int tph = 0;
    int tev = 0;
    auto mark = [&]() {
        if (p.trace && threadIdx.x == 0 && (blockIdx.x + blockIdx.y == 0 || (blockIdx.x == 7 && blockIdx.y == 7)))
            p.trace[(blockIdx.x ? 32 : 0) + tev] = clock64();
        ++tev;
    };
    mark();
    if (p.trace && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        p.trace[128 + blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
    if (p.ready) {  // train_stream: wait for this step's staging copies (no cross-stream event)
        if (threadIdx.x == 0) {
            unsigned long long spins = 0;
            unsigned v;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.ready) : "memory");
                if (v >= p.ready_val) break;
                __nanosleep(64);
                if (++spins > (1ull << 26)) __trap();  // watchdog: a launch error instead of a hung GPU
            }
        }
        __syncthreads();
    }
    if (p.v0_src) {
        // zero-copy v0 (a direct call on the caller's pinned buffer): CTA (s, j) moves rows [16 j, 16 j + 16)
        // of visible slice s into Vcat with their tf32 lo parts; the 8 CTAs of slice s then meet at the
        // slice barrier before phase 1 reads the slice by TMA. Staged / streamed steps find v0 and its lo
        // parts already in place (stage_rows_kernel on the copy stream) and skip this barrier.
        const float* src = p.v0_src;
        const long long lds = p.ld_src;
        const int vlo = v0c, vhi = min(v0c + kRfSliceW, V);
        const int w4 = (vhi - vlo) / 4;  // V % 4 == 0 (host-checked)
        for (int idx = threadIdx.x; idx < 16 * w4; idx += kRfThreads) {
            const int r = 16 * j + idx / w4, c = vlo + (idx % w4) * 4;
            if (r < B) {
                const float4 x = __ldcg(reinterpret_cast<const float4*>(src + (long long)r * lds + c));
                *reinterpret_cast<float4*>(p.Vcat + (long long)r * p.ldv + c) = x;
                *reinterpret_cast<float4*>(p.Vlo + (long long)r * p.ldv + c) =
                    make_float4(tf32_lo(x.x), tf32_lo(x.y), tf32_lo(x.z), tf32_lo(x.w));
            }
        }
        rf_grid_sync(sbar_of(p, s), gridDim.y);
    }
    // v0 of this slice exact in tf32 (all its lo parts zero: e.g. binary data), flagged by the staging
    // kernel; unknown (the zero-copy path) counts as inexact
    const bool v0_exact = p.v0_inexact && __ldcg(p.v0_inexact + s) == 0u;
    // the phase-1 sampling uniforms of this thread (rows 16 s + tid / 16, hidden 4 (tid % 16) of tile j),
    // loaded after v0 (which phase 1 needs first) so a host-memory read overlaps the phase-1 product
    double upre[4] = {2.0, 2.0, 2.0, 2.0};
    {
        const int r = 16 * s + (threadIdx.x >> 4), c = (threadIdx.x & 15) * 4;
        const double* usrc = p.u_src ? p.u_src : p.u;
        if (r < B)
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (h0c + c + i < H) upre[i] = __ldcg(usrc + (long long)r * H + h0c + c + i);
    }
    const uint32_t id_h = umma_idesc_tf32(128, kRfTileH, 0, 0);   // [batch x hidden], both K-major
    const uint32_t id_w = umma_idesc_tf32(128, kRfTileH, 1, 1);   // [visible x hidden], both MN-major
    const uint32_t id_h2 = umma_idesc_tf32(128, 2 * kRfTileH, 0, 0), id_w2 = umma_idesc_tf32(128, 2 * kRfTileH, 1, 1);
    const uint32_t id_v = umma_idesc_tf32(128, kRfSliceW, 0, 1), id_v2 = umma_idesc_tf32(128, 2 * kRfSliceW, 0, 1);

    // ---- phases 1 and 3: [batch x 32 hidden] over this slice's 128 visible units, summed over the slices
    auto hidden_phase = [&](int vrow0, bool first) {
        float bhp[4];  // this thread's 4 hidden biases (column V of W_aug), loaded before the product
        {
            const int c = (threadIdx.x & 15) * 4;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int h = h0c + c + i;
                bhp[i] = h < H ? __ldcg(p.W + (long long)h * p.ldw + V) : 0.0f;
            }
        }
        const int ph = first ? 0 : 2;  // all 4 K-blocks in flight at once (4 stages of 48 KB)
        // phase 1's A is v0: exact in tf32 when the whole slice is (binary data) -- no lo loads or MMAs
        rf_product(ring, full + 4 * ph, empty + 4 * ph, tbar, tph, 4, kRfSliceW / 32, 128 * 32 * 4, kRfTileH * 32 * 4,
                   first && v0_exact ? kRfSliceW / 32 : 0, false, false, id_h, id_h2,
                   [&](int kb, uint8_t* ah, uint8_t* bh, uint8_t* bl, uint8_t* al, uint64_t* bar) {
                       tma_load_2d(ah, &m.vk, bar, v0c + kb * 32, vrow0);
                       tma_load_2d(bh, &m.wk, bar, v0c + kb * 32, h0c);
                       tma_load_2d(bl, &m.wk_lo, bar, v0c + kb * 32, h0c);
                       if (al) tma_load_2d(al, &m.vk_lo, bar, v0c + kb * 32, vrow0);
                   });
        mark();
        rf_tmem_to_smem(tile, kRfTileP, kRfTileH);
        __syncthreads();
        {  // partial [B rows][64] of this slice -> L2 workspace (coalesced float4 rows)
            float* dst = p.ws1 + ((long long)j * kRfSlices + s) * 128 * kRfTileH;
            for (int idx = threadIdx.x; idx < B * (kRfTileH / 4); idx += kRfThreads) {
                const int rr = idx / (kRfTileH / 4), cc = (idx % (kRfTileH / 4)) * 4;
                const float* t = tile + rr * kRfTileP + cc;
                *reinterpret_cast<float4*>(dst + rr * kRfTileH + cc) = make_float4(t[0], t[1], t[2], t[3]);
            }
        }
        cluster_sync_all();  // partials of the 8 slices visible cluster-wide (release / acquire at cluster scope)
        mark();
        // rank s finishes batch rows [16 s, 16 s + 16): sum over the slices in fixed order, all loads first
        const int r = 16 * s + (threadIdx.x >> 4), c = (threadIdx.x & 15) * 4;
        float4 x[kRfSlices];
#pragma unroll
        for (int z = 0; z < kRfSlices; ++z)
            x[z] = r < B ? __ldcg(reinterpret_cast<const float4*>(p.ws1 + (((long long)j * kRfSlices + z) * 128 + r) *
                                                                              kRfTileH + c))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        float av[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int z = 0; z < kRfSlices; ++z) {
            av[0] += x[z].x;
            av[1] += x[z].y;
            av[2] += x[z].z;
            av[3] += x[z].w;
        }
        mark();
        if (r < B) {
            float bh[4];
            double uu[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int h = h0c + c + i;
                bh[i] = bhp[i];
                uu[i] = upre[i];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int h = h0c + c + i;
                if (h >= H) continue;
                const float pr = sigmoid_ref(av[i] + bh[i]);  // + bh
                if (first) {  // energy.hpp:101-110 + unit_sample_inplace :59-61
                    p.Hcat[(long long)r * p.ldh + h] = pr;
                    p.Hlo[(long long)r * p.ldh + h] = tf32_lo(pr);
                    p.HS[(long long)r * p.ldhs + h] = (uu[i] < (double)pr) ? 1.0f : 0.0f;
                } else {
                    p.Hcat[(long long)(B + r) * p.ldh + h] = -pr;  // stored negated for phase 4
                    p.Hlo[(long long)(B + r) * p.ldh + h] = tf32_lo(-pr);
                }
            }
        }
    };

    // dependencies are narrower than the grid: phase 2 of (j, s) reads hs[:, tile j] (written by the 8
    // CTAs of cluster j), the phase-2 reduction of slice s reads the partials of the 8 CTAs (., s), and
    // phase 3 / 4 of (j, s) read v1[:, slice s] (written by (., s)) and -h1[:, tile j] (cluster j): so
    // cluster barriers plus 8-CTA slice barriers (global counters) replace every grid-wide barrier
    unsigned long long* sbar = sbar_of(p, s);
    hidden_phase(0, true);
    mark();
    asm volatile("fence.proxy.async.global;" ::: "memory");
    cluster_sync_all();
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mark();

    // ---- phase 2: [batch x 128 visible] over this tile's 64 hidden units; tiles meet in L2.
    // (Measured alternative: no split of K -- one CTA per 32-column tile over all 500 hidden units --
    // is slower: a single SM streams its operands from L2 at ~100 GB/s, 3.7 us for the product alone.)
    // A = the 0/1 samples: exact in tf32, no lo part -- one MMA per K step
    rf_product(ring, full + 4, empty + 4, tbar, tph, 2, kRfTileH / 32, 128 * 32 * 4, kRfSliceW * 32 * 4, kRfTileH / 32,
               false, true, id_v, id_v2,
               [&](int kb, uint8_t* ah, uint8_t* bh, uint8_t* bl, uint8_t*, uint64_t* bar) {
                   tma_load_2d(ah, &m.hsk, bar, h0c + 32 * kb, 0);
                   for (int q = 0; q < kRfSliceW / 32; ++q) {
                       tma_load_2d(bh + q * 4096, &m.wmn, bar, v0c + 32 * q, h0c + 32 * kb);
                       tma_load_2d(bl + q * 4096, &m.wmn_lo, bar, v0c + 32 * q, h0c + 32 * kb);
                   }
               });
    mark();
    {
        float* stg = reinterpret_cast<float*>(ring);  // [128][132], the operand ring is idle now
        rf_tmem_to_smem(stg, kRfSliceW + 4, kRfSliceW);
        __syncthreads();
        float* dst = p.ws2 + (long long)j * 128 * (kRfSlices * kRfSliceW) + v0c;
        for (int idx = threadIdx.x; idx < B * (kRfSliceW / 4); idx += kRfThreads) {
            const int r = idx / (kRfSliceW / 4), c = (idx % (kRfSliceW / 4)) * 4;
            *reinterpret_cast<float4*>(dst + (long long)r * (kRfSlices * kRfSliceW) + c) =
                *reinterpret_cast<const float4*>(stg + r * (kRfSliceW + 4) + c);
        }
    }
    mark();
    rf_grid_sync(sbar, gridDim.y);
    mark();
    // CTA (j, s) finishes batch rows j, j + jt, j + 2 jt, ... of slice s (interleaved: every CTA gets
    // ~B/jt rows): one warp per row (two rows per warp), 4 columns per lane; every load of both rows
    // is issued before the first use
    {
        const int c = v0c + (threadIdx.x & 31) * 4;
        float4 part[2][8], vz[2];
        int rows[2];
        const float4 bv = c < V ? *reinterpret_cast<const float4*>(p.W + (long long)H * p.ldw + c)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int r = j + (int)gridDim.y * (warp + 8 * rr);  // B <= 16 jt (host-checked)
            rows[rr] = r;
            if (r < B) {
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    part[rr][t] = t < p.jt ? *reinterpret_cast<const float4*>(
                                                 p.ws2 + ((long long)t * 128 + r) * (kRfSlices * kRfSliceW) + c)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
                vz[rr] = c < V ? *reinterpret_cast<const float4*>(p.Vcat + (long long)r * p.ldv + c)
                               : make_float4(0.f, 0.f, 0.f, 0.f);  // slices past V: nothing to read
            }
        }
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int r = rows[rr];
            double pd = 0.0;
            if (r < B) {
                float4 acc = part[rr][0];
#pragma unroll
                for (int t = 1; t < 8; ++t) {
                    acc.x += part[rr][t].x;
                    acc.y += part[rr][t].y;
                    acc.z += part[rr][t].z;
                    acc.w += part[rr][t].w;
                }
                const float av[4] = {acc.x, acc.y, acc.z, acc.w}, bb[4] = {bv.x, bv.y, bv.z, bv.w};
                const float v0v[4] = {vz[rr].x, vz[rr].y, vz[rr].z, vz[rr].w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int v = c + i;
                    if (v >= V) continue;
                    const float pr = sigmoid_ref(av[i] + bb[i]);  // + bv
                    p.Vcat[(long long)(B + r) * p.ldv + v] = pr;
                    p.Vlo[(long long)(B + r) * p.ldv + v] = tf32_lo(pr);
                    const double d = (double)v0v[i] - (double)pr;  // energy.hpp:84-96
                    pd += d * d;
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) pd += __shfl_xor_sync(0xffffffffu, pd, o);
            if (r < B && (threadIdx.x & 31) == 0) p.row_part[(long long)s * p.cap + r] = pd;
        }
    }
    mark();
    rf_grid_sync(sbar, gridDim.y);
    mark();

    // ---- phase 3
    hidden_phase(B, false);
    mark();
    asm volatile("fence.proxy.async.global;" ::: "memory");
    cluster_sync_all();
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mark();

    // ---- phase 4: [128 visible x 64 hidden] over K = 2B batch rows, then W_aug[j, s] += alpha * D^T.
    // The W tile is read into registers before the product (nothing else writes it) so the update is
    // a pure store after the MMAs: W, the bh column (v == V) and the bv row (h == H)
    // thread = visible column mc of the tile, rows n = 2 i + r0 (32 per thread); one base pointer per
    // array and a 32-bit row stride, predicated rather than branched per element
    constexpr int kPer = kRfTileH * kRfSliceW / kRfThreads;
    static_assert(kRfThreads == 2 * kRfSliceW, "two tile rows per pass");
    const int mc4 = threadIdx.x % kRfSliceW, r04 = threadIdx.x / kRfSliceW;
    const bool col_ok = v0c + mc4 <= V;
    const int nrows = min(kRfTileH, H + 1 - h0c);  // W rows + the bv row (h == H)
    const long long base4 = (long long)(h0c + r04) * p.ldw + v0c + mc4;
    const int rstride = 2 * (int)p.ldw;
    float wv[kPer];
    {
        const float* wsrc = p.W + base4;
#pragma unroll
        for (int i = 0; i < kPer; ++i)
            wv[i] = (!p.grad_only && col_ok && 2 * i + r04 < nrows) ? __ldcg(wsrc + i * rstride) : 0.0f;
    }
    // K-blocks of v0 rows only (kb < B / 32) need no A lo when the slice's v0 is exact in tf32
    rf_product(ring, full + 12, empty + 12, tbar, tph, 4, (2 * B + 31) / 32, 128 * 32 * 4, kRfTileH * 32 * 4,
               v0_exact ? B / 32 : 0, true, true, id_w, id_w2,
               [&](int kb, uint8_t* ah, uint8_t* bh, uint8_t* bl, uint8_t* al, uint64_t* bar) {
                   for (int q = 0; q < 4; ++q) {
                       tma_load_2d(ah + q * 4096, &m.vmn, bar, v0c + 32 * q, kb * 32);
                       if (al) tma_load_2d(al + q * 4096, &m.vmn_lo, bar, v0c + 32 * q, kb * 32);
                   }
                   for (int q = 0; q < kRfTileH / 32; ++q) {
                       tma_load_2d(bh + q * 4096, &m.hmn, bar, h0c + 32 * q, kb * 32);
                       tma_load_2d(bl + q * 4096, &m.hmn_lo, bar, h0c + 32 * q, kb * 32);
                   }
               });
    mark();
    rf_tmem_to_smem(tile, kRfTileP, kRfTileH);
    __syncthreads();
    mark();
    {  // all tile reads first, then the stores (no load -> store chain per element)
        float d[kPer];
        const float* trow = tile + mc4 * kRfTileP + r04;
#pragma unroll
        for (int i = 0; i < kPer; ++i) d[i] = trow[2 * i];
        if (col_ok) {
            if (p.grad_only) {
                float* g = p.G + base4;
#pragma unroll
                for (int i = 0; i < kPer; ++i)
                    if (2 * i + r04 < nrows) g[i * rstride] = d[i];
            } else {
                float* w = p.W + base4;
                float* wl = p.Wlo + base4;
#pragma unroll
                for (int i = 0; i < kPer; ++i) {
                    const float x = wv[i] + p.alpha * d[i];
                    if (2 * i + r04 < nrows) {
                        w[i * rstride] = x;
                        wl[i * rstride] = tf32_lo(x);
                    }
                }
            }
        }
    }
    __syncthreads();
    mark();
    // the step's reconstruction error straight into host-mapped memory: the last CTA to finish sums
    // the (slice, row) partials written in phase 2 in recon_tree_sum's order (rows over lanes, slices
    // in order, then a fixed shuffle tree), every load issued before the first add (B <= 128: one
    // round trip) -- no device-to-host copy behind the step
    if (p.recon_out) {
        __shared__ unsigned s_last;
        if (threadIdx.x == 0) {
            __threadfence();
            s_last = atomicAdd(p.done, 1u) == gridDim.x * gridDim.y - 1;
        }
        __syncthreads();
        if (s_last && warp == 0) {
            const int lane = threadIdx.x & 31;
            double v[4][kRfSlices], acc = 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int s2 = 0; s2 < kRfSlices; ++s2)
                    v[i][s2] = lane + 32 * i < B ? __ldcg(p.row_part + (long long)s2 * p.cap + lane + 32 * i) : 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (lane + 32 * i < B)
#pragma unroll
                    for (int s2 = 0; s2 < kRfSlices; ++s2) acc += v[i][s2];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) {
                *reinterpret_cast<volatile double*>(p.recon_out) = acc / p.bg;
                *p.done = 0;
            }
        }
    }
    if (p.trace && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        p.trace[192 + blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
    pdl_trigger();
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(0u, 256);
    }
}

}  // namespace b2n
