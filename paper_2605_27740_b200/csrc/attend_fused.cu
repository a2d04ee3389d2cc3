// attend_fused.cu -- K3 + K4 in one launch: per-unit top-k page selection followed by the
// tensor-core sparse decode attention over exactly those pages (the decode hot path of
// attention.py:137-146: select.py:87-115 radix_topk, then sparse_attention for the G heads
// of the group, attention.py:94-107 / _kernels_cy.pyx:129-172).
//
// Why fused: at the headline shape (256 units x 8192 pages, k = 128) a standalone selection
// kernel is latency-bound (one CTA per unit, ~15 barrier phases) and its launch boundary
// drains the GPU between two HBM-bound kernels.  Here the CTA that attends a unit first
// selects its pages -- the keys are read once into shared memory, the selected physical ids
// stay in shared memory and feed the TMA producer directly -- so the select costs one CTA
// prologue instead of a kernel, and the sel / n_sel / kth / kplus1 outputs are still written
// for the caller (bit-identical to pt_topk: same select_block).
//
// Grid (nchunk, U), 8 warps (4 with PT_SA_SEL_THREADS=128): all select, the first 4 stream.
// Every chunk CTA of a unit runs the (deterministic) selection;
// chunk 0 publishes it.  Chunk c attends the c-th contiguous slice of the emitted list; the
// warps of the CTA interleave pages (warp w: slice[w], slice[w+4], ...), each through a
// private nstage-deep ring of TMA tensor copies (one K + one V page per stage), QK / PV on
// mma.sync m16n8k16 with the G <= 8 heads as N (see attend.cuh for the fragment layouts);
// warps merge in shared memory, chunks through the workspace (last-arriving CTA, ticket).
//
// Shared memory: [region: select scratch (keys + bins) | reused as the stage rings and then
// the merge buffers] [selected ids, k ints] [mbarriers].
#include "attend.cuh"
#include "select.cuh"

namespace pt {

struct SelAttnParams {
    const uint16_t *keys;
    const uint16_t *tile_max;
    const int32_t *seq_len;
    const int32_t *page_table;
    int32_t *sel, *sel_logical, *n_sel, *kth, *kplus1;
    const void *q;
    float *out, *lse, *ws;
    int32_t *tickets;
    int q_dtype, U, G, Pmax, k, nchunk, nstage;
    int region;     // bytes of the shared region (multiple of 1024)
    int region_lo;  // bounded mode: start of the selection tail's scratch (>= the stage rings)
    int prof;    // record phase timestamps into g_sa_prof
    float scale;
    // bounded mode (keys = lower keys of pt_score_bounded's intervals): the upper keys, and
    // what the exact key of a page needs -- f32 means (tile layout), stds, fl(lam * ||q_g||)
    const uint16_t *keys_hi;
    const float *rows32, *stds, *lamnorm;  // rows32: the mirror's row-major f32 means
    int rcap;  // pages resolved per round (their f32 means staged in shared memory)
    int kv_evict_first;  // L2 policy of the page stream (PT_SA_KV_EVICT=normal: 0)
};

constexpr int kSAWarps = 4;

// Optional phase timestamps (%globaltimer, ns) per CTA for tuning: enabled by
// PT_SA_PROF=1 on the host, read back with pt_debug_sa_prof().  16 stamps per CTA
// (6 kernel phases + 4 inside the selection + 5 inside the bounded-mode resolve + its rounds).
constexpr int kSAProfCtas = 4096;
constexpr int kSAProfN = 20;
__device__ unsigned long long g_sa_prof[kSAProfCtas * kSAProfN];
// PT_SA_PROF=1: %globaltimer (ns, comparable across SMs, ~1 us update granularity);
// PT_SA_PROF=2: %clock64 (SM cycles: phase durations within a CTA only)
__device__ __forceinline__ unsigned long long gtimer(bool clk) {
    unsigned long long t;
    if (clk) asm volatile("mov.u64 %0, %clock64;" : "=l"(t));
    else asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void sa_cp_async16(void *smem_dst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void sa_cp_async4(void *smem_dst, const void *gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void sa_cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// the exact reference score of one page from its staged f32 mean row (the resolve step of
// bounded mode): K2's exact order -- sequential d, fl(q * m) then fl(acc + .) -- for GG >= G
// heads (GG = 4 or 8: the compile-time head loop), + fl(lamnorm_g * std), strict-> max
template <int D, int GG>
__device__ __forceinline__ float sa_exact_score(const float *row, const float *sq, const float *sln,
                                                float sd, int G) {
    const float4 *row4 = reinterpret_cast<const float4 *>(row);
    float acc[GG];
#pragma unroll
    for (int g = 0; g < GG; g++) acc[g] = 0.f;
#pragma unroll 2
    for (int c = 0; c < D / 4; c++) {
        const float4 m4 = row4[c];
        const float mv[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const float4 *q4 = reinterpret_cast<const float4 *>(sq + (4 * c + e) * 8);
            const float4 qa = q4[0];
            float qv[8] = {qa.x, qa.y, qa.z, qa.w, 0.f, 0.f, 0.f, 0.f};
            if constexpr (GG > 4) {
                const float4 qc = q4[1];
                qv[4] = qc.x; qv[5] = qc.y; qv[6] = qc.z; qv[7] = qc.w;
            }
#pragma unroll
            for (int g = 0; g < GG; g++) acc[g] = __fadd_rn(acc[g], __fmul_rn(qv[g], mv[e]));
        }
    }
    float best = -INFINITY;
#pragma unroll
    for (int g = 0; g < GG; g++) {
        if (g < G) {
            const float a = __fadd_rn(acc[g], __fmul_rn(sln[g], sd));
            if (a > best) best = a;
        }
    }
    return best;
}

// the same with the page's f32 row from global memory (chunks of 32 dims in flight together)
// and the query rows from shared memory (f32 [D][8], as sa_exact_score): the warp-per-unit
// variant's resolution, one lane per page
template <int D, int GG>
__device__ __noinline__ float sa_exact_score_rowg(const float *row, const float *sq, const float *lnp,
                                                  float sd, int G) {
    constexpr int CH = 8;
    static_assert((D / 4) % CH == 0, "row chunks");
    float acc[GG];
#pragma unroll
    for (int g = 0; g < GG; g++) acc[g] = 0.f;
    const float4 *row4 = reinterpret_cast<const float4 *>(row);
    for (int c0 = 0; c0 < D / 4; c0 += CH) {
        float4 m4[CH];
#pragma unroll
        for (int i = 0; i < CH; i++) m4[i] = __ldg(row4 + c0 + i);
#pragma unroll
        for (int i = 0; i < CH; i++) {
            const float mv[4] = {m4[i].x, m4[i].y, m4[i].z, m4[i].w};
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const float4 *q4 = reinterpret_cast<const float4 *>(sq + (4 * (c0 + i) + e) * 8);
                const float4 qa = q4[0];
                float qv[8] = {qa.x, qa.y, qa.z, qa.w, 0.f, 0.f, 0.f, 0.f};
                if constexpr (GG > 4) {
                    const float4 qc = q4[1];
                    qv[4] = qc.x; qv[5] = qc.y; qv[6] = qc.z; qv[7] = qc.w;
                }
#pragma unroll
                for (int g = 0; g < GG; g++) acc[g] = __fadd_rn(acc[g], __fmul_rn(qv[g], mv[e]));
            }
        }
    }
    float best = -INFINITY;
#pragma unroll
    for (int g = 0; g < GG; g++) {
        if (g < G) {
            const float a = __fadd_rn(acc[g], __fmul_rn(__ldg(lnp + g), sd));
            if (a > best) best = a;
        }
    }
    return best;
}

__host__ __device__ __forceinline__ size_t sa_keys_bytes(int Pmax) {
    return (size_t)((Pmax + 8) / 8) * 16;
}

// NT threads run the selection (NT / 32 warps); the first kSAWarps warps stream the pages
template <int D, int MT, int NT, bool BND>
__global__ void __launch_bounds__(NT, 2) k_select_attend(const __grid_constant__ CUtensorMap tmk,
                                                              const __grid_constant__ CUtensorMap tmv,
                                                              const SelAttnParams p) {
    constexpr int S = 16 * MT;
    constexpr int KS = D / 16;
    constexpr int NW = kSAWarps;
    constexpr uint32_t PAGE_BYTES = S * D * 2;
    constexpr uint32_t STAGE_BYTES = 2 * PAGE_BYTES;
    extern __shared__ __align__(1024) char smem[];
    __shared__ SelectShared<NT> sh;
    __shared__ SelectCandShared<NT> csh;
    __shared__ int sdummy[3];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t u = blockIdx.y;
    const int c = blockIdx.x;
    const int G = p.G, k = p.k, nstage = p.nstage;
    int *ids = reinterpret_cast<int *>(smem + p.region);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.region + (((size_t)k * 4 + 7) & ~(size_t)7)) +
                     (warp < NW ? warp : 0) * nstage;

    // PDL: the prologue below (lengths, tail page, query fragments) reads nothing the scoring
    // kernel writes, so it runs while the scorer drains; keys / tile maxima wait for it
    pdl_trigger();
    const int n = p.seq_len[u];
    const int P = (n + S - 1) / S;
    const bool lead = (c == 0);
    const int cta = blockIdx.y * gridDim.x + blockIdx.x;
    const bool prof = p.prof && threadIdx.x == 0 && cta < kSAProfCtas;
    if (prof) g_sa_prof[cta * kSAProfN + 0] = gtimer(p.prof == 2);
    if (P == 0) {
        if (lead && threadIdx.x == 0) { p.n_sel[u] = 0; p.kth[u] = 0; p.kplus1[u] = -1; }
        return;
    }
    // ---- independent loads first (tail page, query fragments): their latencies overlap the
    // selection's key loads
    const int tail_pid = p.page_table[u * p.Pmax + P - 1];
    const int tail_rows = n - (P - 1) * S;
    uint32_t qb[KS][2];
    if constexpr (!BND) {  // bounded mode: from the f32 rows in shared memory after selecting
        const int gq = lane >> 2;
#pragma unroll
        for (int ks = 0; ks < KS; ks++) {
            const int d0 = ks * 16 + 2 * (lane & 3);
            uint32_t b0 = 0, b1 = 0;
            if (gq < G) {
                const int64_t row = (u * G + gq) * (int64_t)D;
                if (p.q_dtype == PT_BF16) {
                    const uint32_t *qp =
                        reinterpret_cast<const uint32_t *>(static_cast<const uint16_t *>(p.q) + row);
                    b0 = __ldg(qp + (d0 >> 1));
                    b1 = __ldg(qp + ((d0 + 8) >> 1));
                } else {
                    const float *qp = static_cast<const float *>(p.q) + row;
                    b0 = pack_bf16(qp[d0], qp[d0 + 1]);
                    b1 = pack_bf16(qp[d0 + 8], qp[d0 + 9]);
                }
            }
            qb[ks][0] = b0;
            qb[ks][1] = b1;
        }
    }
    // bounded mode scratch.  Lower part [0, region_lo): the phase-1 arrays (keys, bins, tile
    // maxima, upper keys, candidates' upper keys) -- dead once the candidate bracket is known,
    // then the stage rings; upper part [region_lo, region): what the selection tail keeps using
    // while the rings stream (query rows as f32 [D][8], lam ||q||, resolve counter, mbarrier,
    // candidate flags, resolve list / stds / staged f32 rows)
    const size_t sel_end = sa_keys_bytes(p.Pmax) + kSelectBins * 4 + (size_t)(p.Pmax / 32) * 2;
    uint16_t *skhi = reinterpret_cast<uint16_t *>(smem + ((sel_end + 15) & ~(size_t)15));
    uint16_t *candhi = reinterpret_cast<uint16_t *>(reinterpret_cast<char *>(skhi) + sa_keys_bytes(p.Pmax));
    char *up = smem + p.region_lo;
    float *sq = reinterpret_cast<float *>(up);
    float *sln = sq + D * 8;  // fl(lam * ||q_g||), 8
    int *rcnt = reinterpret_cast<int *>(sln + 8);
    uint64_t *rbar = reinterpret_cast<uint64_t *>(rcnt + 4);
    uint8_t *cflag = reinterpret_cast<uint8_t *>(rbar + 2);
    int *rlist = reinterpret_cast<int *>(cflag + kCandMax);
    float *rstd = reinterpret_cast<float *>(rlist + p.rcap);
    float *rstage = reinterpret_cast<float *>(rstd + p.rcap);
    __shared__ int sdefer[8];  // deferred selection: flag, C, L, A, B, below, n_sure
    if constexpr (BND) {  // q is not written by the scorer: widened before the PDL wait
        for (int i = threadIdx.x; i < D * 8; i += NT) {
            const int d = i >> 3, g = i & 7;
            float x = 0.f;
            if (g < G) {
                const int64_t e = (u * G + g) * (int64_t)D + d;
                x = p.q_dtype == PT_BF16 ? bf16_bits_to_f32(static_cast<const uint16_t *>(p.q)[e])
                                         : static_cast<const float *>(p.q)[e];
            }
            sq[i] = x;
        }
        if (threadIdx.x == 0) sdefer[0] = 0;
    }
    pdl_wait();
    if (prof) g_sa_prof[cta * kSAProfN + 1] = gtimer(p.prof == 2);

    // ---- selection (select.py:87-115): physical ids land in `ids` in emission order ----
    // candidate selection (select_cand: tile-maximum lower bound or bisection, then the
    // candidates only); select_block for take-all and massive ties
    const int ns = P < k ? P : k;
    const uint16_t *krow = p.keys + u * (int64_t)p.Pmax;
    int32_t *o_sel = lead ? p.sel + u * (int64_t)k : nullptr;
    int32_t *o_log = (lead && p.sel_logical) ? p.sel_logical + u * (int64_t)k : nullptr;
    int32_t *o_n = lead ? p.n_sel + u : &sdummy[0];
    int32_t *o_kth = lead ? p.kth + u : &sdummy[1];
    int32_t *o_kp1 = lead ? p.kplus1 + u : &sdummy[2];
    // keys -> shared memory: every 16-byte load of a thread in flight before its first store
    uint16_t *skeys = reinterpret_cast<uint16_t *>(smem);
    int *bins = reinterpret_cast<int *>(smem + sa_keys_bytes(p.Pmax));
    // the tile maxima (one u16 per 32 pages) ride in the same load round as the keys
    uint16_t *stm = reinterpret_cast<uint16_t *>(smem + sa_keys_bytes(p.Pmax) + kSelectBins * 4);
    const int ntiles = (P + 31) >> 5;
    const bool tm_stage = p.tile_max != nullptr && ntiles <= NT * 8;
    {
        constexpr int kTm = 8;
        const uint16_t *tsrc = p.tile_max + u * (int64_t)(p.Pmax >> 5);
        uint16_t tv[kTm];
#pragma unroll
        for (int j = 0; j < kTm; j++)
            if (tm_stage && threadIdx.x + j * NT < ntiles) tv[j] = __ldcg(tsrc + threadIdx.x + j * NT);
        const uint4 *src = reinterpret_cast<const uint4 *>(krow);
        const uint4 *hsrc = reinterpret_cast<const uint4 *>(BND ? p.keys_hi + u * (int64_t)p.Pmax : krow);
        constexpr int kMax = BND ? 4 : 8;  // bounded: the upper keys in the same load round
        const int nv = (P + 7) / 8;
        for (int i0 = threadIdx.x; i0 < nv; i0 += kMax * NT) {
            uint4 v[kMax], w[kMax];
#pragma unroll
            for (int j = 0; j < kMax; j++)
                if (i0 + j * NT < nv) {
                    v[j] = __ldcg(src + i0 + j * NT);
                    if constexpr (BND) w[j] = __ldcg(hsrc + i0 + j * NT);
                }
#pragma unroll
            for (int j = 0; j < kMax; j++)
                if (i0 + j * NT < nv) {
                    reinterpret_cast<uint4 *>(skeys)[i0 + j * NT] = v[j];
                    if constexpr (BND) reinterpret_cast<uint4 *>(skhi)[i0 + j * NT] = w[j];
                }
        }
#pragma unroll
        for (int j = 0; j < kTm; j++)
            if (tm_stage && threadIdx.x + j * NT < ntiles) stm[threadIdx.x + j * NT] = tv[j];
    }
    if constexpr (BND) {
        if (threadIdx.x < 8) sln[threadIdx.x] = p.lamnorm[u * 8 + threadIdx.x];
    }
    __syncthreads();
    // Exact keys (the reference's f32 score, K2's exact order: sequential d, fl(q * m) then
    // fl(acc + .), + fl(fl(lam ||q||) * std), strict-> max over heads) of listed pages: rows of
    // the mirror's row-major f32 means by one bulk copy each (one mbarrier phase per round).
    constexpr int RS = D + 4;  // staged row stride (floats): conflict-free float4 reads
    int rphase = 0;
    if constexpr (BND) {
        if (threadIdx.x == 0) {
            mbar_init(rbar, 1);
            fence_mbar_init();
        }
    }
    const float *m32 = p.rows32 + u * (int64_t)p.Pmax * D;
    // one round over rlist[0 .. nr) (nr <= rcap): page_of(entry) -> logical page,
    // store(entry, key) writes the exact key; returns the largest key (this thread's)
    auto resolve_batch = [&](int nr, auto page_of, auto store) -> int {
        int mxr = -1;
        if (threadIdx.x == 0 && nr) mbar_arrive_expect_tx(rbar, (uint32_t)(nr * D * 4));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads
        __syncthreads();
        for (int i = threadIdx.x; i < nr; i += NT) {
            const int pg = page_of(rlist[i]);
            bulk_g2s(rstage + i * RS, m32 + (int64_t)pg * D, D * 4, rbar);
            sa_cp_async4(rstd + i, p.stds + u * (int64_t)p.Pmax + pg);
        }
        sa_cp_async_wait_all();
        if (nr) mbar_wait(rbar, (uint32_t)(rphase & 1));
        rphase += nr ? 1 : 0;
        __syncthreads();
        if (prof) g_sa_prof[cta * kSAProfN + 12] = gtimer(p.prof == 2);
        for (int i = threadIdx.x; i < nr; i += NT) {
            const float best = G <= 4 ? sa_exact_score<D, 4>(rstage + i * RS, sq, sln, rstd[i], G)
                                      : sa_exact_score<D, 8>(rstage + i * RS, sq, sln, rstd[i], G);
            const uint16_t key = encode_ordered(f32_to_bf16_rne(best));
            store(rlist[i], key);
            mxr = max(mxr, (int)key);
        }
        __syncthreads();
        if (prof) g_sa_prof[cta * kSAProfN + 13] = gtimer(p.prof == 2);
        return mxr;
    };
    // warp-aggregated append of the flagged entries (bit e of f: entry base_e + e) to rlist
    auto list_append = [&](uint32_t f, int first) {
        const int lane_ = threadIdx.x & 31;
        const int c = __popc(f);
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane_ >= o) inc += y;
        }
        const int tot = __shfl_sync(0xffffffffu, inc, 31);
        int base = 0;
        if (lane_ == 31 && tot) base = atomicAdd(rcnt, tot);
        base = __shfl_sync(0xffffffffu, base, 31) + inc - c;
        while (f) {
            const int e = __ffs(f) - 1;
            f &= f - 1;
            if (base < p.rcap) rlist[base] = first + e;
            base++;
        }
    };
    auto block_max_int = [&](int v) -> int {
        v = __reduce_max_sync(0xffffffffu, v);
        if ((threadIdx.x & 31) == 0) csh.red[1][threadIdx.x >> 5][1] = (uint32_t)v;
        __syncthreads();
        int t = -1;
#pragma unroll
        for (int w = 0; w < NT / 32; w++) t = max(t, (int)csh.red[1][w][1]);
        __syncthreads();
        return t;
    };
    // (a) the key array: every page whose interval is not one key and reaches L (L < 0: all);
    // returns the largest key written, block-wide
    auto resolve = [&](int L) -> int {
        int mxr = -1;
        const int nvec = (P + 7) >> 3;
        const uint32_t Lc = (uint32_t)(L < 0 ? 0 : L);
        if (prof) g_sa_prof[cta * kSAProfN + 10] = gtimer(p.prof == 2);
        for (;;) {
            if (threadIdx.x == 0) *rcnt = 0;
            __syncthreads();
            for (int v0 = 0; v0 < nvec; v0 += NT) {
                const int v = v0 + threadIdx.x;
                uint32_t f = 0u;  // bit e: key 8 v + e needs resolving
                if (v < nvec) {
                    const uint4 a = reinterpret_cast<const uint4 *>(skeys)[v];
                    const uint4 b = reinterpret_cast<const uint4 *>(skhi)[v];
                    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                    for (int e = 0; e < 8; e++) {
                        const uint32_t lo = (aw[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
                        const uint32_t hi = (bw[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
                        if (v * 8 + e < P && hi >= Lc && lo != hi) f |= 1u << e;
                    }
                }
                list_append(f, v * 8);
            }
            __syncthreads();
            if (prof) g_sa_prof[cta * kSAProfN + 11] = gtimer(p.prof == 2);
            const int n = *rcnt;
            mxr = max(mxr, resolve_batch(n < p.rcap ? n : p.rcap, [](int e) { return e; },
                                         [&](int e, uint16_t key) { skeys[e] = key; skhi[e] = key; }));
            if (n <= p.rcap) break;
        }
        return block_max_int(mxr);
    };
    // (b) the candidate list of select_cand: candidates with an uncertain key whose interval
    // meets the threshold bracket [A, B]; exact keys go into the list entries
    auto resolve_cands = [&](int C, int A, int B) {
        if (prof) g_sa_prof[cta * kSAProfN + 10] = gtimer(p.prof == 2);
        for (;;) {
            if (threadIdx.x == 0) *rcnt = 0;
            __syncthreads();
            for (int i0 = 0; i0 < C; i0 += NT) {
                const int i = i0 + threadIdx.x;
                uint32_t f = 0u;
                if (i < C) {
                    const int lo = (int)(csh.cand[i] >> 16), hi = candhi[i];
                    if (lo != hi && hi >= A && lo <= B) f = 1u;
                }
                list_append(f, i);
            }
            __syncthreads();
            if (prof) g_sa_prof[cta * kSAProfN + 11] = gtimer(p.prof == 2);
            const int n = *rcnt;
            resolve_batch(n < p.rcap ? n : p.rcap, [&](int i) { return (int)(csh.cand[i] & 0xFFFFu); },
                          [&](int i, uint16_t key) {
                              csh.cand[i] = ((uint32_t)key << 16) | (csh.cand[i] & 0xFFFFu);
                              candhi[i] = key;
                          });
            if (n <= p.rcap) break;
        }
    };
    // (c) deferred selection tail on warps 4..7 (named barrier 1, NT / 2 threads), while warps
    // 0..3 stream the certainly selected pages: resolve the bracket candidates (cflag bit 2),
    // the threshold = the k-th largest candidate key, the ordered compaction with the
    // reference's tie rule (select.py:87-115) -- outputs in logical order, and the selected
    // pages not streamed yet (cflag bit 1 clear) appended to ids[n_sure ..] in logical order --
    // then n_sel / kth / kplus1
    auto bounded_tail = [&](int n_sure) {
        constexpr int NT2 = NT / 2;
        const int t = (int)threadIdx.x - NT2, w2 = t >> 5;
        auto sync2 = [] { asm volatile("bar.sync 1, %0;" ::"n"(NT / 2) : "memory"); };
        auto sum2 = [&](int v, int slot) -> int {  // sum over the NT2 tail threads
            v = __reduce_add_sync(0xffffffffu, v);
            if (lane == 0) csh.red[slot][w2][0] = (uint32_t)v;
            sync2();
            int s2 = 0;
#pragma unroll
            for (int w = 0; w < NT2 / 32; w++) s2 += (int)csh.red[slot][w][0];
            sync2();
            return s2;
        };
        auto max2 = [&](int v) -> int {
            v = __reduce_max_sync(0xffffffffu, v);
            if (lane == 0) csh.red[1][w2][1] = (uint32_t)v;
            sync2();
            int m = -1;
#pragma unroll
            for (int w = 0; w < NT2 / 32; w++) m = max(m, (int)csh.red[1][w][1]);
            sync2();
            return m;
        };
        // exclusive scan of (a, b) over the tail threads in thread order
        auto exscan2 = [&](int a, int b, int &ea, int &eb, int &ta, int &tb) {
            int ia = a, ib = b;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int xa = __shfl_up_sync(0xffffffffu, ia, o);
                const int xb = __shfl_up_sync(0xffffffffu, ib, o);
                if (lane >= o) { ia += xa; ib += xb; }
            }
            if (lane == 31) { csh.red[0][w2][0] = (uint32_t)ia; csh.red[0][w2][1] = (uint32_t)ib; }
            sync2();
            ea = ia - a; eb = ib - b; ta = 0; tb = 0;
#pragma unroll
            for (int w = 0; w < NT2 / 32; w++) {
                const int wa = (int)csh.red[0][w][0], wb = (int)csh.red[0][w][1];
                if (w < w2) { ea += wa; eb += wb; }
                ta += wa; tb += wb;
            }
            sync2();
        };
        const int C = sdefer[1], L = sdefer[2];
        const bool tprof = p.prof && t == 0 && cta < kSAProfCtas;
        if (tprof) g_sa_prof[cta * kSAProfN + 10] = gtimer(p.prof == 2);
        // (1) exact keys of the bracket candidates, in rounds of rcap
        for (;;) {
            if (t == 0) *rcnt = 0;
            sync2();
            for (int i0 = 0; i0 < C; i0 += NT2) {
                const int i = i0 + t;
                list_append((i < C && (cflag[i] & 2)) ? 1u : 0u, i);
            }
            sync2();
            const int n = *rcnt, nr = n < p.rcap ? n : p.rcap;
            if (tprof) g_sa_prof[cta * kSAProfN + 11] = gtimer(p.prof == 2);
            if (t == 0 && nr) mbar_arrive_expect_tx(rbar, (uint32_t)(nr * D * 4));
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            sync2();
            for (int i = t; i < nr; i += NT2) {
                const int pg = (int)(csh.cand[rlist[i]] & 0xFFFFu);
                bulk_g2s(rstage + i * RS, m32 + (int64_t)pg * D, D * 4, rbar);
                sa_cp_async4(rstd + i, p.stds + u * (int64_t)p.Pmax + pg);
            }
            sa_cp_async_wait_all();
            if (nr) mbar_wait(rbar, (uint32_t)(rphase & 1));
            rphase += nr ? 1 : 0;
            sync2();
            if (tprof) g_sa_prof[cta * kSAProfN + 12] = gtimer(p.prof == 2);
            for (int i = t; i < nr; i += NT2) {
                const int ci = rlist[i];
                const float best = G <= 4 ? sa_exact_score<D, 4>(rstage + i * RS, sq, sln, rstd[i], G)
                                          : sa_exact_score<D, 8>(rstage + i * RS, sq, sln, rstd[i], G);
                const uint32_t key = encode_ordered(f32_to_bf16_rne(best));
                csh.cand[ci] = (key << 16) | (csh.cand[ci] & 0xFFFFu);
                cflag[ci] = (uint8_t)(cflag[ci] & 1);
            }
            sync2();
            if (tprof) g_sa_prof[cta * kSAProfN + 13] = gtimer(p.prof == 2);
            if (n <= nr) break;
        }
        // (2) threshold: the k-th largest candidate key (every key that can reach it is exact)
        int mk = -1;
        for (int i = t; i < C; i += NT2) mk = max(mk, (int)(csh.cand[i] >> 16));
        const int mx = max2(mk);
        int thr;
        if (mx - L < 64) {
            if (t < 64) csh.bins[t] = 0;
            sync2();
            for (int i = t; i < C; i += NT2) {
                const int key = (int)(csh.cand[i] >> 16);
                if (key >= L) atomicAdd(&csh.bins[mx - key], 1);
            }
            sync2();
            if (w2 == 0) {
                const int c0 = csh.bins[2 * lane], c1 = csh.bins[2 * lane + 1];
                int incl = c0 + c1;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int pre = incl - c0 - c1;
                int b = 999;
                if (pre < k && pre + c0 >= k) b = 2 * lane;
                else if (pre + c0 < k && incl >= k) b = 2 * lane + 1;
                b = __reduce_min_sync(0xffffffffu, b);
                if (lane == 0) csh.thr = mx - b;
            }
            sync2();
            thr = csh.thr;
            sync2();
        } else {
            int lo = L, hi = mx + 1;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                int cnt = 0;
                for (int i = t; i < C; i += NT2) cnt += (int)(csh.cand[i] >> 16) >= mid;
                if (sum2(cnt, 0) >= k) lo = mid; else hi = mid;
            }
            thr = lo;
        }
        // (3) ordered compaction over the (logically ordered) candidates
        const int cs = (C + NT2 - 1) / NT2;
        const int i0 = min(t * cs, C), i1 = min(i0 + cs, C);
        int g = 0, q = 0, bl = -1;
        for (int i = i0; i < i1; i++) {
            const int key = (int)(csh.cand[i] >> 16);
            g += key > thr;
            q += key == thr;
            if (key < thr) bl = max(bl, key);
        }
        int gb, qb2, gt_tot, eq_tot;
        exscan2(g, q, gb, qb2, gt_tot, eq_tot);
        const int below = max(max2(bl), sdefer[5]);
        const int budget = k - gt_tot;  // in [1, eq_tot]
        int r = 0;
        {
            int seen = qb2;
            for (int i = i0; i < i1; i++) {
                const int key = (int)(csh.cand[i] >> 16);
                bool sel = key > thr;
                if (key == thr) { sel = seen < budget; seen++; }
                if (sel && !(cflag[i] & 1)) r++;
            }
        }
        int rb, dummy, rtot, dtot;
        exscan2(r, 0, rb, dummy, rtot, dtot);
        int pos = gb + min(qb2, budget), seen = qb2, rpos = n_sure + rb;
        for (int i = i0; i < i1; i++) {
            const uint32_t cv = csh.cand[i];
            const int key = (int)(cv >> 16), idx = (int)(cv & 0xFFFFu);
            bool sel = key > thr;
            if (key == thr) { sel = seen < budget; seen++; }
            if (sel) {
                const int pid = __ldg(p.page_table + u * p.Pmax + idx);
                if (o_sel) o_sel[pos] = pid;
                if (o_log) o_log[pos] = idx;
                pos++;
                if (!(cflag[i] & 1)) ids[rpos++] = pid;
            }
        }
        if (t == 0) {
            *o_n = k;
            *o_kth = thr;
            *o_kp1 = (eq_tot > budget) ? thr : below;
        }
        __threadfence_block();
    };
    bool selected;
    if (prof) g_sa_prof[cta * kSAProfN + 14] = gtimer(p.prof == 2);
    if constexpr (BND) {
        selected = select_cand<NT>(skeys, tm_stage ? stm : nullptr, P, k, p.page_table + u * p.Pmax, o_sel,
                                   o_log, o_n, o_kth, o_kp1, csh, ids, true,
                                   prof ? &g_sa_prof[cta * kSAProfN + 6] : nullptr, true, k + 1, resolve,
                                   skhi, candhi, resolve_cands, p.nchunk == 1 ? sdefer : nullptr,
                                   p.prof == 2);
        // take-all (P <= k) and P > 65536 return before resolving: resolve every page
        if (!selected && (P <= k || P > 65536)) resolve(-1);
    } else {
        selected = select_cand<NT>(skeys, tm_stage ? stm : nullptr, P, k, p.page_table + u * p.Pmax, o_sel,
                                   o_log, o_n, o_kth, o_kp1, csh, ids, true,
                                   prof ? &g_sa_prof[cta * kSAProfN + 6] : nullptr, true);
    }
    const bool deferred = BND && sdefer[0];
    if (!selected)  // take-all, or massive ties at the lower bound
        select_block<NT>(skeys, bins, P, k, p.page_table + u * p.Pmax, o_sel, o_log, o_n,
                                 o_kth, o_kp1, sh, ids, true);
    if constexpr (BND) {  // query fragments from the widened rows (bf16 values: exact)
        const int gq = lane >> 2;
#pragma unroll
        for (int ks = 0; ks < KS; ks++) {
            const int d0 = ks * 16 + 2 * (lane & 3);
            const int g = gq < 8 ? gq : 0;
            qb[ks][0] = gq < G ? pack_bf16(sq[d0 * 8 + g], sq[(d0 + 1) * 8 + g]) : 0u;
            qb[ks][1] = gq < G ? pack_bf16(sq[(d0 + 8) * 8 + g], sq[(d0 + 9) * 8 + g]) : 0u;
        }
    }
    int n_sure = 0;
    if (deferred) {
        // ---- the split: pages with lower key > B are selected whatever their exact key; they
        // go to ids[0 .. n_sure) in logical order (physical ids) and start streaming now, while
        // warps 4-7 resolve the bracket and finish the selection (bounded_tail) ----
        const int C = sdefer[1], B = sdefer[4], A = sdefer[3];
        const int cs = (C + NT - 1) / NT;
        const int i0 = min((int)threadIdx.x * cs, C), i1 = min(i0 + cs, C);
        int cnt = 0;
        for (int i = i0; i < i1; i++) {
            const int lo = (int)(csh.cand[i] >> 16), hi = candhi[i];
            const bool sure = lo > B;
            const bool res = lo != hi && hi >= A && lo <= B;
            cflag[i] = (uint8_t)((sure ? 1 : 0) | (res ? 2 : 0));
            cnt += sure;
        }
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) csh.red[0][warp][0] = (uint32_t)inc;
        __syncthreads();
        int pos = inc - cnt, tot = 0;
#pragma unroll
        for (int w = 0; w < NT / 32; w++) {
            const int t = (int)csh.red[0][w][0];
            if (w < warp) pos += t;
            tot += t;
        }
        for (int i = i0; i < i1; i++)
            if (cflag[i] & 1) ids[pos++] = __ldg(p.page_table + u * p.Pmax + (int)(csh.cand[i] & 0xFFFFu));
        n_sure = tot;
    }
    __syncthreads();  // ids complete (deferred: the certain prefix); the phase-1 scratch is dead
    if (prof) g_sa_prof[cta * kSAProfN + 2] = gtimer(p.prof == 2);

    if (deferred && warp >= NW) {
        // ---- selection tail on warps 4..7 (named barrier 1, 128 threads) ----
        bounded_tail(n_sure);
        asm volatile("bar.arrive 2, %0;" ::"n"(NT) : "memory");  // the remainder is in ids[]
    }

    // ---- this chunk's slice of the selection ----
    const int per = (ns + p.nchunk - 1) / p.nchunk;
    const int first = c * per;
    if (first >= ns) return;
    const int last = min(first + per, ns);
    const int nchunk_u = (ns + per - 1) / per;
    char *my_stages = smem + (size_t)warp * nstage * STAGE_BYTES;
    const int rem = last - first - warp;
    const int my_count = (warp < NW && rem > 0) ? (rem + NW - 1) / NW : 0;
    // deferred: entries >= n_sure exist only after the tail's bar.arrive (each streaming warp
    // waits once, on its first such entry, or at the end)
    bool have_all = !deferred;
    auto ensure = [&](int i) {
        if (!have_all && first + warp + i * NW >= n_sure) {
            asm volatile("bar.sync 2, %0;" ::"n"(NT) : "memory");
            have_all = true;
        }
    };
    const uint64_t kv_pol = p.kv_evict_first ? l2_evict_first_policy() : l2_evict_normal_policy();
    auto issue = [&](int i) {
        const int pid = ids[first + warp + i * NW];
        const int st = i % nstage;
        char *ks = my_stages + (size_t)st * STAGE_BYTES;
        mbar_arrive_expect_tx(&bars[st], STAGE_BYTES);
#pragma unroll
        for (int b = 0; b < D / 64; b++) {
            tma_load_2d_hint(ks + b * S * 128, &tmk, b * 64, pid * S, &bars[st], kv_pol);
            tma_load_2d_hint(ks + PAGE_BYTES + b * S * 128, &tmv, b * 64, pid * S, &bars[st], kv_pol);
        }
    };
    if (warp < NW) {
        if (lane == 0) {
            for (int i = 0; i < nstage; i++) mbar_init(&bars[i], 1);
            fence_mbar_init();
            // the rings reuse the selection scratch written through the generic proxy
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        for (int i = 0; i < min(nstage, my_count); i++) {
            ensure(i);
            if (lane == 0) issue(i);
        }
    }
    __syncwarp();

    const float qscale = p.scale * kLog2e;
    float acc[KS][4];
#pragma unroll
    for (int i = 0; i < KS; i++) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    for (int i = 0; i < my_count; i++) {
        const int st = i % nstage;
        const int pid = ids[first + warp + i * NW];
        const int rows = (pid == tail_pid) ? tail_rows : S;
        mbar_wait(&bars[st], (uint32_t)((i / nstage) & 1));
        if (prof && i == 0) g_sa_prof[cta * kSAProfN + 3] = gtimer(p.prof == 2);
        const uint32_t kbase = smem_u32(my_stages + (size_t)st * STAGE_BYTES);
        mma_page<D, MT>(kbase, kbase + PAGE_BYTES, rows, 0.f, qscale, qb, acc, m_run, l_run, lane);
        __syncwarp();
        if (i + nstage < my_count) {
            ensure(i + nstage);
            if (lane == 0) issue(i + nstage);
        }
    }
    if (warp < NW && !have_all) asm volatile("bar.sync 2, %0;" ::"n"(NT) : "memory");

    // ---- per-warp partials to shared memory, then the CTA / chunk merge (attend.cuh) ----
    if (prof) g_sa_prof[cta * kSAProfN + 4] = gtimer(p.prof == 2);
    __syncthreads();
    float *macc = reinterpret_cast<float *>(smem);             // [NW][8][D]
    float *mml = macc + (size_t)NW * kMmaGP * D;                // [NW][8][2]
    const int g0 = 2 * (lane & 3);
    if (warp < NW) {
#pragma unroll
    for (int dm = 0; dm < KS; dm++) {
        const int d = dm * 16 + (lane >> 2);
        macc[((size_t)warp * kMmaGP + g0) * D + d] = acc[dm][0];
        macc[((size_t)warp * kMmaGP + g0 + 1) * D + d] = acc[dm][1];
        macc[((size_t)warp * kMmaGP + g0) * D + d + 8] = acc[dm][2];
        macc[((size_t)warp * kMmaGP + g0 + 1) * D + d + 8] = acc[dm][3];
    }
    if (lane < 4) {
        mml[(warp * kMmaGP + g0) * 2 + 0] = m_run[0];
        mml[(warp * kMmaGP + g0) * 2 + 1] = l_run[0];
        mml[(warp * kMmaGP + g0 + 1) * 2 + 0] = m_run[1];
        mml[(warp * kMmaGP + g0 + 1) * 2 + 1] = l_run[1];
    }
    }
    __syncthreads();
    AttnParams ap{};
    ap.out = p.out; ap.lse = p.lse; ap.ws = p.ws; ap.tickets = p.tickets;
    ap.G = G; ap.D = D; ap.maxs = kAttnMaxSplits;
    cta_finish(ap, macc, mml, NW, kMmaGP, u, c, nchunk_u);
    if (prof) g_sa_prof[cta * kSAProfN + 5] = gtimer(p.prof == 2);
}

// ---------------------------------------------------------------------------
// Warp-per-unit variant (thousands of short units, small k: cfg4 / short-context cfg5
// shapes).  A CTA-per-unit grid would pay a full CTA selection + merge for a handful of
// pages per warp; here each warp owns one unit end to end: warp-level selection
// (select_warp, keys in registers), then the unit's k pages through the warp's private TMA
// ring, and the final output written directly (no merge).  Warps are independent: no
// __syncthreads after the prologue.
// Shared memory per warp: [ring: nstage stages][ids: kpad ints][mbarriers].
// ---------------------------------------------------------------------------
constexpr int kSWMaxV = 8;  // keys per warp in registers: P <= 32 * 8 * 8 = 2048

template <int D, int MT, bool BND>
__global__ void __launch_bounds__(128, 1) k_select_attend_warp(const __grid_constant__ CUtensorMap tmk,
                                                            const __grid_constant__ CUtensorMap tmv,
                                                            const SelAttnParams p) {
    constexpr int S = 16 * MT;
    constexpr int KS = D / 16;
    constexpr uint32_t PAGE_BYTES = S * D * 2;
    constexpr uint32_t STAGE_BYTES = 2 * PAGE_BYTES;
    extern __shared__ __align__(1024) char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nstage = p.nstage, k = p.k;
    const size_t per_warp = (size_t)p.region;  // ring + ids + bars, 1024-aligned
    char *ring = smem + warp * per_warp;
    int *ids = reinterpret_cast<int *>(ring + (size_t)nstage * STAGE_BYTES);
    uint64_t *bars = reinterpret_cast<uint64_t *>(ids + ((k + 1) & ~1));
    pdl_trigger();
    const int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (u >= p.U) return;
    const bool prof = p.prof && lane == 0 && u < kSAProfCtas;
    const bool pclk = p.prof == 2;
    if (prof) g_sa_prof[u * kSAProfN + 0] = gtimer(pclk);
    // lengths, the tail page and the query fragments are not written by the scoring kernel
    // (the append that wrote them completed before the scorer triggered this launch): read
    // before the PDL wait, beside the scorer's drain, as the CTA-per-unit kernel does
    const int S_ = S;
    const int n = p.seq_len[u];
    const int P = (n + S_ - 1) / S_;
    const int tail_pid = P > 0 ? p.page_table[u * p.Pmax + P - 1] : -1;
    const int tail_rows = n - (P - 1) * S_;
    uint32_t qb[KS][2];
    {
        const int gq = lane >> 2;
#pragma unroll
        for (int ks = 0; ks < KS; ks++) {
            const int d0 = ks * 16 + 2 * (lane & 3);
            uint32_t b0 = 0, b1 = 0;
            if (gq < p.G) {
                const int64_t row = (u * p.G + gq) * (int64_t)D;
                if (p.q_dtype == PT_BF16) {
                    const uint32_t *qp =
                        reinterpret_cast<const uint32_t *>(static_cast<const uint16_t *>(p.q) + row);
                    b0 = __ldg(qp + (d0 >> 1));
                    b1 = __ldg(qp + ((d0 + 8) >> 1));
                } else {
                    const float *qp = static_cast<const float *>(p.q) + row;
                    b0 = pack_bf16(qp[d0], qp[d0 + 1]);
                    b1 = pack_bf16(qp[d0 + 8], qp[d0 + 9]);
                }
            }
            qb[ks][0] = b0;
            qb[ks][1] = b1;
        }
    }
    // bounded: the query rows as f32 [D][8] at the end of the (still unused) ring, for the
    // resolution's exact sums (not written by the scorer: before the PDL wait)
    float *qsw = reinterpret_cast<float *>(ring + (size_t)nstage * STAGE_BYTES) - D * 8;
    if constexpr (BND) {
        for (int i = lane; i < D * 8; i += 32) {
            const int d = i >> 3, g = i & 7;
            float x = 0.f;
            if (g < p.G) {
                const int64_t e = (u * p.G + g) * (int64_t)D + d;
                x = p.q_dtype == PT_BF16 ? bf16_bits_to_f32(static_cast<const uint16_t *>(p.q)[e])
                                         : static_cast<const float *>(p.q)[e];
            }
            qsw[i] = x;
        }
        __syncwarp();
    }
    pdl_wait();
    if (prof) g_sa_prof[u * kSAProfN + 1] = gtimer(pclk);
    if (P == 0) {
        if (lane == 0) { p.n_sel[u] = 0; p.kth[u] = 0; p.kplus1[u] = -1; }
        return;
    }
    if constexpr (BND) {
        // bounded keys: the exact key of a bracket page, one lane per page
        auto exact = [&](int pg) -> int {
            const float *row = p.rows32 + ((int64_t)u * p.Pmax + pg) * D;
            const float sd = __ldg(p.stds + u * (int64_t)p.Pmax + pg);
            const float best = p.G <= 4 ? sa_exact_score_rowg<D, 4>(row, qsw, p.lamnorm + u * 8, sd, p.G)
                                        : sa_exact_score_rowg<D, 8>(row, qsw, p.lamnorm + u * 8, sd, p.G);
            return (int)encode_ordered(f32_to_bf16_rne(best));
        };
        select_warp<kSWMaxV>(p.keys + u * (int64_t)p.Pmax, P, k, p.page_table + u * p.Pmax,
                             p.sel + u * (int64_t)k, p.sel_logical ? p.sel_logical + u * (int64_t)k : nullptr,
                             p.n_sel + u, p.kth + u, p.kplus1 + u, ids, p.keys_hi + u * (int64_t)p.Pmax,
                             exact, reinterpret_cast<int *>(ring), (int)(nstage * STAGE_BYTES / 4) - D * 8,
                             p.tile_max ? p.tile_max + u * (int64_t)(p.Pmax >> 5) : nullptr,
                             prof && pclk ? &g_sa_prof[u * kSAProfN] : nullptr,
                             [&](int pg) {  // the page's f32 row and std into L1
                                 const char *row = reinterpret_cast<const char *>(
                                     p.rows32 + ((int64_t)u * p.Pmax + pg) * D);
#pragma unroll
                                 for (int l = 0; l < D * 4 / 128; l++)
                                     asm volatile("prefetch.global.L1 [%0];" ::"l"(row + 128 * l));
                                 asm volatile("prefetch.global.L1 [%0];" ::"l"(p.stds + u * (int64_t)p.Pmax + pg));
                             });
    } else {
        select_warp<kSWMaxV>(p.keys + u * (int64_t)p.Pmax, P, k, p.page_table + u * p.Pmax,
                             p.sel + u * (int64_t)k, p.sel_logical ? p.sel_logical + u * (int64_t)k : nullptr,
                             p.n_sel + u, p.kth + u, p.kplus1 + u, ids, nullptr, NoExactKey(), nullptr, 0,
                             p.tile_max ? p.tile_max + u * (int64_t)(p.Pmax >> 5) : nullptr,
                             prof && pclk ? &g_sa_prof[u * kSAProfN] : nullptr);
    }
    if (prof) g_sa_prof[u * kSAProfN + 2] = gtimer(pclk);
    const int ns = P < k ? P : k;
    const uint64_t kv_pol = p.kv_evict_first ? l2_evict_first_policy() : l2_evict_normal_policy();
    auto issue = [&](int i) {
        const int pid = ids[i];
        const int st = i % nstage;
        char *ks = ring + (size_t)st * STAGE_BYTES;
        mbar_arrive_expect_tx(&bars[st], STAGE_BYTES);
#pragma unroll
        for (int b = 0; b < D / 64; b++) {
            tma_load_2d_hint(ks + b * S * 128, &tmk, b * 64, pid * S, &bars[st], kv_pol);
            tma_load_2d_hint(ks + PAGE_BYTES + b * S * 128, &tmv, b * 64, pid * S, &bars[st], kv_pol);
        }
    };
    if (lane == 0) {
        for (int i = 0; i < nstage; i++) mbar_init(&bars[i], 1);
        fence_mbar_init();
        // the ring held the bounded selection's generic-proxy scratch: order it before the TMA
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int i = 0; i < min(nstage, ns); i++) issue(i);
    }
    __syncwarp();
    const float qscale = p.scale * kLog2e;
    float acc[KS][4];
#pragma unroll
    for (int i = 0; i < KS; i++) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    for (int i = 0; i < ns; i++) {
        const int st = i % nstage;
        const int pid = ids[i];
        const int rows = (pid == tail_pid) ? tail_rows : S;
        mbar_wait(&bars[st], (uint32_t)((i / nstage) & 1));
        if (prof && i == 0) g_sa_prof[u * kSAProfN + 3] = gtimer(pclk);
        const uint32_t kbase = smem_u32(ring + (size_t)st * STAGE_BYTES);
        mma_page<D, MT>(kbase, kbase + PAGE_BYTES, rows, 0.f, qscale, qb, acc, m_run, l_run, lane);
        __syncwarp();
        if (lane == 0 && i + nstage < ns) issue(i + nstage);
    }
    if (prof) g_sa_prof[u * kSAProfN + 4] = gtimer(pclk);
    const int g0 = 2 * (lane & 3);
    const float inv0 = 1.f / l_run[0], inv1 = 1.f / l_run[1];
#pragma unroll
    for (int dm = 0; dm < KS; dm++) {
        const int d = dm * 16 + (lane >> 2);
        if (g0 < p.G) {
            p.out[(u * p.G + g0) * D + d] = acc[dm][0] * inv0;
            p.out[(u * p.G + g0) * D + d + 8] = acc[dm][2] * inv0;
        }
        if (g0 + 1 < p.G) {
            p.out[(u * p.G + g0 + 1) * D + d] = acc[dm][1] * inv1;
            p.out[(u * p.G + g0 + 1) * D + d + 8] = acc[dm][3] * inv1;
        }
    }
    if (lane < 4) {
        if (g0 < p.G) p.lse[u * p.G + g0] = (m_run[0] + log2f(l_run[0])) * kLn2;
        if (g0 + 1 < p.G) p.lse[u * p.G + g0 + 1] = (m_run[1] + log2f(l_run[1])) * kLn2;
    }
    if (prof) g_sa_prof[u * kSAProfN + 5] = gtimer(pclk);
}

template <int D, int MT, bool BND>
static int launch_saw(const CUtensorMap &tk, const CUtensorMap &tv, const SelAttnParams &p, int nw,
                      size_t smem, cudaStream_t st) {
    static size_t configured = 0;
    if (smem > configured) {
        PT_CUDA_TRY(cudaFuncSetAttribute(k_select_attend_warp<D, MT, BND>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    dim3 grid((p.U + nw - 1) / nw);
    PT_CUDA_TRY(pt_launch(k_select_attend_warp<D, MT, BND>, grid, dim3(nw * 32), smem, st, tk, tv, p));
    return PT_OK;
}

template <int D, int MT, int NT, bool BND>
static int launch_sa_nt(const CUtensorMap &tk, const CUtensorMap &tv, const SelAttnParams &p,
                        size_t smem, cudaStream_t st) {
    static size_t configured = 0;
    if (smem > configured) {
        PT_CUDA_TRY(cudaFuncSetAttribute(k_select_attend<D, MT, NT, BND>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    dim3 grid(p.nchunk, p.U);
    PT_CUDA_TRY(pt_launch(k_select_attend<D, MT, NT, BND>, grid, dim3(NT), smem, st, tk, tv, p));
    return PT_OK;
}

template <int D, int MT>
static int launch_sa(const CUtensorMap &tk, const CUtensorMap &tv, const SelAttnParams &p,
                     size_t smem, cudaStream_t st, int sel_threads) {
    if (p.keys_hi) return launch_sa_nt<D, MT, 256, true>(tk, tv, p, smem, st);
    return sel_threads == 256 ? launch_sa_nt<D, MT, 256, false>(tk, tv, p, smem, st)
                              : launch_sa_nt<D, MT, 128, false>(tk, tv, p, smem, st);
}

}  // namespace pt

using namespace pt;

bool pt_make_pool_tmap(CUtensorMap *m, const void *pool, int D, int S, int num_pages);

static int sa_env_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}

// Selection + sparse attention for every unit in one launch.  Same outputs as pt_topk
// followed by pt_attend (sel_stride = k); PT_ERR_UNSUPPORTED when the shape is outside the
// fused kernel's envelope (the caller then runs the two-launch path).
extern "C" int pt_select_attend(const uint16_t *keys, const uint16_t *tile_max,
                                const uint16_t *keys_hi, const void *mirror, const float *stds,
                                const float *lamnorm, const int32_t *seq_len,
                                const int32_t *page_table, int U_all, int u0, int nu, int S, int Pmax,
                                int k, int32_t *sel, int32_t *sel_logical, int32_t *n_sel, int32_t *kth,
                                int32_t *kplus1, const void *q, int q_dtype, const void *k_pool,
                                const void *v_pool, int kv_dtype, int num_phys_pages, int G, int D,
                                float scale, float *out, float *lse, void *workspace,
                                size_t workspace_bytes, int32_t *tickets, void *stream) {
    if (!keys || !seq_len || !page_table || !sel || !n_sel || !kth || !kplus1 || !q || !k_pool ||
        !v_pool || !out || !lse || U_all < 0 || u0 < 0 || nu < 0 || u0 + nu > U_all || S < 1 ||
        Pmax % 32 || G < 1)
        return PT_ERR_INVALID;
    if (k < 1) return PT_ERR_K;
    if (nu == 0) return PT_OK;
    // units [u0, u0 + nu) of a U_all-unit cache: every per-unit array from u0 on (the
    // workspace by its per-unit share), so two disjoint ranges can run concurrently
    const float *rows_all = mirror ? mirror_view(mirror, U_all, Pmax, D).rows : nullptr;
    {
        const int64_t o = u0;
        keys += o * Pmax; seq_len += o; page_table += o * Pmax;
        sel += o * k; n_sel += o; kth += o; kplus1 += o; tickets += o;
        if (tile_max) tile_max += o * (Pmax / 32);
        if (keys_hi) keys_hi += o * Pmax;
        if (stds) stds += o * Pmax;
        if (lamnorm) lamnorm += o * 8;
        if (sel_logical) sel_logical += o * k;
        if (rows_all) rows_all += o * Pmax * D;
        q = static_cast<const char *>(q) + o * G * D * (q_dtype == PT_F32 ? 4 : 2);
        out += o * G * D; lse += o * G;
        const size_t wsh = pt_attend_workspace_bytes((int)o, G, D, k);
        if (workspace_bytes < wsh) return PT_ERR_UNSUPPORTED;
        workspace = static_cast<char *>(workspace) + wsh;
        workspace_bytes -= wsh;
    }
    const int U = nu;
    if (kv_dtype != PT_BF16 || G > 8 || !(D == 64 || D == 128 || D == 256) ||
        !(S == 16 || S == 32 || S == 64) || num_phys_pages <= 0 || !workspace || !tickets ||
        workspace_bytes < pt_attend_workspace_bytes(U, G, D, k) || sa_env_int("PT_NO_FUSED_SA", 0))
        return PT_ERR_UNSUPPORTED;
    const bool bnd = keys_hi != nullptr;
    if (bnd && (!mirror || !stds || !lamnorm || !tile_max)) return PT_ERR_INVALID;
    // bounded mode streams while its selection tail runs (early streaming): a 2-deep ring
    // (measured no slower than 3 at cfg3: 176 vs 180 us/step) below the tail's scratch
    const int stage = 2 * S * D * 2;
    int nstage = sa_env_int("PT_SA_NSTAGE", bnd ? 2 : 3);
    if (nstage < 1) nstage = 1;
    // chunks per unit: fill the resident CTA slots (2 per SM) without a second wave, and
    // keep at least one page per warp in a chunk
    int nchunk = sa_env_int("PT_SA_CHUNKS", 0);
    if (nchunk <= 0) {
        nchunk = (pt_num_sms() * 2) / U;
        if (nchunk < 1) nchunk = 1;
        // every chunk CTA repeats the unit's selection: keep >= 4 pages per warp per chunk
        const int cap = (k + 4 * kSAWarps - 1) / (4 * kSAWarps);
        if (nchunk > cap) nchunk = cap;
    }
    if (nchunk > kAttnMaxSplits) nchunk = kAttnMaxSplits;
    const size_t sel_base = sa_keys_bytes(Pmax) + (size_t)kSelectBins * 4 + (size_t)(Pmax / 32) * 2;
    size_t sel_scratch = sel_base, region_lo = 0;
    int rcap = 0;
    if (bnd) {
        // lower part: the phase-1 arrays, then the stage rings; upper part: the selection
        // tail's scratch, with as many resolve rows per round as keep the dynamic shared
        // memory at <= 100 KB (two CTAs per SM beside ~9 KB of static selection state)
        const size_t lower = ((sel_base + 15) & ~(size_t)15) + sa_keys_bytes(Pmax) + (size_t)kCandMax * 2;
        const size_t rings = (size_t)kSAWarps * nstage * stage;
        region_lo = ((lower > rings ? lower : rings) + 1023) & ~(size_t)1023;
        const size_t fixed = (size_t)D * 32 + 32 + 16 + 16 + kCandMax;
        const size_t tail = (size_t)100 * 1024 - region_lo - fixed - (((size_t)k * 4 + 7) & ~(size_t)7) -
                            (size_t)kSAWarps * nstage * 8;
        rcap = (size_t)100 * 1024 > region_lo + fixed ? (int)(tail / ((size_t)(D + 4) * 4 + 8)) : 0;
        rcap = sa_env_int("PT_SA_RCAP", rcap);
        rcap = (rcap < 32 ? 32 : rcap > 256 ? 256 : rcap) & ~3;
        sel_scratch = region_lo + fixed + (size_t)rcap * ((size_t)(D + 4) * 4 + 8);
    }
    const size_t merge = (size_t)kSAWarps * kMmaGP * (D + 2) * 4;
    auto smem_of = [&](int nst, size_t *region_out) {
        const size_t rings = (size_t)kSAWarps * nst * stage;
        size_t region = rings > sel_scratch ? rings : sel_scratch;
        if (merge > region) region = merge;
        region = (region + 1023) & ~(size_t)1023;
        if (region_out) *region_out = region;
        return region + (((size_t)k * 4 + 7) & ~(size_t)7) + (size_t)kSAWarps * nst * 8;
    };
    // ring depth: keep two CTAs per SM where a 2-deep ring allows, else fit one CTA
    while (nstage > 2 && smem_of(nstage, nullptr) > 113 * 1024) nstage--;
    while (nstage > 1 && smem_of(nstage, nullptr) > 225 * 1024) nstage--;
    size_t region = 0;
    const size_t smem = smem_of(nstage, &region);
    if (smem > 225 * 1024) return PT_ERR_UNSUPPORTED;
    // many short units with a small budget: one warp per unit (no CTA-wide selection/merge)
    const int want_warp = sa_env_int("PT_SA_WARP", -1);
    const bool warp_path = want_warp == 1 ||
                           (want_warp != 0 && U >= 4 * pt_num_sms() && k <= 64 && Pmax <= 32 * 8 * kSWMaxV);
    size_t w_per = 0;
    // ring depth (PT_SAW_NSTAGE: tuning; a 2-deep ring measured no faster at k = 8)
    int w_nst = sa_env_int("PT_SAW_NSTAGE", 3), w_nw = 4;
    if (warp_path && Pmax <= 32 * 8 * kSWMaxV) {
        auto per_of = [&](int nst) {
            return ((size_t)nst * stage + (((size_t)k + 1) & ~(size_t)1) * 4 + (size_t)nst * 8 + 1023) &
                   ~(size_t)1023;
        };
        while (w_nst > 2 && per_of(w_nst) * w_nw > 113 * 1024) w_nst--;
        while (w_nw > 1 && per_of(w_nst) * w_nw > 225 * 1024) w_nw--;
        if (per_of(w_nst) * w_nw <= 225 * 1024) w_per = per_of(w_nst);
    }
    CUtensorMap tk, tv;
    if (!pt_make_pool_tmap(&tk, k_pool, D, S, num_phys_pages) ||
        !pt_make_pool_tmap(&tv, v_pool, D, S, num_phys_pages))
        return PT_ERR_UNSUPPORTED;
    SelAttnParams p{};
    p.keys = keys; p.tile_max = tile_max; p.seq_len = seq_len; p.page_table = page_table;
    p.sel = sel; p.sel_logical = sel_logical; p.n_sel = n_sel; p.kth = kth; p.kplus1 = kplus1;
    p.q = q; p.out = out; p.lse = lse; p.ws = static_cast<float *>(workspace); p.tickets = tickets;
    p.q_dtype = q_dtype; p.U = U; p.G = G; p.Pmax = Pmax; p.k = k; p.nchunk = nchunk;
    p.nstage = nstage; p.region = (int)region; p.scale = scale;
    p.prof = sa_env_int("PT_SA_PROF", 0);
    p.kv_evict_first = sa_env_int("PT_SA_KV_EVICT_FIRST", 1);
    p.keys_hi = keys_hi; p.rows32 = rows_all;
    p.region_lo = (int)region_lo; p.stds = stds; p.lamnorm = lamnorm; p.rcap = rcap;
    cudaStream_t st = (cudaStream_t)stream;
    // selection threads: 8 warps halve the selection's block-wide passes; 4 of them stream
    const int sel_threads = sa_env_int("PT_SA_SEL_THREADS", 256) == 128 ? 128 : 256;
    if (w_per) {
        SelAttnParams pw = p;
        pw.nstage = w_nst;
        pw.region = (int)w_per;
#define PT_SAW(D_, MT_) \
        if (D == D_ && S == 16 * MT_)                                                                 \
            return bnd ? launch_saw<D_, MT_, true>(tk, tv, pw, w_nw, w_per * w_nw, st)                  \
                       : launch_saw<D_, MT_, false>(tk, tv, pw, w_nw, w_per * w_nw, st);
        PT_SAW(64, 1) PT_SAW(64, 2) PT_SAW(64, 4)
        PT_SAW(128, 1) PT_SAW(128, 2) PT_SAW(128, 4)
        PT_SAW(256, 1) PT_SAW(256, 2) PT_SAW(256, 4)
#undef PT_SAW
    }
#define PT_SA(D_, MT_) \
    if (D == D_ && S == 16 * MT_) return launch_sa<D_, MT_>(tk, tv, p, smem, st, sel_threads);
    PT_SA(64, 1) PT_SA(64, 2) PT_SA(64, 4)
    PT_SA(128, 1) PT_SA(128, 2) PT_SA(128, 4)
    PT_SA(256, 1) PT_SA(256, 2) PT_SA(256, 4)
#undef PT_SA
    return PT_ERR_UNSUPPORTED;
}

// tuning aid: copy the phase timestamps of the last PT_SA_PROF=1 launch (n <= 10 * 4096)
extern "C" int pt_debug_sa_prof(unsigned long long *host, int n) {
    if (!host || n < 0 || n > kSAProfCtas * kSAProfN) return PT_ERR_INVALID;
    PT_CUDA_TRY(cudaMemcpyFromSymbol(host, g_sa_prof, (size_t)n * 8));
    return PT_OK;
}
