// score.cu -- K2: offset-augmented page scoring with the GQA group max, fused with the
// bf16 rounding and the order-preserving key encoding of the selection stage.
//
// Restates, per page p of unit u (query group g = 0..G-1):
//   scoring.py:39-47   norm_g = f32(sqrt(np.sum(f64(q_g)**2)))        (unless given)
//   _kernels_cy.pyx:19-43
//       acc = 0; for d: acc = fl(acc + fl(q[g,d] * mean[p,d]))     (sequential d)
//       acc = fl(acc + fl(fl(lam * norm_g) * std[p]));  best = max_g (strict >)
//   bf16.py:18-33      f32 -> bf16 RNE;   select.py:51-57  ordered u16 key
// The sequential per-page chain is kept (one thread = one page, G independent chains
// for ILP) so the f32 scores are bit-identical to the reference's compiled backend.
// Fusion: one launch reads each page's stats once and writes one key per page
// (traffic_of_fused, scoring.py:146-156); keys go straight to the top-k kernel.
//
// Memory layout: the page-interleaved tile layout of the means (common.cuh) makes each
// warp-wide step one contiguous 512-byte, 128-bit-per-lane load with lane = page.
#include <stdlib.h>

#include "score_stream.cuh"
#include "select.cuh"

namespace pt {

constexpr int kScoreMaxD = 256;

template <int SDT>
struct MeanVec;
template <>
struct MeanVec<PT_F32> {
    static constexpr int V = 4;
    __device__ __forceinline__ static void load(const void *p, float (&m)[4]) {
        float4 v = __ldg(static_cast<const float4 *>(p));
        m[0] = v.x; m[1] = v.y; m[2] = v.z; m[3] = v.w;
    }
};
template <>
struct MeanVec<PT_BF16> {
    static constexpr int V = 8;
    __device__ __forceinline__ static void load(const void *p, float (&m)[8]) {
        uint4 v = __ldg(static_cast<const uint4 *>(p));
        m[0] = bf16_lo(v.x); m[1] = bf16_hi(v.x); m[2] = bf16_lo(v.y); m[3] = bf16_hi(v.y);
        m[4] = bf16_lo(v.z); m[5] = bf16_hi(v.z); m[6] = bf16_lo(v.w); m[7] = bf16_hi(v.w);
    }
};

// Q products are exact in f32 when both factors are bf16 values (8-bit significands):
// then fma(q, m, acc) == fl(acc + q*m) and one FFMA replaces FMUL+FADD.
//
// Memory pipeline: a CTA owns TILES page tiles (32 pages each) of one unit.  At entry one
// thread issues every byte the CTA will read as 1-D bulk copies (cp.async.bulk, SASS
// UBLKCP) -- the tile layout makes each (tile, d-range) a single contiguous block --
// split into NST d-range stages with one mbarrier each, so compute on the first dims
// starts while the rest is in flight (64 KB in flight per CTA, 3 CTAs per SM).  Threads
// then read their page's 16-byte chunks from shared memory (lane-contiguous, no bank
// conflicts) in the reference's sequential d order.
constexpr int kScoreStages = 4;

struct ScoreParams {
    const void *q;
    const float *norms_in;
    const void *means;
    const float *stds;
    const int32_t *seq_len;
    uint16_t *keys;
    float *scores;
    // fused selection (counters == nullptr: scoring only)
    int32_t *counters;
    const int32_t *page_table;
    int32_t *sel, *sel_logical, *n_sel, *kth, *kplus1;
    int D, S, Pmax, k;
    float lam;
    uint16_t *tile_max;  // [U][Pmax/32] or null
};

constexpr int kFusedThreads = 128;  // the fused selection runs with the 4-tile CTA

template <int QDT, int SDT, int G>
__global__ void __launch_bounds__(128) k_score(const ScoreParams prm) {
    const void *__restrict__ q = prm.q;
    const float *__restrict__ norms_in = prm.norms_in;
    const void *__restrict__ means = prm.means;
    const float *__restrict__ stds = prm.stds;
    const int D = prm.D, S = prm.S, Pmax = prm.Pmax;
    const float lam = prm.lam;
    uint16_t *__restrict__ keys = prm.keys;
    float *__restrict__ scores = prm.scores;
    constexpr int V = MeanVec<SDT>::V;
    constexpr int ES = SDT == PT_F32 ? 4 : 2;
    constexpr bool kExactProduct = (QDT == PT_BF16 && SDT == PT_BF16);
    extern __shared__ __align__(128) char tiles[];
    __shared__ __align__(16) float qs[G][kScoreMaxD];
    __shared__ float lam_norm[G];
    __shared__ uint64_t bars[kScoreStages];
    const int64_t u = blockIdx.y;
    const int tid = threadIdx.x;
    const int TILES = blockDim.x >> 5;
    const int n = prm.seq_len[u];
    const int P = (n + S - 1) / S;
    const int64_t p0 = (int64_t)blockIdx.x * blockDim.x;
    if (p0 >= P) return;
    const int nch = D / V;                                   // 16-byte chunks per page row
    const int cps = (nch + kScoreStages - 1) / kScoreStages; // chunks per stage
    const int nst = (nch + cps - 1) / cps;
    const int tile_bytes = 32 * D * ES;
    const int ntiles = min(TILES, (int)((P - p0 + 31) >> 5));
    const char *gbase = static_cast<const char *>(means) +
                        (u * Pmax * D + (p0 >> 5) * 32 * (int64_t)D) * ES;
    if (tid == 0) {  // first thing: put every byte of this CTA in flight
        for (int st = 0; st < nst; st++) mbar_init(&bars[st], 1);
        fence_mbar_init();
        for (int st = 0; st < nst; st++) {
            const int c0 = st * cps, c1 = min(nch, c0 + cps);
            const uint32_t bytes = (uint32_t)(c1 - c0) * 512;
            mbar_arrive_expect_tx(&bars[st], bytes * ntiles);
            for (int t = 0; t < ntiles; t++)
                bulk_g2s(tiles + t * tile_bytes + c0 * 512, gbase + (int64_t)t * tile_bytes + c0 * 512,
                         bytes, &bars[st]);
        }
    }
    for (int i = tid; i < G * D; i += blockDim.x) {
        const int g = i / D, d = i % D;
        qs[g][d] = load_elem<QDT>(q, (u * G + g) * (int64_t)D + d);
    }
    __syncthreads();
    if (tid < G) {  // overlaps the copies in flight
        const float nrm = norms_in ? norms_in[u * G + tid]
                                   : __double2float_rn(__dsqrt_rn(np_sum(SquaresOfF32{qs[tid]}, D)));
        lam_norm[tid] = __fmul_rn(lam, nrm);
    }
    __syncthreads();

    const int64_t p = p0 + tid;
    const bool live = p < P;
    const char *mp = tiles + (tid >> 5) * tile_bytes + (tid & 31) * 16;
    float acc[G];
#pragma unroll
    for (int g = 0; g < G; g++) acc[g] = 0.0f;
    for (int st = 0; st < nst; st++) {
        mbar_wait(&bars[st], 0);  // every thread waits: no copy outlives the CTA
        if (!live) continue;
        const int c0 = st * cps, c1 = min(nch, c0 + cps);
#pragma unroll 4
        for (int c = c0; c < c1; c++) {
            float m[V];
            if constexpr (SDT == PT_F32) {
                const float4 v = *reinterpret_cast<const float4 *>(mp + c * 512);
                m[0] = v.x; m[1] = v.y; m[2] = v.z; m[3] = v.w;
            } else {
                const uint4 v = *reinterpret_cast<const uint4 *>(mp + c * 512);
                m[0] = bf16_lo(v.x); m[1] = bf16_hi(v.x); m[2] = bf16_lo(v.y); m[3] = bf16_hi(v.y);
                m[4] = bf16_lo(v.z); m[5] = bf16_hi(v.z); m[6] = bf16_lo(v.w); m[7] = bf16_hi(v.w);
            }
#pragma unroll
            for (int j = 0; j < V; j++) {
                const int d = c * V + j;
#pragma unroll
                for (int g = 0; g < G; g++) {
                    if constexpr (kExactProduct) acc[g] = __fmaf_rn(qs[g][d], m[j], acc[g]);
                    else acc[g] = __fadd_rn(acc[g], __fmul_rn(qs[g][d], m[j]));
                }
            }
        }
    }
    if (live) {
        const float sd = stds[u * Pmax + p];
        float best = -INFINITY;
#pragma unroll
        for (int g = 0; g < G; g++) {
            const float a = __fadd_rn(acc[g], __fmul_rn(lam_norm[g], sd));
            if (a > best) best = a;
        }
        keys[u * Pmax + p] = encode_ordered(f32_to_bf16_rne(best));
        if (scores) scores[u * Pmax + p] = best;
    }
    if (prm.tile_max) {  // warp = one 32-page tile (p0 is a multiple of 32)
        const uint32_t key = live ? (uint32_t)keys[u * Pmax + p] : 0u;
        const uint32_t m = __reduce_max_sync(0xffffffffu, key);
        if ((tid & 31) == 0 && p < P) prm.tile_max[u * (Pmax >> 5) + (p >> 5)] = (uint16_t)m;
    }
    if (prm.counters == nullptr) return;

    // ---- fused selection: the last CTA to finish scoring unit u selects its top-k ----
    // (select.py:87-115 via select.cuh) while other CTAs keep streaming other units.
    __shared__ int is_last;
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const int nblk = (P + blockDim.x - 1) / blockDim.x;
        is_last = (atomicAdd(&prm.counters[u], 1) == nblk - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    if (tid == 0) prm.counters[u] = 0;  // self-resetting for graph replay
    uint16_t *sk = reinterpret_cast<uint16_t *>(tiles);  // page tiles are consumed: reuse
    const uint4 *src = reinterpret_cast<const uint4 *>(keys + u * (int64_t)Pmax);
    for (int i = tid; i < (P + 7) / 8; i += blockDim.x)
        reinterpret_cast<uint4 *>(sk)[i] = __ldcg(src + i);
    __syncthreads();
    __shared__ SelectShared<kFusedThreads> ssh;
    __shared__ int sbins[kSelectBins];
    const int k = prm.k;
    select_block<kFusedThreads>(sk, sbins, P, k, prm.page_table + u * Pmax, prm.sel + u * (int64_t)k,
                                prm.sel_logical ? prm.sel_logical + u * (int64_t)k : nullptr,
                                prm.n_sel + u, prm.kth + u, prm.kplus1 + u, ssh);
}



// lam * ||q_g|| for every (unit, g), numpy's float64 order (scoring.py:45), padded to 8.
// A CTA stages kLnRows query rows in shared memory with coalesced loads (one load round),
// then thread r runs numpy's pairwise float64 sum over row r from shared memory -- the
// accessor-driven sum over global memory would be a chain of dependent load rounds.
constexpr int kLnRows = 32;
// LATE (pt_lam_norms_chained): the kernel reads only q, so it runs beside the kernel launched
// before it and takes its PDL wait at the very end -- it completes only after that kernel, so
// a PDL successor that waits on it also sees the earlier kernel's writes (a straight chain
// append -> norms -> score instead of a fork/join of two streams).
template <int QDT, bool LATE = false>
__global__ void __launch_bounds__(256) k_lam_norms(const void *__restrict__ q,
                                                   const float *__restrict__ norms_in, int rows,
                                                   int G, int D, float lam, float *__restrict__ out,
                                                   float *__restrict__ qnorm) {
    __shared__ float qs[kLnRows * (kScoreMaxD + 1)];
    pdl_trigger();
    if (!LATE) pdl_wait();
    const int r0 = blockIdx.x * kLnRows;
    const int nr = min(kLnRows, rows - r0);
    const int ld = D + 1;  // odd stride: thread r's sequential reads hit distinct banks
    if (!norms_in || qnorm) {
        const char *src = static_cast<const char *>(q) + (int64_t)r0 * D * (QDT == PT_F32 ? 4 : 2);
        stage_rows_f32<QDT, 8>(qs, ld, src, nr * D, D, threadIdx.x, blockDim.x);
    }
    __syncthreads();
    const int r = threadIdx.x;
    float val = 0.f, qn = 0.f;
    if (r < nr) {
        float nrm = 0.f;
        double ss = 0.0;
        if (!norms_in || qnorm) {
            struct Sq {
                const float *row;
                __device__ double operator()(int i) const {
                    const double v = (double)row[i];
                    return __dmul_rn(v, v);
                }
            } sq{qs + r * ld};
            ss = np_sum(sq, D);
        }
        nrm = norms_in ? norms_in[r0 + r] : __double2float_rn(__dsqrt_rn(ss));
        val = __fmul_rn(lam, nrm);
        // bounded scoring: an upper bound of the true ||q_g|| (f64 sum of exact squares,
        // relative error < 1e-13, then rounded up)
        qn = __double2float_ru(__dsqrt_ru(ss) * (1.0 + 0x1p-30));
    }
    // LATE: the norms are computed beside the predecessor, but stored only after its wait --
    // the previous step's scorer may still be reading lamnorm until then (WAR across steps)
    if (LATE) pdl_wait();
    if (r < nr) {
        const int u = (r0 + r) / G, g = (r0 + r) - u * G;
        out[(int64_t)u * 8 + g] = val;
        if (qnorm) qnorm[(int64_t)u * 8 + g] = qn;
    }
}

// row-major f32 means [U][P][D] -> tiled stats layout (stats dtype)
template <int SDT>
__global__ void k_tile_means(const float *__restrict__ src, int U, int P, int D, int Pmax,
                             void *__restrict__ dst) {
    constexpr int V = SDT == PT_F32 ? 4 : 8;
    const int64_t total = (int64_t)U * P * D;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t u = i / ((int64_t)P * D);
        const int64_t r = i % ((int64_t)P * D);
        const int64_t p = r / D;
        const int d = (int)(r % D);
        store_elem<SDT>(dst, mean_offset(u, p, d, D, Pmax, V), src[i]);
    }
}

}  // namespace pt

using namespace pt;

// tiles per CTA: 64 KB of page means per CTA (3 CTAs per SM)
static int score_tiles(int D, int es) {
    const int tile = 32 * D * es;
    int t = 65536 / tile;
    return t < 1 ? 1 : (t > 4 ? 4 : t);
}

template <int QDT, int SDT>
static int launch_score(ScoreParams prm, int U, int G, cudaStream_t st) {
    const int es = SDT == PT_F32 ? 4 : 2;
    const int tiles = score_tiles(prm.D, es);
    const int threads = 32 * tiles;
    const size_t smem = (size_t)tiles * 32 * prm.D * es;
    if (prm.counters && (threads != kFusedThreads || (size_t)(prm.Pmax + 8) * 2 > smem))
        return PT_ERR_UNSUPPORTED;  // caller falls back to pt_score + pt_topk
    dim3 grid((prm.Pmax + threads - 1) / threads, U);
#define PT_SCORE_CASE(G_)                                                                      \
    case G_: {                                                                                 \
        static size_t configured = 0;                                                          \
        if (smem > configured) { /* dynamic + static may pass 48 KB */                    \
            PT_CUDA_TRY(cudaFuncSetAttribute(k_score<QDT, SDT, G_>,                            \
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                             (int)smem));                                      \
            configured = smem;                                                                 \
        }                                                                                      \
        k_score<QDT, SDT, G_><<<grid, threads, smem, st>>>(prm);                               \
        break;                                                                                 \
    }
    switch (G) {
        PT_SCORE_CASE(1)
        PT_SCORE_CASE(2)
        PT_SCORE_CASE(3)
        PT_SCORE_CASE(4)
        PT_SCORE_CASE(5)
        PT_SCORE_CASE(6)
        PT_SCORE_CASE(7)
        PT_SCORE_CASE(8)
        default: return PT_ERR_UNSUPPORTED;
    }
#undef PT_SCORE_CASE
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}

static int dispatch_score(const ScoreParams &prm, int q_dtype, int stats_dtype, int U, int G,
                          cudaStream_t st) {
    if (q_dtype == PT_F32 && stats_dtype == PT_F32) return launch_score<PT_F32, PT_F32>(prm, U, G, st);
    if (q_dtype == PT_BF16 && stats_dtype == PT_F32) return launch_score<PT_BF16, PT_F32>(prm, U, G, st);
    if (q_dtype == PT_BF16 && stats_dtype == PT_BF16) return launch_score<PT_BF16, PT_BF16>(prm, U, G, st);
    if (q_dtype == PT_F32 && stats_dtype == PT_BF16) return launch_score<PT_F32, PT_BF16>(prm, U, G, st);
    return PT_ERR_INVALID;
}

namespace pt {
int launch_score_stream_q32(const StreamScoreParams &sp, int sdt, int G, int D, cudaStream_t st);
int launch_score_stream_q16(const StreamScoreParams &sp, int sdt, int G, int D, cudaStream_t st);
}  // namespace pt

extern "C" int pt_score(const void *q, int q_dtype, const float *norms, const void *means,
                        int stats_dtype, const float *stds, const int32_t *seq_len, int U, int G,
                        int D, int S, int Pmax, float lam, uint16_t *keys, float *scores,
                        float *lamnorm_ws, uint16_t *tile_max, void *stream) {
    if (!q || !means || !stds || !seq_len || !keys || U < 0 || S < 1 || Pmax % 32 || G < 1)
        return PT_ERR_INVALID;
    const int V = stats_dtype == PT_F32 ? 4 : 8;
    if (D < 1 || D > kScoreMaxD || D % V) return PT_ERR_UNSUPPORTED;
    if (U == 0) return PT_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int es = stats_dtype == PT_F32 ? 4 : 2, qes = q_dtype == PT_F32 ? 4 : 2;
    if (lamnorm_ws && G <= 8 && (D == 64 || D == 128) && !getenv("PT_SCORE_CTA") &&
        (long long)U * (Pmax / 32) < (1LL << 31)) {
        const int rc0 = pt_lam_norms(q, q_dtype, norms, U, G, D, lam, lamnorm_ws, nullptr, st);
        if (rc0) return rc0;
        StreamScoreParams sp{q, lamnorm_ws, means, stds, seq_len, keys, scores, U, S, Pmax, tile_max,
                             ss_contig(stats_dtype)};
        const int rc = q_dtype == PT_F32 ? launch_score_stream_q32(sp, stats_dtype, G, D, st)
                                         : launch_score_stream_q16(sp, stats_dtype, G, D, st);
        if (rc != PT_ERR_UNSUPPORTED) return rc;
    }
    ScoreParams prm{};
    prm.q = q; prm.norms_in = norms; prm.means = means; prm.stds = stds; prm.seq_len = seq_len;
    prm.keys = keys; prm.scores = scores; prm.counters = nullptr; prm.tile_max = tile_max;
    prm.D = D; prm.S = S; prm.Pmax = Pmax; prm.lam = lam; prm.k = 0;
    return dispatch_score(prm, q_dtype, stats_dtype, U, G, st);
}

// lam * ||q_g|| of every query row into the padded [U][8] layout of the streaming kernel
// (scoring.py:39-47 norms, numpy's float64 pairwise order; or lam * the given norms).
template <bool LATE>
static int lam_norms_launch(const void *q, int q_dtype, const float *norms, int U, int G, int D,
                            float lam, float *lamnorm, float *qnorm, void *stream) {
    if (!q || !lamnorm || U < 0 || G < 1 || G > 8 || D < 1 || D > kScoreMaxD) return PT_ERR_INVALID;
    if (U == 0) return PT_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int rows = U * G;
    const dim3 grid((rows + kLnRows - 1) / kLnRows);
    if (q_dtype == PT_F32)
        PT_CUDA_TRY(pt_launch(k_lam_norms<PT_F32, LATE>, grid, dim3(256), 0, st, q, norms, rows, G, D, lam, lamnorm, qnorm));
    else
        PT_CUDA_TRY(pt_launch(k_lam_norms<PT_BF16, LATE>, grid, dim3(256), 0, st, q, norms, rows, G, D, lam, lamnorm, qnorm));
    return PT_OK;
}

extern "C" int pt_lam_norms(const void *q, int q_dtype, const float *norms, int U, int G, int D,
                            float lam, float *lamnorm, float *qnorm, void *stream) {
    return lam_norms_launch<false>(q, q_dtype, norms, U, G, D, lam, lamnorm, qnorm, stream);
}

extern "C" int pt_lam_norms_chained(const void *q, int q_dtype, const float *norms, int U, int G,
                                    int D, float lam, float *lamnorm, float *qnorm, void *stream) {
    return lam_norms_launch<true>(q, q_dtype, norms, U, G, D, lam, lamnorm, qnorm, stream);
}

// K2 with lam * ||q|| precomputed by pt_lam_norms (so the norms launch can run beside the
// append); streaming kernel only -- PT_ERR_UNSUPPORTED outside its envelope.
extern "C" int pt_score_prenorm(const void *q, int q_dtype, const float *lamnorm,
                                const void *means, int stats_dtype, const float *stds,
                                const int32_t *seq_len, int U, int G, int D, int S, int Pmax,
                                uint16_t *keys, float *scores, uint16_t *tile_max, void *stream) {
    if (!q || !lamnorm || !means || !stds || !seq_len || !keys || U < 0 || S < 1 || Pmax % 32 ||
        G < 1)
        return PT_ERR_INVALID;
    if (G > 8 || !(D == 64 || D == 128) || getenv("PT_SCORE_CTA") ||
        (long long)U * (Pmax / 32) >= (1LL << 31))
        return PT_ERR_UNSUPPORTED;
    if (U == 0) return PT_OK;
    cudaStream_t st = (cudaStream_t)stream;
    StreamScoreParams sp{q, lamnorm, means, stds, seq_len, keys, scores, U, S, Pmax, tile_max,
                         ss_contig(stats_dtype)};
    return q_dtype == PT_F32 ? launch_score_stream_q32(sp, stats_dtype, G, D, st)
                             : launch_score_stream_q16(sp, stats_dtype, G, D, st);
}

extern "C" int pt_score_select(const void *q, int q_dtype, const float *norms, const void *means,
                               int stats_dtype, const float *stds, const int32_t *seq_len,
                               const int32_t *page_table, int U, int G, int D, int S, int Pmax,
                               float lam, int k, uint16_t *keys, float *scores, int32_t *sel,
                               int32_t *sel_logical, int32_t *n_sel, int32_t *kth,
                               int32_t *kplus1, int32_t *counters, void *stream) {
    if (!q || !means || !stds || !seq_len || !page_table || !keys || !sel || !n_sel || !kth ||
        !kplus1 || !counters || U < 0 || S < 1 || Pmax % 32 || G < 1)
        return PT_ERR_INVALID;
    if (k < 1) return PT_ERR_K;
    const int V = stats_dtype == PT_F32 ? 4 : 8;
    if (D < 1 || D > kScoreMaxD || D % V) return PT_ERR_UNSUPPORTED;
    if (U == 0) return PT_OK;
    ScoreParams prm{};
    prm.q = q; prm.norms_in = norms; prm.means = means; prm.stds = stds; prm.seq_len = seq_len;
    prm.keys = keys; prm.scores = scores; prm.counters = counters; prm.page_table = page_table;
    prm.sel = sel; prm.sel_logical = sel_logical; prm.n_sel = n_sel; prm.kth = kth;
    prm.kplus1 = kplus1;
    prm.D = D; prm.S = S; prm.Pmax = Pmax; prm.lam = lam; prm.k = k;
    return dispatch_score(prm, q_dtype, stats_dtype, U, G, (cudaStream_t)stream);
}

// dst[i] = max(dst[i], src[i]) over ordered u16 keys: the group max of a GQA group wider
// than the kernels' 8 heads, scored as sub-groups (key(max_g s_g) = max_g key(s_g): the
// bf16 rounding and the ordered encoding are monotone)
__global__ void k_keys_max(uint16_t *__restrict__ dst, const uint16_t *__restrict__ src, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = max(dst[i], src[i]);
}

extern "C" int pt_keys_max(uint16_t *dst, const uint16_t *src, int64_t n, void *stream) {
    if (!dst || !src || n < 0) return PT_ERR_INVALID;
    if (n == 0) return PT_OK;
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)pt_num_sms() * 8) blocks = (int64_t)pt_num_sms() * 8;
    k_keys_max<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(dst, src, n);
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}

extern "C" int pt_tile_means(const float *src, int U, int P, int D, int Pmax, void *dst,
                             int stats_dtype, void *stream) {
    if (!src || !dst || U < 0 || P < 0 || P > Pmax || Pmax % 32) return PT_ERR_INVALID;
    if ((int64_t)U * P * D == 0) return PT_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int64_t total = (int64_t)U * P * D;
    int blocks = (int)((total + 255) / 256);
    if (blocks > pt_num_sms() * 16) blocks = pt_num_sms() * 16;
    if (stats_dtype == PT_F32) k_tile_means<PT_F32><<<blocks, 256, 0, st>>>(src, U, P, D, Pmax, dst);
    else if (stats_dtype == PT_BF16) k_tile_means<PT_BF16><<<blocks, 256, 0, st>>>(src, U, P, D, Pmax, dst);
    else return PT_ERR_INVALID;
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}
