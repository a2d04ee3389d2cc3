/*
 * pagetopk_b200.h -- C ABI of the B200-native UNIQUE decode hot path.
 *
 * The reference (`pagetopk`, /root/reference/pkg/src/pagetopk/) crosses exactly one
 * boundary on this path: the kernel-backend module contract of backend.py:14-58,
 * i.e. three functions bound from Python (`_kernels_cy.pyx`, `_kernels_py.py`).
 * Section A mirrors those three calls one for one (host buffers in, host buffers out,
 * same argument meaning) so a maintainer can register this library as a third backend
 * (INTEGRATION.md).  Section B is the batched, stream-ordered device API the package
 * `paper_2605_27740_b200` drives: caller-allocated device buffers, no host sync,
 * graph-capturable.
 *
 * Conventions: every entry point returns 0 on success, a PT_ERR_* precondition code,
 * or PT_ERR_CUDA_BASE + cudaError_t.  `stream` is a cudaStream_t passed as void*.
 * Units are (sequence b, kv-head h) pairs, u = b * H_kv + h; query heads are grouped
 * contiguously, q-head h_q -> kv-head h_q / G (attention.py:138).
 */
#ifndef PAGETOPK_B200_H
#define PAGETOPK_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PT_API __attribute__((visibility("default")))
#else
#define PT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* element types of the KV pool / page means / queries */
#define PT_F32 0
#define PT_BF16 1

/* status codes */
#define PT_OK 0
#define PT_ERR_INVALID 1     /* bad argument (null pointer, negative size, ...)          */
#define PT_ERR_UNSUPPORTED 2 /* shape outside the compiled envelope (D, G, S limits)     */
#define PT_ERR_K 3           /* k < 1: "k must be at least 1" (select.py:94-95)          */
#define PT_ERR_EMPTY 4       /* no pages: "no pages to select from" (select.py:98-99)    */
#define PT_ERR_CAPACITY 5    /* pool exhausted: CapacityError (kvcache.py:164-166)       */
#define PT_ERR_CUDA_BASE 1000

/* library identity */
PT_API int pt_version(void);
PT_API const char *pt_status_string(int status);

/* ======================================================================== */
/* A. Reference backend contract, host buffers (backend.py:14-58)            */
/* ======================================================================== */

/* _kernels_cy.pyx:19-43 fused_scores(queries f32[G,D], norms f32[G], means f32[P,D],
 * stds f32[P], lam) -> f32[P].  Bit-identical to the reference's compiled backend. */
PT_API int pt_fused_scores_host(const float *queries, const float *norms, const float *means,
                         const float *stds, int G, int64_t P, int D, float lam, float *out);

/* _kernels_cy.pyx:46-126 radix_select_desc(keys u16[P], k) -> (ids int64[k] (unordered;
 * emitted here in ascending index order), threshold, kplus1, passes=3).
 * Precondition 1 <= k < P as in the reference. */
PT_API int pt_radix_select_desc_host(const uint16_t *keys, int64_t P, int64_t k, int64_t *ids_out,
                              int *threshold_out, int *kplus1_out);

/* _kernels_cy.pyx:129-172 stream_attention(q f32[D], keys f32[N,D], values f32[N,D],
 * scale, block, block_bias f32[ceil(N/block)] or NULL) -> (out f32[D], lse). */
PT_API int pt_stream_attention_host(const float *q, const float *keys, const float *values, int64_t n,
                             int D, float scale, int64_t block, const float *block_bias,
                             float *out, double *lse);

/* ======================================================================== */
/* B. Batched device API (device pointers, stream-ordered, no host sync)     */
/* ======================================================================== */
/*
 * Device layouts:
 *   k_pool, v_pool : [num_phys_pages][S][D]           kv_dtype
 *   page_table     : int32 [U][Pmax]  logical -> physical page id   (kvcache.py:74-120)
 *   seq_len        : int32 [U]        tokens per unit
 *   means          : page-interleaved tiles [U][Pmax/32][D/V][32][V], V = 16 B / elem,
 *                    stats_dtype (f32 = exact reference stats; bf16 = compact mode)
 *   stds           : f32 [U][Pmax]
 *   keys           : u16 [U][Pmax]    ordered bf16 score keys (select.py:51-57)
 *   Pmax % 32 == 0.
 */

/* The mirror block (bounded scoring): one device allocation of
 * pt_mirror_bytes(U, Pmax, D) bytes holding, for every page, its f32 mean rounded to bf16
 * (page-interleaved tiles [U][Pmax/32][D/8][32][8]), the f32 mean again row-major ([U][Pmax][D],
 * one contiguous row per page) and an upper bound of ||bf16 mean - f32 mean|| plus the
 * accumulation slack of pt_score_bounded (f32 [U][Pmax]).  Written by K1 / K1b / the fused
 * extend when they are given one (f32 stats, D % 8 == 0); NULL: no mirror. */
PT_API size_t pt_mirror_bytes(int U, int Pmax, int D);

/* K1. kvcache.py:59-71 + :178-183: page statistics of logical pages
 * [page_begin[u], ceil(seq_len[u]/S)) of every unit (page_begin NULL -> all pages).
 * float64 accumulation in numpy's order; means rounded to stats_dtype, std to f32. */
PT_API int pt_page_stats(const void *k_pool, int kv_dtype, const int32_t *page_table,
                  const int32_t *seq_len, const int32_t *page_begin, int U, int S, int D,
                  int Pmax, void *means, int stats_dtype, float *stds, void *mirror, void *stream);

/* K1b. kvcache.py:185-208 append, batched: one new K/V row per unit ([U][D] kv_dtype)
 * lands in the unit's tail page; a full/absent tail page takes a fresh physical page
 * (free list first, then bump; deterministic in unit order, kvcache.py:154-176); the
 * touched page's stats are recomputed exactly.  pool_state int32[4] =
 * {bump_next, free_count, max_pages, error_flag}; error_flag set to PT_ERR_CAPACITY
 * when the pool is exhausted (that unit is left unchanged).  slot_scratch: int32 [2U + 4]
 * device scratch, zero-initialised once (per-unit target page, the launch's internal flags
 * (self-resetting), a snapshot of the lengths).  One launch. */
PT_API int pt_append(const void *k_new, const void *v_new, void *k_pool, void *v_pool, int kv_dtype,
              int32_t *page_table, int32_t *seq_len, int U, int S, int D, int Pmax, void *means,
              int stats_dtype, float *stds, int32_t *pool_state, const int32_t *free_list,
              int32_t *slot_scratch, void *mirror, void *stream);

/* Copy n_rows[u] rows per unit from a dense [U][n_max][D] staging buffer into the pool
 * starting at token position row_begin[u] (kvcache.py:210-233 extend; pages must
 * already be mapped by the caller). */
PT_API int pt_write_rows(const void *k_rows, const void *v_rows, int n_max, const int32_t *row_begin,
                  const int32_t *n_rows, void *k_pool, void *v_pool, int kv_dtype,
                  const int32_t *page_table, int U, int S, int D, int Pmax, void *stream);

/* K1 fused with the row scatter (the prefill path, kvcache.py:210-233 + :178-183): the
 * pt_write_rows copy followed by pt_page_stats over every touched page, in ONE launch that
 * never re-reads the pool (one warp per touched page: old rows of a partial tail page from
 * the pool, new rows from the staging buffer).  Pages must already be mapped; seq_len is not
 * read (row_begin / n_rows give the ranges).  Identical results to the two calls. */
PT_API int pt_extend(const void *k_rows, const void *v_rows, int n_max, const int32_t *row_begin,
                     const int32_t *n_rows, void *k_pool, void *v_pool, int kv_dtype,
                     const int32_t *page_table, int U, int S, int D, int Pmax, void *means,
                     int stats_dtype, float *stds, void *mirror, void *stream);

/* K2. scoring.py:108-124 + _kernels_cy.pyx:19-43 + bf16.py:18-33 + select.py:51-57:
 * q [U*G][D] (q_dtype); norms f32 [U*G] or NULL (computed as scoring.py:39-47);
 * score = max_g fl(fl(sum_d q*mean) + fl(fl(lam*norm_g)*std)), sequential d order;
 * writes keys u16 [U][Pmax] and optionally scores f32 [U][Pmax].
 * lamnorm_ws: f32 [U*8] device scratch enabling the streaming kernel (NULL: CTA kernel).
 * tile_max: u16 [U][Pmax/32] or NULL -- the largest key of every 32-page tile (a lower
 * bound for the k-th largest key that lets pt_select_attend skip most keys). */
PT_API int pt_score(const void *q, int q_dtype, const float *norms, const void *means, int stats_dtype,
             const float *stds, const int32_t *seq_len, int U, int G, int D, int S, int Pmax,
             float lam, uint16_t *keys, float *scores, float *lamnorm_ws, uint16_t *tile_max,
             void *stream);

/* K2 split in two launches so the first can run concurrently with the append:
 * pt_lam_norms writes fl(lam * ||q_g||) (norms NULL: computed in numpy's float64 order,
 * scoring.py:39-47) into lamnorm f32 [U][8]; pt_score_prenorm is pt_score's streaming
 * kernel reading it (same keys / scores / tile_max, bit for bit).  pt_score_prenorm
 * returns PT_ERR_UNSUPPORTED outside that kernel's envelope (G <= 8, D in {64, 128}).
 * qnorm: f32 [U][8] or NULL -- upper bounds of ||q_g|| (for pt_score_bounded). */
PT_API int pt_lam_norms(const void *q, int q_dtype, const float *norms, int U, int G, int D,
                        float lam, float *lamnorm, float *qnorm, void *stream);
/* pt_lam_norms_chained: the same norms for a straight PDL chain (append -> norms -> score):
 * it runs beside the kernel launched before it on the stream (it reads only q) and completes
 * only after that kernel, so the scoring kernel launched next sees both kernels' writes. */
PT_API int pt_lam_norms_chained(const void *q, int q_dtype, const float *norms, int U, int G,
                                int D, float lam, float *lamnorm, float *qnorm, void *stream);
PT_API int pt_score_prenorm(const void *q, int q_dtype, const float *lamnorm, const void *means,
                            int stats_dtype, const float *stds, const int32_t *seq_len, int U,
                            int G, int D, int S, int Pmax, uint16_t *keys, float *scores,
                            uint16_t *tile_max, void *stream);

/* K2b. Bounded scoring over the bf16 mirror of the f32 page means (half the bytes of K2):
 * for every page, keys_lo / keys_hi u16 [U][Pmax] = the ordered keys of a lower and an upper
 * bound of the reference score (the exact key lies in [keys_lo, keys_hi]), and tile_max u16
 * [U][Pmax/32] = the largest keys_lo of each 32-page tile.  pt_select_attend given keys_hi
 * turns these into the exact selection of the f32 reference.  bf16 queries, G <= 8,
 * D in {64, 128}, nu <= 2048; PT_ERR_UNSUPPORTED otherwise (use pt_score_prenorm).
 * Scores units [u0, u0 + nu) of a U-unit cache (every array is the whole cache's). */
PT_API int pt_score_bounded(const void *q, int q_dtype, const float *lamnorm, const float *qnorm,
                            const void *mirror, const float *stds, const int32_t *seq_len, int U,
                            int u0, int nu, int G, int D, int S, int Pmax, uint16_t *keys_lo,
                            uint16_t *keys_hi, uint16_t *tile_max, void *stream);

/* The decode step's K1b + K2b with the scorer overlapping the append (no reference
 * counterpart: an internal schedule of DecodeEngine.step).  pt_append_step = pt_append that
 * also publishes, in step_sync (int32[4], zero-initialised once, one per step sequence),
 * when every unit's length is snapshotted and when all its stores are visible;
 * pt_score_bounded_step, launched right after it on the same stream with the same
 * slot_scratch / step_sync (all U units), streams every 32-page tile except the units' tail
 * tiles from the snapshot lengths + 1 while the append runs, then the tail tiles.  Same
 * keys as pt_append + pt_score_bounded.  The two calls must be paired (PT_ERR_UNSUPPORTED
 * from the scorer where pt_score_bounded is unsupported: check before appending). */
PT_API int pt_append_step(const void *k_new, const void *v_new, void *k_pool, void *v_pool,
                          int kv_dtype, int32_t *page_table, int32_t *seq_len, int U, int S, int D,
                          int Pmax, void *means, int stats_dtype, float *stds, int32_t *pool_state,
                          const int32_t *free_list, int32_t *slot_scratch, void *mirror,
                          int32_t *step_sync, void *stream);
PT_API int pt_score_bounded_step(const void *q, int q_dtype, const float *lamnorm,
                                 const float *qnorm, const void *mirror, const float *stds,
                                 const int32_t *seq_len, int U, int G, int D, int S, int Pmax,
                                 uint16_t *keys_lo, uint16_t *keys_hi, uint16_t *tile_max,
                                 const int32_t *slot_scratch, int32_t *step_sync, void *stream);

/* K2+K3 fused: pt_score followed by pt_topk in ONE launch -- the last CTA to finish a unit's
 * pages selects that unit's top-k while other CTAs keep scoring (same outputs as the two
 * separate calls).  counters: int32 [U] zero-initialised once (self-resetting).  Returns
 * PT_ERR_UNSUPPORTED when the unit's keys exceed the kernel's shared-memory envelope; the
 * caller then uses pt_score + pt_topk. */
PT_API int pt_score_select(const void *q, int q_dtype, const float *norms, const void *means,
                           int stats_dtype, const float *stds, const int32_t *seq_len,
                           const int32_t *page_table, int U, int G, int D, int S, int Pmax,
                           float lam, int k, uint16_t *keys, float *scores, int32_t *sel,
                           int32_t *sel_logical, int32_t *n_sel, int32_t *kth, int32_t *kplus1,
                           int32_t *counters, void *stream);

/* K3. select.py:87-115 + _kernels_cy.pyx:46-126: per unit, k highest keys, ties to the
 * lowest logical index; P <= k takes every page.  sel: int32 [U][k] physical ids in
 * ascending logical order (sel_logical, if non-NULL, the logical ids); n_sel[U];
 * kth[U] = ordered key of the k-th pick; kplus1[U] = key just below the cut or -1. */
PT_API int pt_topk(const uint16_t *keys, const int32_t *seq_len, const int32_t *page_table, int U,
            int S, int Pmax, int k, int32_t *sel, int32_t *sel_logical, int32_t *n_sel,
            int32_t *kth, int32_t *kplus1, void *stream);

/* K4. attention.py:94-107 + :57-75 + _kernels_cy.pyx:129-172: split-KV paged decode.
 * For unit u, the G query heads attend over the n_sel[u] pages sel[u][0..n_sel) (physical
 * ids, row stride sel_stride); a page equal to the unit's tail page holds
 * seq_len - (P-1)*S rows, others S.  bias f32 [U][sel_stride] per page or NULL.
 * n_sel == NULL selects dense mode (attention.py:78-91): every page of the unit, i.e.
 * pass sel = page_table, sel_stride = Pmax.
 * num_phys_pages: pool extent (for the TMA tensor maps of the bf16 tensor-core path).
 * out f32 [U*G][D], lse f32 [U*G].  workspace: pt_attend_workspace_bytes();
 * tickets int32 [U] zero-initialised once (self-resetting).  nsplit 0 = automatic. */
PT_API size_t pt_attend_workspace_bytes(int U, int G, int D, int sel_stride);
PT_API int pt_attend(const void *q, int q_dtype, const void *k_pool, const void *v_pool, int kv_dtype,
              int num_phys_pages, const int32_t *sel, int sel_stride, const int32_t *n_sel,
              const int32_t *page_table, const int32_t *seq_len, int U, int G, int D, int S,
              int Pmax, const float *bias, float scale, float *out, float *lse, void *workspace,
              size_t workspace_bytes, int32_t *tickets, int nsplit, void *stream);

/* K3+K4 fused (the engine's default after pt_score): per unit, the selection of pt_topk
 * (same outputs: sel [U][k], sel_logical or NULL, n_sel, kth, kplus1) followed by the
 * sparse attention of pt_attend over exactly those pages (sel_stride = k, no bias), in
 * ONE launch -- the selected ids stay in shared memory and feed the TMA producer.
 * Replaces the select.py:105-107 -> attention.py:143-146 pair of calls of decode_step
 * (attention.py:137-146).  bf16 KV, G <= 8, D in {64,128,256}, S in {16,32,64}; returns
 * PT_ERR_UNSUPPORTED outside that envelope (the caller runs pt_topk + pt_attend).
 * tile_max: pt_score's per-tile maxima or NULL (they let the selection skip the keys below
 * the k-th largest tile maximum).  Emission order equals pt_topk's (ascending logical).
 * Launched with programmatic dependent launch: its prologue reads seq_len, page_table and q
 * before waiting on the preceding kernel, which therefore must not write those (the
 * package's scorers do not).
 * Bounded mode (keys_hi non-NULL): keys / keys_hi / tile_max are pt_score_bounded's; the
 * exact key of every page whose interval reaches the cut is recomputed from the mirror's
 * row-major f32 means, stds and lamnorm (pt_lam_norms' [U][8]) -- the outputs equal the
 * exact mode's over the f32 reference keys.  NULL: keys are exact (the other three unused).
 * Processes units [u0, u0 + nu) of a U-unit cache (every per-unit array is the whole cache's;
 * the workspace is used from u0's share on): two disjoint ranges may run concurrently. */
PT_API int pt_select_attend(const uint16_t *keys, const uint16_t *tile_max,
                            const uint16_t *keys_hi, const void *mirror, const float *stds,
                            const float *lamnorm, const int32_t *seq_len, const int32_t *page_table,
                            int U, int u0, int nu, int S, int Pmax, int k, int32_t *sel, int32_t *sel_logical,
                            int32_t *n_sel, int32_t *kth, int32_t *kplus1, const void *q,
                            int q_dtype, const void *k_pool, const void *v_pool, int kv_dtype,
                            int num_phys_pages, int G, int D, float scale, float *out, float *lse,
                            void *workspace, size_t workspace_bytes, int32_t *tickets, void *stream);

/* Tuning aid: per-CTA phase timestamps (%globaltimer ns; 10 per CTA: entry, keys staged,
 * selection done, first page landed, stream done, exit, then inside the selection: range,
 * threshold, compaction, translation) of the last pt_select_attend launch made with
 * PT_SA_PROF=1 in the environment.  n <= 10 * 4096. */
PT_API int pt_debug_sa_prof(unsigned long long *host, int n);

/* Tuning aid: per-CTA timestamps (entry, after the PDL wait, exit) of the last
 * pt_score_bounded launch made with PT_SB_PROF=1.  n <= 4 * 2048. */
PT_API int pt_debug_sb_prof(unsigned long long *host, int n);

/* Tuning aid: per-unit phase timestamps of the last pt_append launch made with PT_APP_PROF=1
 * (8 per unit: entry, after the PDL wait, row loaded, tail page id known, page staged, stats
 * stored, length snapshot seen, exit).  n <= 8 * 8192. */
PT_API int pt_debug_append_prof(unsigned long long *host, int n);

/* Soft-mask training path (softmask.py:178-217 gated_attention_backward), batched over units:
 * the backward of attention over every page with a per-page additive log-gate bias, for the G
 * query heads of each unit.  gates f32 [U][Pmax] (0 = hard-masked page, skipped); out / lse /
 * dout: the forward's output, log-sum-exp and the loss gradient ([U*G][D], [U*G]).  Writes
 * dk_pool / dv_pool (f32, pool layout [pages][S][D], only the rows of attended pages),
 * dgates [U][Pmax] (summed over heads) and ACCUMULATES into dq [U*G][D] (zero it first).
 * The forward is pt_attend in dense mode with bias = log(gate) (soft) or over the kept pages
 * (hard).  f32 arithmetic (the reference is float64). */
PT_API int pt_gated_attend_bwd(const void *q, int q_dtype, const void *k_pool, const void *v_pool,
                               int kv_dtype, const int32_t *page_table, const int32_t *seq_len,
                               const float *gates, const float *out, const float *lse,
                               const float *dout, int U, int G, int D, int S, int Pmax, float scale,
                               float *dq, float *dk_pool, float *dv_pool, float *dgates,
                               void *stream);

/* Soft-mask forward prologue (softmask.py:108-176, soft mode): checks every gate of a live
 * page (page < ceil(seq_len[u] / S)) lies in (0, 1] and writes bias[u][p] = f32(log(gate)) for
 * all U x Pmax slots (gates float64 [U][Pmax]).  *flag (device int32) is set to 1 when a live
 * gate is out of range ("soft gates must lie in (0, 1]"); the caller reads it. */
PT_API int pt_gate_bias(const double *gates, const int32_t *seq_len, int U, int S, int Pmax,
                        float *bias, int32_t *flag, void *stream);

/* Serving loop (runtime.cu): a depth-slot pipeline of decode steps.  pt_pipe_submit queues
 * one step on slot `slot`: H2D of in_bytes from pinned host_in into dev_in on the h2d
 * stream, launch of the slot's captured step graph (cudaGraphExec_t) on the compute stream,
 * D2H of out_bytes from dev_out into pinned host_out on the d2h stream -- with the event
 * edges that overlap the copies of neighbouring steps with the kernels (a slot's next H2D
 * waits for its graph, its next graph waits for its D2H).  pt_pipe_wait blocks until the
 * slot's outputs are on the host. */
PT_API int pt_pipe_create(void *compute_stream, void *h2d_stream, void *d2h_stream, int depth,
                          void **pipe_out);
PT_API int pt_pipe_submit(void *pipe, int slot, void *graph_exec, void *dev_in, const void *host_in,
                          size_t in_bytes, void *host_out, const void *dev_out, size_t out_bytes);
PT_API int pt_pipe_wait(void *pipe, int slot);
PT_API int pt_pipe_destroy(void *pipe);

/* dst[i] = max(dst[i], src[i]) over n ordered u16 keys: the group maximum of a GQA group of
 * more than 8 query heads scored as sub-groups of <= 8 (the key of a max is the max of keys). */
PT_API int pt_keys_max(uint16_t *dst, const uint16_t *src, int64_t n, void *stream);

/* Layout helper: row-major means f32 [U][P][D] -> tiled stats layout (stats_dtype). */
PT_API int pt_tile_means(const float *means_rowmajor, int U, int P, int D, int Pmax, void *means_tiled,
                  int stats_dtype, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* PAGETOPK_B200_H */
