/*
 * pagetopk_oracle.c -- CPU restatement of the reference `pagetopk` decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200 kernels
 * in paper_2605_27740_b200/csrc.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The product path
 * never calls it (and has no CPU fallback).
 *
 * Every routine restates one reference function (paths relative to
 * /root/reference/pkg/src/pagetopk/) with the SAME floating-point operation order,
 * so that, compiled without FMA contraction (-ffp-contract=off, no -march), it is
 * bit-identical to the reference's compiled backend (`_kernels_cy.pyx`, built
 * with the reference's own flags: -O2/-O3, no -march, hence no FMA) and to the
 * numpy float64 statistics in kvcache.py / scoring.py.  Pinning: see
 * tests/test_oracle_vs_reference.py (live reference, this container) and
 * tests/test_oracle_golden.py (committed golden vectors, any box).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------- */
/* bf16.py:18-33  f32_to_bf16 (RNE, NaN quieted); bf16.py:42-45 is_nan_bf16    */
/* ------------------------------------------------------------------------- */
static inline uint16_t bf16_rne(float x) {
    uint32_t b;
    memcpy(&b, &x, 4);
    if (x != x) return (uint16_t)((b >> 16) | 0x0040u);
    uint32_t lsb = (b >> 16) & 1u;
    return (uint16_t)((b + 0x7FFFu + lsb) >> 16);
}

static inline int bf16_is_nan(uint16_t b) {
    return ((b & 0x7F80u) == 0x7F80u) && ((b & 0x007Fu) != 0);
}

/* select.py:51-57 encode_ordered: sign set -> ~bits, else bits | 0x8000 */
static inline uint16_t encode_key(uint16_t b) {
    return (b & 0x8000u) ? (uint16_t)~b : (uint16_t)(b | 0x8000u);
}

OR_EXPORT void or_f32_to_bf16(const float *x, uint16_t *out, int64_t n) {
    for (int64_t i = 0; i < n; i++) out[i] = bf16_rne(x[i]);
}

/* returns 0, or -1 if any NaN pattern is present (select.py:54-55) */
OR_EXPORT int or_encode_ordered(const uint16_t *bits, uint16_t *out, int64_t n) {
    for (int64_t i = 0; i < n; i++) {
        if (bf16_is_nan(bits[i])) return -1;
        out[i] = encode_key(bits[i]);
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* numpy float64 reductions, restated                                         */
/* ------------------------------------------------------------------------- */
/* numpy's pairwise_sum for contiguous float64 (numpy/_core/src/umath/loops_utils.h.src);
 * a 1-D np.sum is `0.0 + pairwise(a, n)` (identity-initialised reduce; checked
 * empirically in tests against numpy 2.3). */
static double np_pairwise(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
    }
}

OR_EXPORT double or_np_sum(const double *a, int64_t n) { return 0.0 + np_pairwise(a, n); }

/* kvcache.py:59-71 compute_page_stats:
 *   rows = f64(keys); mean = rows.mean(0)  (sequential over rows, / count)
 *   var = mean((rows - mean)**2, 0); std = f32(sqrt(var.sum()))
 * `scratch` holds D doubles (NULL -> malloc). */
OR_EXPORT void or_page_stats(const float *rows, int count, int D, float *mean_out,
                             float *std_out) {
    double stackbuf[2 * 512];
    double *mean = stackbuf, *var = stackbuf + 512;
    double *heap = NULL;
    if (D > 512) {
        heap = (double *)malloc(sizeof(double) * 2 * (size_t)D);
        mean = heap;
        var = heap + D;
    }
    for (int d = 0; d < D; d++) {
        double s = 0.0;
        for (int i = 0; i < count; i++) s = s + (double)rows[(int64_t)i * D + d];
        mean[d] = s / (double)count;
    }
    for (int d = 0; d < D; d++) {
        double s = 0.0;
        for (int i = 0; i < count; i++) {
            double t = (double)rows[(int64_t)i * D + d] - mean[d];
            s = s + t * t;
        }
        var[d] = s / (double)count;
    }
    double tot = 0.0 + np_pairwise(var, D);
    *std_out = (float)sqrt(tot);
    for (int d = 0; d < D; d++) mean_out[d] = (float)mean[d];
    free(heap);
}

/* scoring.py:39-47 QueryGroup.from_queries: norms = f32(sqrt(sum(f64(q)**2, axis=1))) */
OR_EXPORT void or_query_norms(const float *q, int G, int D, float *norms) {
    double buf[1024];
    double *sq = D <= 1024 ? buf : (double *)malloc(sizeof(double) * (size_t)D);
    for (int g = 0; g < G; g++) {
        for (int d = 0; d < D; d++) {
            double v = (double)q[(int64_t)g * D + d];
            sq[d] = v * v;
        }
        norms[g] = (float)sqrt(0.0 + np_pairwise(sq, D));
    }
    if (sq != buf) free(sq);
}

/* ------------------------------------------------------------------------- */
/* _kernels_cy.pyx:19-43 fused_scores                                         */
/* ------------------------------------------------------------------------- */
OR_EXPORT void or_fused_scores(const float *queries, const float *norms, const float *means,
                               const float *stds, int G, int64_t P, int D, float lam,
                               float *out) {
    for (int64_t p = 0; p < P; p++) {
        float best = -INFINITY;
        for (int g = 0; g < G; g++) {
            float acc = 0.0f;
            for (int d = 0; d < D; d++) acc = acc + queries[(int64_t)g * D + d] * means[p * D + d];
            acc = acc + lam * norms[g] * stds[p];
            if (acc > best) best = acc;
        }
        out[p] = best;
    }
}

/* ------------------------------------------------------------------------- */
/* _kernels_cy.pyx:46-126 radix_select_desc (ids in the Cython emission order) */
/* returns 0; ids_out must hold k entries; *kplus1 = -1 never happens for k<n  */
/* ------------------------------------------------------------------------- */
OR_EXPORT int or_radix_select_desc(const uint16_t *keys, int64_t n, int64_t k, int64_t *ids_out,
                                   int *threshold_out, int *kplus1_out) {
    int64_t hist_hi[256], hist_lo[256];
    memset(hist_hi, 0, sizeof hist_hi);
    memset(hist_lo, 0, sizeof hist_lo);
    for (int64_t i = 0; i < n; i++) hist_hi[keys[i] >> 8]++;
    int64_t above = 0;
    int hi = 0;
    for (int b = 255; b >= 0; b--) {
        if (above + hist_hi[b] >= k) { hi = b; break; }
        above += hist_hi[b];
    }
    int64_t need = k - above;
    int64_t *bucket = (int64_t *)malloc(sizeof(int64_t) * (size_t)(hist_hi[hi] > 0 ? hist_hi[hi] : 1));
    int64_t nsel = 0, nb = 0;
    int max_below_hi = -1;
    for (int64_t i = 0; i < n; i++) {
        uint16_t kk = keys[i];
        int b = kk >> 8;
        if (b > hi) ids_out[nsel++] = i;
        else if (b == hi) { bucket[nb++] = i; hist_lo[kk & 0xFF]++; }
        else if ((int)kk > max_below_hi) max_below_hi = (int)kk;
    }
    int64_t above2 = 0;
    int lo = 0;
    for (int b = 255; b >= 0; b--) {
        if (above2 + hist_lo[b] >= need) { lo = b; break; }
        above2 += hist_lo[b];
    }
    int64_t tie_budget = need - above2;
    int64_t leftover = hist_lo[lo] - tie_budget;
    int threshold = (hi << 8) | lo;
    int max_below_thr = max_below_hi;
    for (int64_t j = 0; j < nb; j++) {
        int64_t i = bucket[j];
        int lb = keys[i] & 0xFF;
        if (lb > lo) ids_out[nsel++] = i;
        else if (lb == lo) {
            if (tie_budget > 0) { ids_out[nsel++] = i; tie_budget--; }
        } else if ((int)keys[i] > max_below_thr) max_below_thr = (int)keys[i];
    }
    free(bucket);
    *threshold_out = threshold;
    *kplus1_out = leftover > 0 ? threshold : max_below_thr;
    return 0;
}

/* ------------------------------------------------------------------------- */
/* _kernels_cy.pyx:129-172 stream_attention (f32 accumulate, expf, lse double) */
/* ------------------------------------------------------------------------- */
OR_EXPORT void or_stream_attention(const float *q, const float *keys, const float *values,
                                   int64_t n, int D, float scale, int64_t block,
                                   const float *block_bias, float *out, double *lse) {
    float stackbuf[4096];
    float *buf = block <= 4096 ? stackbuf : (float *)malloc(sizeof(float) * (size_t)block);
    float m = -INFINITY, l = 0.0f;
    for (int d = 0; d < D; d++) out[d] = 0.0f;
    int64_t bi = 0;
    for (int64_t start = 0; start < n; start += block) {
        int64_t rows = start + block <= n ? block : n - start;
        float bias = block_bias ? block_bias[bi] : 0.0f;
        bi++;
        float m_new = m;
        for (int64_t i = 0; i < rows; i++) {
            float s = 0.0f;
            for (int d = 0; d < D; d++) s = s + keys[(start + i) * D + d] * q[d];
            s = s * scale + bias;
            buf[i] = s;
            if (s > m_new) m_new = s;
        }
        float carry = expf(m - m_new);
        l = l * carry;
        for (int d = 0; d < D; d++) out[d] = out[d] * carry;
        for (int64_t i = 0; i < rows; i++) {
            float w = expf(buf[i] - m_new);
            l = l + w;
            for (int d = 0; d < D; d++) out[d] = out[d] + w * values[(start + i) * D + d];
        }
        m = m_new;
    }
    for (int d = 0; d < D; d++) out[d] = out[d] / l;
    *lse = (double)m + log((double)l);
    if (buf != stackbuf) free(buf);
}

/* ------------------------------------------------------------------------- */
/* Batched restatements over units u = b * H_kv + h                           */
/* ------------------------------------------------------------------------- */

/* kvcache.py:178-183 _refresh_stats / :210-233 extend, for every page of every unit.
 * pool layout [phys][S][D] f32; page_table [U][Pmax]; means [U][Pmax][D]; stds [U][Pmax]. */
OR_EXPORT void or_build_stats(const float *kpool, const int32_t *page_table, const int32_t *seq_len,
                              int U, int S, int D, int Pmax, float *means, float *stds,
                              int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int u = 0; u < U; u++) {
        int n = seq_len[u];
        int P = (n + S - 1) / S;
        for (int p = 0; p < P; p++) {
            int rows = (p == P - 1) ? n - p * S : S;
            int64_t pid = page_table[(int64_t)u * Pmax + p];
            or_page_stats(kpool + pid * S * D, rows, D, means + ((int64_t)u * Pmax + p) * D,
                          stds + (int64_t)u * Pmax + p);
        }
    }
}

/* attention.py:110-147 decode_step, batched over units, with the cython backend's
 * kernels: per unit: QueryGroup norms -> fused_scores -> f32_to_bf16 -> encode ->
 * radix (or take-all when P <= k, select.py:100-101) -> mapping[ids] ->
 * per q-head sparse_attention over the gathered rows (kvcache.py:266-280) with
 * block = S (attention.py:94-107).
 *
 * q [U*G][D] f32; kpool/vpool [phys][S][D] f32; means [U][Pmax][D]; stds [U][Pmax].
 * Outputs: out [U*G][D], lse [U*G] (double), sel [U][k] physical ids in the
 * reference's emission order, n_sel[U], kth[U] (ordered key), kplus1[U] (key or -1),
 * scores_out [U][Pmax] f32 / keys_out [U][Pmax] u16 (may be NULL).
 * Returns 0, or -1 if a NaN score was met (select.py:54-55). */
OR_EXPORT int or_decode_units(int U, int G, int D, int S, int Pmax, int64_t k, const float *q,
                              const float *kpool, const float *vpool, const int32_t *page_table,
                              const int32_t *seq_len, const float *means, const float *stds,
                              float lam, float scale, int nthreads, float *out, double *lse,
                              int32_t *sel, int32_t *n_sel, int32_t *kth, int32_t *kplus1,
                              float *scores_out, uint16_t *keys_out) {
    int err = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(| : err)
#endif
    for (int u = 0; u < U; u++) {
        int n = seq_len[u];
        int64_t P = (n + S - 1) / S;
        const int32_t *map = page_table + (int64_t)u * Pmax;
        float *norms = (float *)malloc(sizeof(float) * (size_t)G);
        float *sc = (float *)malloc(sizeof(float) * (size_t)(P > 0 ? P : 1));
        uint16_t *bits = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)(P > 0 ? P : 1));
        int64_t *ids = (int64_t *)malloc(sizeof(int64_t) * (size_t)(P > k ? k : (P > 0 ? P : 1)));
        const float *qu = q + (int64_t)u * G * D;
        or_query_norms(qu, G, D, norms);
        or_fused_scores(qu, norms, means + (int64_t)u * Pmax * D, stds + (int64_t)u * Pmax, G, P,
                        D, lam, sc);
        int bad = 0;
        for (int64_t p = 0; p < P; p++) {
            uint16_t b = bf16_rne(sc[p]);
            if (bf16_is_nan(b)) bad = 1;
            bits[p] = encode_key(b);
        }
        if (scores_out) memcpy(scores_out + (int64_t)u * Pmax, sc, sizeof(float) * (size_t)P);
        if (keys_out) memcpy(keys_out + (int64_t)u * Pmax, bits, sizeof(uint16_t) * (size_t)P);
        int64_t ns;
        if (bad || P == 0) {
            err |= 1;
            ns = 0;
            n_sel[u] = 0;
        } else if (P <= k) {
            int mn = 0xFFFF;
            for (int64_t p = 0; p < P; p++) {
                ids[p] = p;
                if (bits[p] < mn) mn = bits[p];
            }
            ns = P;
            kth[u] = mn;
            kplus1[u] = -1;
        } else {
            int thr, kp1;
            or_radix_select_desc(bits, P, k, ids, &thr, &kp1);
            ns = k;
            kth[u] = thr;
            kplus1[u] = kp1;
        }
        n_sel[u] = (int32_t)ns;
        if (ns > 0) {
            /* gather (kvcache.py:266-280): rows of each page in selection order */
            int64_t tot = 0;
            for (int64_t j = 0; j < ns; j++) {
                int64_t lp = ids[j];
                tot += (lp == P - 1) ? n - lp * S : S;
            }
            float *gk = (float *)malloc(sizeof(float) * (size_t)(tot * D));
            float *gv = (float *)malloc(sizeof(float) * (size_t)(tot * D));
            int64_t r = 0;
            for (int64_t j = 0; j < ns; j++) {
                int64_t lp = ids[j];
                int64_t rows = (lp == P - 1) ? n - lp * S : S;
                int64_t pid = map[lp];
                sel[(int64_t)u * k + j] = (int32_t)pid;
                memcpy(gk + r * D, kpool + pid * S * D, sizeof(float) * (size_t)(rows * D));
                memcpy(gv + r * D, vpool + pid * S * D, sizeof(float) * (size_t)(rows * D));
                r += rows;
            }
            for (int g = 0; g < G; g++)
                or_stream_attention(qu + (int64_t)g * D, gk, gv, tot, D, scale, S, NULL,
                                    out + ((int64_t)u * G + g) * D, lse + (int64_t)u * G + g);
            free(gk);
            free(gv);
        }
        free(norms);
        free(sc);
        free(bits);
        free(ids);
    }
    return err ? -1 : 0;
}

/* attention.py:78-91 dense_attention over every unit's full context (the denominator) */
OR_EXPORT void or_dense_units(int U, int G, int D, int S, int Pmax, const float *q,
                              const float *kpool, const float *vpool, const int32_t *page_table,
                              const int32_t *seq_len, float scale, int nthreads, float *out,
                              double *lse) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int u = 0; u < U; u++) {
        int n = seq_len[u];
        int64_t P = (n + S - 1) / S;
        float *gk = (float *)malloc(sizeof(float) * (size_t)((int64_t)n * D + 1));
        float *gv = (float *)malloc(sizeof(float) * (size_t)((int64_t)n * D + 1));
        for (int64_t p = 0; p < P; p++) {
            int64_t rows = (p == P - 1) ? n - p * S : S;
            int64_t pid = page_table[(int64_t)u * Pmax + p];
            memcpy(gk + p * S * D, kpool + pid * S * D, sizeof(float) * (size_t)(rows * D));
            memcpy(gv + p * S * D, vpool + pid * S * D, sizeof(float) * (size_t)(rows * D));
        }
        for (int g = 0; g < G; g++)
            or_stream_attention(q + ((int64_t)u * G + g) * D, gk, gv, n, D, scale, S, NULL,
                                out + ((int64_t)u * G + g) * D, lse + (int64_t)u * G + g);
        free(gk);
        free(gv);
    }
}

OR_EXPORT int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
