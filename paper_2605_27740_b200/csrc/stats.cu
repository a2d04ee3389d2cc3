// stats.cu -- K1: per-page key statistics (prefill build + decode append).
//
// Restates kvcache.py:59-71 compute_page_stats and :178-183 _refresh_stats with the
// reference's float64 operation order (numpy: sequential row sums for axis-0 means and
// variances, pairwise summation for var.sum()), so cached stats are bit-identical to
// the reference cache built from the same rows.  DFMA contraction is prevented with
// explicit __dadd_rn/__dmul_rn.
//
// Layout: one warp per page; lane owns dims d = lane + 32*j (a warp load is one
// contiguous row slice, coalesced); float64 per-dim accumulators live in registers;
// the D per-dim variances go through shared memory for numpy's pairwise sum.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace pt {

constexpr int kStatsWarps = 8;
constexpr int kMaxD = 512;

template <int DT, int SDT, int DJ>
__device__ __forceinline__ void page_stats_warp(const void *k_pool, int64_t pid, int rows, int S,
                                                int D, int64_t u, int64_t p, int64_t Pmax,
                                                void *means, float *stds, double *var_smem,
                                                const MirrorView mv) {
    const int lane = threadIdx.x & 31;
    const int64_t base = pid * (int64_t)S * D;
    double mean[DJ];
#pragma unroll
    for (int j = 0; j < DJ; j++) {
        const int d = lane + 32 * j;
        double s = 0.0;
        if (d < D) {
            for (int r = 0; r < rows; r++)
                s = __dadd_rn(s, (double)load_elem<DT>(k_pool, base + (int64_t)r * D + d));
        }
        mean[j] = __ddiv_rn(s, (double)rows);
    }
#pragma unroll
    for (int j = 0; j < DJ; j++) {
        const int d = lane + 32 * j;
        if (d < D) {
            double s = 0.0;
            for (int r = 0; r < rows; r++) {
                double t = __dsub_rn((double)load_elem<DT>(k_pool, base + (int64_t)r * D + d), mean[j]);
                s = __dadd_rn(s, __dmul_rn(t, t));
            }
            var_smem[d] = __ddiv_rn(s, (double)rows);
            constexpr int V = StatsTile<SDT>::V;
            store_elem<SDT>(means, mean_offset(u, p, d, D, Pmax, V), __double2float_rn(mean[j]));
        }
    }
    if (mv.tiles) store_mirror<DJ>(mean, D, u, p, Pmax, mv, lane);
    __syncwarp();
    if (lane == 0) stds[u * Pmax + p] = __double2float_rn(__dsqrt_rn(np_sum(DoubleArray{var_smem}, D)));
    __syncwarp();
}

// grid: (ceil(Pmax / kStatsWarps), U); warp w of block x handles logical page x*8+w.
template <int DT, int SDT, int DJ>
__global__ void __launch_bounds__(kStatsWarps * 32)
    k_page_stats(const void *__restrict__ k_pool, const int32_t *__restrict__ page_table,
                 const int32_t *__restrict__ seq_len, const int32_t *__restrict__ page_begin,
                 int S, int D, int Pmax, void *__restrict__ means, float *__restrict__ stds,
                 const MirrorView mv) {
    __shared__ double var_smem[kStatsWarps][kMaxD];
    const int warp = threadIdx.x >> 5;
    const int64_t u = blockIdx.y;
    const int64_t p = (int64_t)blockIdx.x * kStatsWarps + warp;
    const int n = seq_len[u];
    const int P = (n + S - 1) / S;
    const int p0 = page_begin ? page_begin[u] : 0;
    if (p >= P || p < p0) return;
    const int rows = (p == P - 1) ? n - (int)p * S : S;
    const int64_t pid = page_table[u * Pmax + p];
    page_stats_warp<DT, SDT, DJ>(k_pool, pid, rows, S, D, u, p, Pmax, means, stds, var_smem[warp], mv);
}

// ---------------------------------------------------------------------------
// decode append (kvcache.py:185-208), batched over units
// ---------------------------------------------------------------------------
// Decode append, one launch (kvcache.py:185-208 for every unit).
//
// The FIRST CTA to arrive (an atomic ticket, not a fixed block index) snapshots every
// unit's length (global scratch) and publishes `flag_read`; if any unit starts a new page it
// runs the deterministic unit-order allocation -- the batched _alloc_page
// (kvcache.py:154-176): free list popped from its end (list.pop()), then the bump pointer;
// pool or page-table exhaustion -> error flag, unit skipped (no page consumed) -- and
// publishes `flag_alloc`.  Every warp owns one unit: units continuing their tail page (15 of
// 16 steps at S = 16) never wait; a unit starting a page waits for the allocation.  The warp
// writes the new K/V row and recomputes the tail page's stats from a shared-memory copy of
// its rows (one load round), then -- once the snapshot is taken (flag_read; normally long
// set) -- advances its own sequence length.  The last CTA to finish re-arms the flags.
// No deadlock for any dispatch order or grid size: waiting CTAs only ever wait for the
// allocating CTA, which took the first ticket, i.e. is already resident and never waits.
__host__ __device__ __forceinline__ size_t append_per_warp(int S, int D, int ES) {
    return (((size_t)S * D * ES + 15) & ~(size_t)15) + (size_t)D * 8;
}

// raw 16-byte-chunk copy global -> shared of nbytes; every load of a thread is issued before
// its first store.  Falls back to 2-byte words when not 16-byte aligned.
template <int MAXC>
__device__ __forceinline__ void stage_raw(char *dst, const char *src, int nbytes, int lane) {
    if ((nbytes & 15) == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
        const int nch = nbytes >> 4;
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
        for (int c0 = lane; c0 < nch; c0 += 32 * MAXC) {
            uint4 v[MAXC];
#pragma unroll
            for (int j = 0; j < MAXC; j++)
                if (c0 + 32 * j < nch) v[j] = __ldg(s4 + c0 + 32 * j);
#pragma unroll
            for (int j = 0; j < MAXC; j++)
                if (c0 + 32 * j < nch) reinterpret_cast<uint4 *>(dst)[c0 + 32 * j] = v[j];
        }
    } else {
        for (int i = lane; i < nbytes / 2; i += 32)
            reinterpret_cast<uint16_t *>(dst)[i] = reinterpret_cast<const uint16_t *>(src)[i];
    }
}

__device__ __forceinline__ void spin_flag(int *flag, bool acquire) {
    while (atomicAdd(flag, 0) == 0) __nanosleep(32);
    if (acquire) __threadfence();  // the allocation's page table / slot writes
}

__device__ void alloc_scan(int32_t *__restrict__ page_table, const int *__restrict__ sn, int U,
                           int S, int Pmax, int32_t *__restrict__ pool_state,
                           const int32_t *__restrict__ free_list, int32_t *__restrict__ slot,
                           int *warp_tot, int *carry) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int bump0 = pool_state[0], free0 = pool_state[1], max_pages = pool_state[2];
    if (tid == 0) *carry = 0;
    __syncthreads();
    for (int base = 0; base < U; base += blockDim.x) {
        const int u = base + tid;
        const int n = u < U ? sn[u] : 1;
        const bool starts = u < U && n % S == 0;
        // a unit whose page table is full takes no rank (no page is consumed for it)
        const int need = (starts && n / S < Pmax) ? 1 : 0;
        if (starts && !need) {
            slot[u] = -1;
            pool_state[3] = PT_ERR_CAPACITY;
        }
        const unsigned m = __ballot_sync(0xffffffffu, need);
        const int wpre = __popc(m & ((1u << lane) - 1u));
        if (lane == 0) warp_tot[warp] = __popc(m);
        __syncthreads();
        int before = *carry, chunk_total = 0;
        for (int w = 0; w < nwarps; w++) {
            if (w < warp) before += warp_tot[w];
            chunk_total += warp_tot[w];
        }
        const int rank = before + wpre;
        if (need) {
            const int pid = rank < free0 ? free_list[free0 - 1 - rank] : bump0 + (rank - free0);
            const int lp = n / S;
            if (pid >= max_pages) {
                slot[u] = -1;
                pool_state[3] = PT_ERR_CAPACITY;
            } else {
                page_table[(int64_t)u * Pmax + lp] = pid;
                slot[u] = pid;
            }
        }
        __syncthreads();
        if (tid == 0) *carry += chunk_total;
        __syncthreads();
    }
    if (tid == 0) {
        const int tot = *carry;
        const int from_free = tot < free0 ? tot : free0;
        const int bump = bump0 + (tot - from_free);
        pool_state[1] = free0 - from_free;
        pool_state[0] = bump < max_pages ? bump : max_pages;
    }
}

// Optional per-unit phase timestamps (%globaltimer, ns) for tuning: PT_APP_PROF=1 on the host,
// read back with pt_debug_append_prof().  8 stamps per unit.
constexpr int kAppProfUnits = 8192;
__device__ unsigned long long g_app_prof[kAppProfUnits * 8];
// PT_APP_PROF=1: %globaltimer; PT_APP_PROF=2: %clock64 (per-unit phase durations only)
__device__ __forceinline__ void app_stamp(bool on, int64_t u, int i, bool clk = false) {
    if (on) {
        unsigned long long t;
        if (clk) asm volatile("mov.u64 %0, %clock64;" : "=l"(t));
        else asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        g_app_prof[u * 8 + i] = t;
    }
}

template <int DT, int SDT, int DJ>
__global__ void __launch_bounds__(256)
    k_append(const void *__restrict__ k_new, const void *__restrict__ v_new,
             void *__restrict__ k_pool, void *__restrict__ v_pool,
             int32_t *__restrict__ page_table, int32_t *__restrict__ seq_len, int U, int S, int D,
             int Pmax, void *__restrict__ means, float *__restrict__ stds,
             int32_t *__restrict__ pool_state, const int32_t *__restrict__ free_list,
             int32_t *__restrict__ slot, int prof, const MirrorView mv,
             int32_t *__restrict__ step_sync) {
    extern __shared__ __align__(16) char asmem[];
    __shared__ int warp_tot[8];
    __shared__ int carry;
    __shared__ int is_last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpc = blockDim.x >> 5;
    int *flag_alloc = slot + U, *done = slot + U + 1, *flag_read = slot + U + 2, *arrive = slot + U + 3;
    __shared__ int first_cta;
    constexpr int ES = DT == PT_F32 ? 4 : 2;
    const size_t per_warp = append_per_warp(S, D, ES);
    const int64_t u = (int64_t)blockIdx.x * wpc + warp;
    const bool pr = prof && lane == 0 && u < U && u < kAppProfUnits;
    app_stamp(pr, u, 0, prof == 2);
    pdl_trigger();
    pdl_wait();
    app_stamp(pr, u, 1, prof == 2);
    using Bits = typename std::conditional<DT == PT_F32, uint32_t, uint16_t>::type;
    // this unit's length (read before anyone advances it) and the new K/V row
    const int n = u < U ? seq_len[u] : 0;
    Bits kb[DJ], vb[DJ];
#pragma unroll
    for (int j = 0; j < DJ; j++) {
        const int d = lane + 32 * j;
        if (u < U && d < D) {
            kb[j] = static_cast<const Bits *>(k_new)[u * D + d];
            vb[j] = static_cast<const Bits *>(v_new)[u * D + d];
        }
    }
    if (threadIdx.x == 0) first_cta = atomicAdd(arrive, 1) == 0;
    __syncthreads();
    if (first_cta) {
        int *sn = slot + U + 4;  // global scratch: no per-CTA shared memory for U lengths
        int any = 0;
        for (int i = threadIdx.x; i < U; i += blockDim.x) {
            const int ni = seq_len[i];
            sn[i] = ni;
            any |= (ni % S == 0);
        }
        if (step_sync) __threadfence();  // every thread's snapshot stores, before the epoch
        any = __syncthreads_or(any);
        if (threadIdx.x == 0) { __threadfence(); atomicExch(flag_read, 1); }
        // decode step with an early scorer (pt_score_bounded_step): the lengths are snapshotted
        if (step_sync && threadIdx.x == 0) atomicAdd(&step_sync[0], 1);
        if (any) alloc_scan(page_table, sn, U, S, Pmax, pool_state, free_list, slot, warp_tot, &carry);
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) atomicExch(flag_alloc, 1);
    }
    // the tail page's rows stay in their storage format (bf16: half the shared memory of f32,
    // so short-page-count / many-unit steps keep more warps resident); widened on use
    Bits *rows_s = reinterpret_cast<Bits *>(asmem + warp * per_warp);
    double *var_s = reinterpret_cast<double *>(asmem + warp * per_warp +
                                               (((size_t)S * D * ES + 15) & ~(size_t)15));
    auto rowval = [&](int i) -> double {
        return DT == PT_F32 ? (double)__uint_as_float((uint32_t)rows_s[i])
                            : (double)bf16_bits_to_f32((uint32_t)rows_s[i]);
    };
    app_stamp(pr, u, 2, prof == 2);
    if (u < U) {
        int pid;
        if (n % S == 0) {  // starts a page: the allocating CTA's result
            if (lane == 0) spin_flag(flag_alloc, true);
            __syncwarp();
            pid = __ldcg(&slot[u]);
        } else {
            pid = page_table[u * Pmax + n / S];
        }
        app_stamp(pr, u, 3, prof == 2);
        if (pid >= 0) {
            const int row = n % S;
            const int64_t base = (int64_t)pid * S * D;
            // stage the page's existing rows (one load round) and the new row
            stage_raw<8>(reinterpret_cast<char *>(rows_s),
                         static_cast<const char *>(k_pool) + base * ES, row * D * ES, lane);
#pragma unroll
            for (int j = 0; j < DJ; j++) {
                const int d = lane + 32 * j;
                if (d < D) {
                    rows_s[row * D + d] = kb[j];
                    static_cast<Bits *>(k_pool)[base + (int64_t)row * D + d] = kb[j];
                    static_cast<Bits *>(v_pool)[base + (int64_t)row * D + d] = vb[j];
                }
            }
            __syncwarp();
            app_stamp(pr, u, 4, prof == 2);
            const int cnt = row + 1;
            // rows outer, the lane's DJ columns inner: DJ independent f64 chains in flight (each
            // column still sums its rows in row order, as numpy's axis-0 reduction)
            const bool dok = (D % 32 == 0) || lane + 32 * (DJ - 1) < D;
            double mean[DJ], vacc[DJ];
#pragma unroll
            for (int j = 0; j < DJ; j++) mean[j] = 0.0;
#pragma unroll 4
            for (int r = 0; r < cnt; r++)
#pragma unroll
                for (int j = 0; j < DJ; j++)
                    if (dok || lane + 32 * j < D) mean[j] = __dadd_rn(mean[j], rowval(r * D + lane + 32 * j));
#pragma unroll
            for (int j = 0; j < DJ; j++) { mean[j] = __ddiv_rn(mean[j], (double)cnt); vacc[j] = 0.0; }
#pragma unroll 4
            for (int r = 0; r < cnt; r++)
#pragma unroll
                for (int j = 0; j < DJ; j++)
                    if (dok || lane + 32 * j < D) {
                        const double t = __dsub_rn(rowval(r * D + lane + 32 * j), mean[j]);
                        vacc[j] = __dadd_rn(vacc[j], __dmul_rn(t, t));
                    }
            constexpr int V = StatsTile<SDT>::V;
#pragma unroll
            for (int j = 0; j < DJ; j++) {
                const int d = lane + 32 * j;
                if (d < D) {
                    var_s[d] = __ddiv_rn(vacc[j], (double)cnt);
                    store_elem<SDT>(means, mean_offset(u, n / S, d, D, Pmax, V), __double2float_rn(mean[j]));
                }
            }
            if (mv.tiles) store_mirror<DJ>(mean, D, u, n / S, Pmax, mv, lane);
            __syncwarp();
            const double vsum = np_sum_warp(var_s, D, lane);
            if (lane == 0) {
                stds[u * Pmax + n / S] = __double2float_rn(__dsqrt_rn(vsum));
                app_stamp(pr, u, 5, prof == 2);
                spin_flag(flag_read, false);  // every length is snapshotted (no data to acquire)
                app_stamp(pr, u, 6, prof == 2);
                seq_len[u] = n + 1;
            }
        }
    }
    if (step_sync) __threadfence();  // this CTA's row / stats / length stores, before the epoch
    __syncthreads();
    if (threadIdx.x == 0) {
        // every flag use of this CTA precedes this atomic in program order: no fence needed
        if (atomicAdd(done, 1) == (int)gridDim.x - 1) {  // re-arm for the next append
            atomicExch(flag_alloc, 0);
            atomicExch(flag_read, 0);
            atomicExch(arrive, 0);
            atomicExch(done, 0);
            // every CTA's stores are visible: the early scorer may read the tail tiles now
            if (step_sync) { __threadfence(); atomicAdd(&step_sync[1], 1); }
        }
    }
    if (prof && lane == 0 && u < U && u < kAppProfUnits) app_stamp(true, u, 7, prof == 2);
}

// ---------------------------------------------------------------------------
// Fused extend (kvcache.py:210-233 + :178-183 for every touched page): the prefill path.
// One warp per touched page: the page's rows already in the pool (a partially filled tail)
// and the new rows from the dense staging buffer land in shared memory as f32 (one round
// of 16-byte loads); the new K and V rows are stored to the pool from the same registers;
// mean/std are then computed from shared memory exactly as page_stats_warp (f64, numpy
// order).  HBM traffic = staging read + pool write + stats write (the pool is not re-read).
// ---------------------------------------------------------------------------
template <int DT, int MAXC>
__device__ __forceinline__ void copy_new_rows(const char *__restrict__ ks, const char *__restrict__ vs,
                                              char *__restrict__ kd, char *__restrict__ vd,
                                              float *__restrict__ rows_f32, int nbytes, int lane) {
    constexpr int EPC = DT == PT_F32 ? 4 : 8;
    const int nch = nbytes >> 4;
    const uint4 *k4 = reinterpret_cast<const uint4 *>(ks);
    const uint4 *v4 = reinterpret_cast<const uint4 *>(vs);
    for (int c0 = lane; c0 < nch; c0 += 32 * MAXC) {
        uint4 kv[MAXC], vv[MAXC];
#pragma unroll
        for (int j = 0; j < MAXC; j++) {
            const int c = c0 + 32 * j;
            if (c < nch) { kv[j] = __ldcs(k4 + c); vv[j] = __ldcs(v4 + c); }
        }
#pragma unroll
        for (int j = 0; j < MAXC; j++) {
            const int c = c0 + 32 * j;
            if (c >= nch) break;
            reinterpret_cast<uint4 *>(kd)[c] = kv[j];
            reinterpret_cast<uint4 *>(vd)[c] = vv[j];
            float *o = rows_f32 + c * EPC;
            if constexpr (DT == PT_F32) {
                o[0] = __uint_as_float(kv[j].x); o[1] = __uint_as_float(kv[j].y);
                o[2] = __uint_as_float(kv[j].z); o[3] = __uint_as_float(kv[j].w);
            } else {
                const uint32_t w[4] = {kv[j].x, kv[j].y, kv[j].z, kv[j].w};
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    o[2 * q] = __uint_as_float(w[q] << 16);
                    o[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
                }
            }
        }
    }
}

template <int DT, int SDT, int DJ>
__global__ void __launch_bounds__(256)
    k_extend(const void *__restrict__ k_rows, const void *__restrict__ v_rows, int n_max,
             const int32_t *__restrict__ row_begin, const int32_t *__restrict__ n_rows,
             void *__restrict__ k_pool, void *__restrict__ v_pool,
             const int32_t *__restrict__ page_table, int S, int D, int Pmax,
             void *__restrict__ means, float *__restrict__ stds, const MirrorView mv) {
    extern __shared__ __align__(16) char esmem[];
    constexpr int ES = DT == PT_F32 ? 4 : 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, wpc = blockDim.x >> 5;
    const int64_t u = blockIdx.y;
    const int n0 = row_begin[u], nr = n_rows[u], n1 = n0 + nr;
    if (nr <= 0) return;
    const int p = n0 / S + blockIdx.x * wpc + warp;
    if ((int64_t)p * S >= n1) return;
    const size_t per_warp = (size_t)S * D * 4 + (size_t)D * 8;
    float *rows_s = reinterpret_cast<float *>(esmem + warp * per_warp);
    double *var_s = reinterpret_cast<double *>(esmem + warp * per_warp + (size_t)S * D * 4);
    const int64_t pid = page_table[u * Pmax + p];
    const int cnt = min(S, n1 - p * S);  // rows in the page after the extend
    const int r0 = max(0, n0 - p * S);   // rows it already held
    const char *kp = static_cast<const char *>(k_pool);
    if (r0 > 0) stage_rows_f32<DT, 8>(rows_s, D, kp + pid * S * D * ES, r0 * D, D, lane, 32);
    const int64_t srow = u * (int64_t)n_max + ((int64_t)p * S + r0 - n0);
    const int64_t prow = pid * S + r0;
    const char *ks = static_cast<const char *>(k_rows) + srow * D * ES;
    const char *vs = static_cast<const char *>(v_rows) + srow * D * ES;
    char *kd = static_cast<char *>(k_pool) + prow * D * ES;
    char *vd = static_cast<char *>(v_pool) + prow * D * ES;
    if ((D * ES) % 16 == 0) {
        copy_new_rows<DT, 8>(ks, vs, kd, vd, rows_s + r0 * D, (cnt - r0) * D * ES, lane);
    } else {
        for (int i = lane; i < (cnt - r0) * D; i += 32) {
            if constexpr (DT == PT_F32) {
                const float a = reinterpret_cast<const float *>(ks)[i];
                reinterpret_cast<float *>(kd)[i] = a;
                reinterpret_cast<float *>(vd)[i] = reinterpret_cast<const float *>(vs)[i];
                rows_s[r0 * D + i] = a;
            } else {
                const uint16_t a = reinterpret_cast<const uint16_t *>(ks)[i];
                reinterpret_cast<uint16_t *>(kd)[i] = a;
                reinterpret_cast<uint16_t *>(vd)[i] = reinterpret_cast<const uint16_t *>(vs)[i];
                rows_s[r0 * D + i] = bf16_bits_to_f32(a);
            }
        }
    }
    __syncwarp();
    double mean[DJ];
#pragma unroll
    for (int j = 0; j < DJ; j++) {
        const int d = lane + 32 * j;
        double sacc = 0.0;
        if (d < D)
            for (int r = 0; r < cnt; r++) sacc = __dadd_rn(sacc, (double)rows_s[r * D + d]);
        mean[j] = __ddiv_rn(sacc, (double)cnt);
    }
    constexpr int V = StatsTile<SDT>::V;
#pragma unroll
    for (int j = 0; j < DJ; j++) {
        const int d = lane + 32 * j;
        if (d < D) {
            double sacc = 0.0;
            for (int r = 0; r < cnt; r++) {
                const double t = __dsub_rn((double)rows_s[r * D + d], mean[j]);
                sacc = __dadd_rn(sacc, __dmul_rn(t, t));
            }
            var_s[d] = __ddiv_rn(sacc, (double)cnt);
            store_elem<SDT>(means, mean_offset(u, p, d, D, Pmax, V), __double2float_rn(mean[j]));
        }
    }
    if (mv.tiles) store_mirror<DJ>(mean, D, u, p, Pmax, mv, lane);
    __syncwarp();
    if (lane == 0) stds[u * Pmax + p] = __double2float_rn(__dsqrt_rn(np_sum(DoubleArray{var_s}, D)));
}

// extend (kvcache.py:210-233): scatter dense staged rows into mapped pages
template <typename E>
__global__ void k_write_rows(const E *__restrict__ k_rows, const E *__restrict__ v_rows,
                             int n_max, const int32_t *__restrict__ row_begin,
                             const int32_t *__restrict__ n_rows, E *__restrict__ k_pool,
                             E *__restrict__ v_pool, const int32_t *__restrict__ page_table,
                             int S, int D, int Pmax) {
    const int64_t u = blockIdx.y;
    const int nr = n_rows[u];
    const int r0 = row_begin[u];
    const int64_t total = (int64_t)nr * D;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(i / D), d = (int)(i % D);
        const int pos = r0 + r;
        const int64_t pid = page_table[u * Pmax + pos / S];
        const int64_t dst = (pid * S + pos % S) * D + d;
        const int64_t src = (u * n_max + r) * D + d;
        k_pool[dst] = k_rows[src];
        v_pool[dst] = v_rows[src];
    }
}

}  // namespace pt

using namespace pt;

template <int DT, int SDT>
static int launch_stats(const void *k_pool, const int32_t *pt_, const int32_t *sl,
                        const int32_t *pb, int U, int S, int D, int Pmax, void *means,
                        float *stds, const MirrorView mv, cudaStream_t st) {
    dim3 grid((Pmax + kStatsWarps - 1) / kStatsWarps, U);
    const int dj = (D + 31) / 32;
#define PT_STATS_CASE(DJ_)                                                                    \
    case DJ_:                                                                                 \
        k_page_stats<DT, SDT, DJ_><<<grid, kStatsWarps * 32, 0, st>>>(k_pool, pt_, sl, pb, S, D, \
                                                                       Pmax, means, stds, mv);    \
        break;
    switch (dj) {
        PT_STATS_CASE(1)
        PT_STATS_CASE(2)
        PT_STATS_CASE(3)
        PT_STATS_CASE(4)
        PT_STATS_CASE(8)
        PT_STATS_CASE(16)
        default: return PT_ERR_UNSUPPORTED;
    }
#undef PT_STATS_CASE
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}

static int stats_dj_ok(int D) {
    const int dj = (D + 31) / 32;
    return D >= 1 && D <= kMaxD && (dj <= 4 || dj == 8 || dj == 16);
}

extern "C" int pt_page_stats(const void *k_pool, int kv_dtype, const int32_t *page_table,
                             const int32_t *seq_len, const int32_t *page_begin, int U, int S,
                             int D, int Pmax, void *means, int stats_dtype, float *stds,
                             void *mirror, void *stream) {
    if (!k_pool || !page_table || !seq_len || !means || !stds || U < 0 || S < 1 || Pmax % 32 ||
        (mirror && (stats_dtype != PT_F32 || D % 8)))
        return PT_ERR_INVALID;
    if (!stats_dj_ok(D)) return PT_ERR_UNSUPPORTED;
    if (U == 0) return PT_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (kv_dtype == PT_F32 && stats_dtype == PT_F32)
        return launch_stats<PT_F32, PT_F32>(k_pool, page_table, seq_len, page_begin, U, S, D, Pmax, means, stds, mirror_view(mirror, U, Pmax, D), st);
    if (kv_dtype == PT_BF16 && stats_dtype == PT_F32)
        return launch_stats<PT_BF16, PT_F32>(k_pool, page_table, seq_len, page_begin, U, S, D, Pmax, means, stds, mirror_view(mirror, U, Pmax, D), st);
    if (kv_dtype == PT_BF16 && stats_dtype == PT_BF16)
        return launch_stats<PT_BF16, PT_BF16>(k_pool, page_table, seq_len, page_begin, U, S, D, Pmax, means, stds, mirror_view(mirror, U, Pmax, D), st);
    if (kv_dtype == PT_F32 && stats_dtype == PT_BF16)
        return launch_stats<PT_F32, PT_BF16>(k_pool, page_table, seq_len, page_begin, U, S, D, Pmax, means, stds, mirror_view(mirror, U, Pmax, D), st);
    return PT_ERR_INVALID;
}

template <int DT, int SDT>
static int launch_append(const void *kn, const void *vn, void *kp, void *vp, int32_t *ptab,
                         int32_t *sl, int U, int S, int D, int Pmax, void *means, float *stds,
                         int32_t *pool_state, const int32_t *free_list, int32_t *slot,
                         const MirrorView mv, cudaStream_t st, int32_t *step_sync) {
    const size_t per_warp = append_per_warp(S, D, DT == PT_F32 ? 4 : 2);
    if (per_warp > 200 * 1024) return PT_ERR_UNSUPPORTED;
    int wpc = (int)((200 * 1024) / per_warp);
    // spread the latency-bound per-unit warps over more SMs; thousands of units: keep the
    // whole grid resident in one wave
    int wmax = U >= 2048 ? 8 : 4;
    if (const char *we = getenv("PT_APP_WPC")) {  // tuning
        if (atoi(we) >= 1) wmax = atoi(we);
    }
    if (wpc > wmax) wpc = wmax;
    const size_t smem = per_warp * wpc;
    const int grid = (U + wpc - 1) / wpc;
    const int dj = (D + 31) / 32;
    const char *pe = getenv("PT_APP_PROF");
    const int app_prof = (pe && (*pe == '1' || *pe == '2')) ? *pe - '0' : 0;
#define PT_APP_CASE(DJ_)                                                                      \
    case DJ_: {                                                                               \
        static size_t configured = 0;                                                         \
        if (smem > configured) {                                                              \
            PT_CUDA_TRY(cudaFuncSetAttribute(k_append<DT, SDT, DJ_>,                          \
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                             (int)smem));                                     \
            PT_CUDA_TRY(cudaFuncSetAttribute(k_append<DT, SDT, DJ_>,                          \
                                             cudaFuncAttributePreferredSharedMemoryCarveout, \
                                             (int)cudaSharedmemCarveoutMaxShared));           \
            configured = smem;                                                                \
        }                                                                                     \
        PT_CUDA_TRY(pt_launch(k_append<DT, SDT, DJ_>, dim3(grid), dim3(wpc * 32), smem, st,   \
                              kn, vn, kp, vp, ptab, sl, U, S, D, Pmax, means, stds,           \
                              pool_state, free_list, slot, app_prof, mv, step_sync));         \
        break;                                                                                \
    }
    switch (dj) {
        PT_APP_CASE(1)
        PT_APP_CASE(2)
        PT_APP_CASE(3)
        PT_APP_CASE(4)
        PT_APP_CASE(8)
        PT_APP_CASE(16)
        default: return PT_ERR_UNSUPPORTED;
    }
#undef PT_APP_CASE
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}

static int append_impl(const void *k_new, const void *v_new, void *k_pool, void *v_pool,
                       int kv_dtype, int32_t *page_table, int32_t *seq_len, int U, int S, int D,
                       int Pmax, void *means, int stats_dtype, float *stds,
                       int32_t *pool_state, const int32_t *free_list, int32_t *slot_scratch,
                       void *mirror, void *stream, int32_t *step_sync) {
    if (!k_new || !v_new || !k_pool || !v_pool || !page_table || !seq_len || !means || !stds ||
        !pool_state || !slot_scratch || U < 0 || S < 1 || Pmax % 32 ||
        (mirror && (stats_dtype != PT_F32 || D % 8)))
        return PT_ERR_INVALID;
    if (!stats_dj_ok(D)) return PT_ERR_UNSUPPORTED;
    if (U == 0) return PT_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int32_t *slot = slot_scratch;
    if (kv_dtype == PT_F32 && stats_dtype == PT_F32)
        return launch_append<PT_F32, PT_F32>(k_new, v_new, k_pool, v_pool, page_table, seq_len, U, S, D, Pmax, means, stds, pool_state, free_list, slot, mirror_view(mirror, U, Pmax, D), st, step_sync);
    if (kv_dtype == PT_BF16 && stats_dtype == PT_F32)
        return launch_append<PT_BF16, PT_F32>(k_new, v_new, k_pool, v_pool, page_table, seq_len, U, S, D, Pmax, means, stds, pool_state, free_list, slot, mirror_view(mirror, U, Pmax, D), st, step_sync);
    if (kv_dtype == PT_BF16 && stats_dtype == PT_BF16)
        return launch_append<PT_BF16, PT_BF16>(k_new, v_new, k_pool, v_pool, page_table, seq_len, U, S, D, Pmax, means, stds, pool_state, free_list, slot, mirror_view(mirror, U, Pmax, D), st, step_sync);
    if (kv_dtype == PT_F32 && stats_dtype == PT_BF16)
        return launch_append<PT_F32, PT_BF16>(k_new, v_new, k_pool, v_pool, page_table, seq_len, U, S, D, Pmax, means, stds, pool_state, free_list, slot, mirror_view(mirror, U, Pmax, D), st, step_sync);
    return PT_ERR_INVALID;
}

extern "C" int pt_append(const void *k_new, const void *v_new, void *k_pool, void *v_pool,
                         int kv_dtype, int32_t *page_table, int32_t *seq_len, int U, int S, int D,
                         int Pmax, void *means, int stats_dtype, float *stds,
                         int32_t *pool_state, const int32_t *free_list, int32_t *slot_scratch,
                         void *mirror, void *stream) {
    return append_impl(k_new, v_new, k_pool, v_pool, kv_dtype, page_table, seq_len, U, S, D, Pmax,
                       means, stats_dtype, stds, pool_state, free_list, slot_scratch, mirror, stream,
                       nullptr);
}

// pt_append as the first link of a decode step whose scorer starts before the append has
// finished (pt_score_bounded_step, same step_sync): the append publishes two epochs --
// step_sync[0] once every unit's length is snapshotted (slot_scratch + U + 4), step_sync[1]
// once all its stores are visible
extern "C" int pt_append_step(const void *k_new, const void *v_new, void *k_pool, void *v_pool,
                              int kv_dtype, int32_t *page_table, int32_t *seq_len, int U, int S,
                              int D, int Pmax, void *means, int stats_dtype, float *stds,
                              int32_t *pool_state, const int32_t *free_list, int32_t *slot_scratch,
                              void *mirror, int32_t *step_sync, void *stream) {
    if (!step_sync) return PT_ERR_INVALID;
    return append_impl(k_new, v_new, k_pool, v_pool, kv_dtype, page_table, seq_len, U, S, D, Pmax,
                       means, stats_dtype, stds, pool_state, free_list, slot_scratch, mirror, stream,
                       step_sync);
}

// tuning aid: copy the phase timestamps of the last PT_APP_PROF=1 append (n <= 8 * 8192)
extern "C" int pt_debug_append_prof(unsigned long long *host, int n) {
    if (!host || n < 0 || n > kAppProfUnits * 8) return PT_ERR_INVALID;
    PT_CUDA_TRY(cudaMemcpyFromSymbol(host, g_app_prof, (size_t)n * 8));
    return PT_OK;
}

extern "C" int pt_write_rows(const void *k_rows, const void *v_rows, int n_max,
                             const int32_t *row_begin, const int32_t *n_rows, void *k_pool,
                             void *v_pool, int kv_dtype, const int32_t *page_table, int U, int S,
                             int D, int Pmax, void *stream) {
    if (!k_rows || !v_rows || !row_begin || !n_rows || !k_pool || !v_pool || !page_table ||
        U < 0 || n_max < 0)
        return PT_ERR_INVALID;
    if (U == 0 || n_max == 0) return PT_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int64_t per_unit = (int64_t)n_max * D;
    int gx = (int)((per_unit + 255) / 256);
    if (gx > 1024) gx = 1024;
    dim3 grid(gx, U);
    if (kv_dtype == PT_F32)
        k_write_rows<float><<<grid, 256, 0, st>>>((const float *)k_rows, (const float *)v_rows, n_max,
                                                  row_begin, n_rows, (float *)k_pool, (float *)v_pool,
                                                  page_table, S, D, Pmax);
    else if (kv_dtype == PT_BF16)
        k_write_rows<uint16_t><<<grid, 256, 0, st>>>((const uint16_t *)k_rows, (const uint16_t *)v_rows,
                                                     n_max, row_begin, n_rows, (uint16_t *)k_pool,
                                                     (uint16_t *)v_pool, page_table, S, D, Pmax);
    else
        return PT_ERR_INVALID;
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}

template <int DT, int SDT>
static int launch_extend(const void *kr, const void *vr, int n_max, const int32_t *rb,
                         const int32_t *nrw, void *kp, void *vp, const int32_t *ptab, int U, int S,
                         int D, int Pmax, void *means, float *stds, const MirrorView mv,
                         cudaStream_t st) {
    const size_t per_warp = (size_t)S * D * 4 + (size_t)D * 8;
    int wpc = (int)((96 * 1024) / per_warp);  // >= 2 CTAs per SM
    if (wpc > 8) wpc = 8;
    if (wpc < 1) return PT_ERR_UNSUPPORTED;
    const size_t smem = per_warp * wpc;
    const int pages = n_max / S + 2;  // pages one unit's rows can touch
    dim3 grid((pages + wpc - 1) / wpc, U);
    const int dj = (D + 31) / 32;
#define PT_EXT_CASE(DJ_)                                                                      \
    case DJ_: {                                                                               \
        static size_t configured = 0;                                                         \
        if (smem > configured) {                                                              \
            PT_CUDA_TRY(cudaFuncSetAttribute(k_extend<DT, SDT, DJ_>,                          \
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                             (int)smem));                                     \
            configured = smem;                                                                \
        }                                                                                     \
        k_extend<DT, SDT, DJ_><<<grid, wpc * 32, smem, st>>>(kr, vr, n_max, rb, nrw, kp, vp,  \
                                                             ptab, S, D, Pmax, means, stds,   \
                                                             mv);                             \
        break;                                                                                \
    }
    switch (dj) {
        PT_EXT_CASE(1)
        PT_EXT_CASE(2)
        PT_EXT_CASE(3)
        PT_EXT_CASE(4)
        PT_EXT_CASE(8)
        PT_EXT_CASE(16)
        default: return PT_ERR_UNSUPPORTED;
    }
#undef PT_EXT_CASE
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}

extern "C" int pt_extend(const void *k_rows, const void *v_rows, int n_max,
                         const int32_t *row_begin, const int32_t *n_rows, void *k_pool,
                         void *v_pool, int kv_dtype, const int32_t *page_table, int U, int S,
                         int D, int Pmax, void *means, int stats_dtype, float *stds,
                         void *mirror, void *stream) {
    if (!k_rows || !v_rows || !row_begin || !n_rows || !k_pool || !v_pool || !page_table ||
        !means || !stds || U < 0 || n_max < 0 || S < 1 || Pmax % 32 ||
        (mirror && (stats_dtype != PT_F32 || D % 8)))
        return PT_ERR_INVALID;
    if (!stats_dj_ok(D)) return PT_ERR_UNSUPPORTED;
    if (U == 0 || n_max == 0) return PT_OK;
    cudaStream_t st = (cudaStream_t)stream;
#define PT_EXT(DT_, SDT_)                                                                     \
    if (kv_dtype == DT_ && stats_dtype == SDT_)                                               \
        return launch_extend<DT_, SDT_>(k_rows, v_rows, n_max, row_begin, n_rows, k_pool,     \
                                        v_pool, page_table, U, S, D, Pmax, means, stds, mirror_view(mirror, U, Pmax, D), st);
    PT_EXT(PT_F32, PT_F32) PT_EXT(PT_BF16, PT_F32) PT_EXT(PT_BF16, PT_BF16) PT_EXT(PT_F32, PT_BF16)
#undef PT_EXT
    return PT_ERR_INVALID;
}
