// select.cuh -- block-wide top-k page selection over ordered u16 keys staged in shared
// memory; shared by the standalone K3 kernel (topk.cu) and the fused score+select tail
// (score.cu).
//
// Restates select.py:87-115 + _kernels_cy.pyx:46-126.  The reference finds the threshold
// key (the k-th largest) with two 8-bit radix histogram rounds; here the same key is found
// with one histogram over the keys' actual range (or a bisection when that range is wide).
// Given the threshold:
//   selected = keys > thr  +  the first (k - #>thr) keys == thr in ascending LOGICAL index
//   (the reference's tie rule) -- an ordered compaction by block-wide
//   exclusive scans over the contiguous segments;
//   kplus1 = thr if ties are left over, else the largest key below thr;
//   P <= k -> every page, kth = min key, kplus1 = -1 (select.py:75-84, 100-101).
// Results are bit-identical to the reference's (ids as a set, emitted in ascending
// logical order, translated logical -> physical through the page table).
#pragma once
#include "common.cuh"

namespace pt {

template <int NT>
struct SelectShared {
    int warp_a[NT / 32];
    int warp_b[NT / 32];
};

// block-wide sum of one int (all threads get the total)
template <int NT>
__device__ __forceinline__ int block_sum(int v, SelectShared<NT> &sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = __reduce_add_sync(0xffffffffu, v);
    __syncthreads();
    if (lane == 0) sh.warp_a[warp] = v;
    __syncthreads();
    int t = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; w++) t += sh.warp_a[w];
    return t;
}

// block-wide exclusive scan of two counters (+ totals)
template <int NT>
__device__ __forceinline__ void block_exscan2(int a, int b, int &ea, int &eb, int &ta, int &tb,
                                              SelectShared<NT> &sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int ia = a, ib = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int xa = __shfl_up_sync(0xffffffffu, ia, o);
        const int xb = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) { ia += xa; ib += xb; }
    }
    __syncthreads();
    if (lane == 31) { sh.warp_a[warp] = ia; sh.warp_b[warp] = ib; }
    __syncthreads();
    int pa = 0, pb = 0, sa = 0, sb = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; w++) {
        const int wa = sh.warp_a[w], wb = sh.warp_b[w];
        if (w < warp) { pa += wa; pb += wb; }
        sa += wa;
        sb += wb;
    }
    ea = pa + ia - a;
    eb = pb + ib - b;
    ta = sa;
    tb = sb;
}

// Select for one unit.  `skeys` (shared, 16-byte aligned, room for P + 1 keys) holds the
// unit's P keys; `bins` (shared, kSelectBins ints) is histogram scratch.  Writes
// out/out_l [k]; thread 0 writes n_sel, kth, kplus1.
//
// Threshold search: one pass for the key range [mn, mx]; when it spans <= kSelectBins
// values (always, in practice: scores cluster in a few dozen bf16 values) a single
// shared-memory histogram of (key - mn) and a descending block scan over the bins give the
// k-th largest key; otherwise a bisection over [mn, mx] with block-wide counts.
constexpr int kSelectBins = 4096;

template <int NT>
__device__ void select_block(uint16_t *skeys, int *bins, int P, int k,
                             const int32_t *__restrict__ map, int32_t *__restrict__ out,
                             int32_t *__restrict__ out_l, int32_t *__restrict__ n_sel,
                             int32_t *__restrict__ kth, int32_t *__restrict__ kplus1,
                             SelectShared<NT> &sh) {
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    if (P <= k) {  // _take_all
        int mn = 0xFFFF;
        for (int i = tid; i < P; i += NT) {
            out[i] = map[i];
            if (out_l) out_l[i] = i;
            mn = min(mn, (int)skeys[i]);
        }
        mn = __reduce_min_sync(0xffffffffu, mn);
        __syncthreads();
        if (lane == 0) sh.warp_a[warp] = mn;
        __syncthreads();
        if (tid == 0) {
            int m = 0xFFFF;
            for (int w = 0; w < NT / 32; w++) m = min(m, sh.warp_a[w]);
            *n_sel = P;
            *kth = m;
            *kplus1 = -1;
        }
        return;
    }
    if (tid == 0 && (P & 1)) skeys[P] = skeys[P - 1];  // pad: duplicate (counted only below)
    __syncthreads();
    const uint32_t *w = reinterpret_cast<const uint32_t *>(skeys);
    const int nw = P >> 1;  // full words; an odd tail key is handled separately
    // ---- key range ----
    int mn = 0xFFFF, mx = 0;
    for (int i = tid; i < nw; i += NT) {
        const uint32_t x = w[i];
        const int lo = x & 0xFFFF, hi = x >> 16;
        mn = min(mn, min(lo, hi));
        mx = max(mx, max(lo, hi));
    }
    if ((P & 1) && tid == 0) { mn = min(mn, (int)skeys[P - 1]); mx = max(mx, (int)skeys[P - 1]); }
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    __syncthreads();
    if (lane == 0) { sh.warp_a[warp] = mn; sh.warp_b[warp] = mx; }
    __syncthreads();
    mn = 0xFFFF;
    mx = 0;
#pragma unroll
    for (int i = 0; i < NT / 32; i++) { mn = min(mn, sh.warp_a[i]); mx = max(mx, sh.warp_b[i]); }
    const int R = mx - mn + 1;
    int thr;
    if (R <= kSelectBins) {
        // ---- one-pass histogram of (key - mn) ----
        for (int i = tid; i < R; i += NT) bins[i] = 0;
        __syncthreads();
        for (int i = tid; i < nw; i += NT) {
            const uint32_t x = w[i];
            atomicAdd(&bins[(int)(x & 0xFFFF) - mn], 1);
            atomicAdd(&bins[(int)(x >> 16) - mn], 1);
        }
        if ((P & 1) && tid == 0) atomicAdd(&bins[(int)skeys[P - 1] - mn], 1);
        __syncthreads();
        // descending segments of bins: thread t owns [top_t - seg + 1, top_t]
        const int seg = (R + NT - 1) / NT;
        const int top = R - 1 - tid * seg;
        int s = 0;
        for (int j = 0; j < seg; j++) {
            const int bb = top - j;
            if (bb >= 0) s += bins[bb];
        }
        int above, dummy, tot, dummy2;
        block_exscan2<NT>(s, 0, above, dummy, tot, dummy2, sh);
        __syncthreads();
        if (above < k && above + s >= k) {  // the crossing segment
            int cum = above;
            for (int j = 0; j < seg; j++) {
                const int bb = top - j;
                cum += bins[bb];
                if (cum >= k) { sh.warp_a[0] = mn + bb; break; }
            }
        }
        __syncthreads();
        thr = sh.warp_a[0];
    } else {
        // ---- bisection over [mn, mx]: thr = max t with #(keys >= t) >= k ----
        int lo = mn, hi = mx + 1;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            int c = 0;
            for (int i = tid; i < nw; i += NT) {
                const uint32_t x = w[i];
                c += ((int)(x & 0xFFFF) >= mid) + ((int)(x >> 16) >= mid);
            }
            if ((P & 1) && tid == 0) c += (int)skeys[P - 1] >= mid;
            const int tot = block_sum<NT>(c, sh);
            if (tot >= k) lo = mid; else hi = mid;
        }
        thr = lo;
    }
    // ---- ordered compaction over contiguous per-thread segments (logical order) ----
    const int kseg = (P + NT - 1) / NT;
    const int i0 = min(tid * kseg, P), i1 = min(i0 + kseg, P);
    int gt = 0, eq = 0, below = -1;
    for (int i = i0; i < i1; i++) {
        const int key = skeys[i];
        gt += key > thr;
        eq += key == thr;
        if (key < thr) below = max(below, key);
    }
    int eq_before, gt_before, eq_tot, gt_tot;
    block_exscan2<NT>(eq, gt, eq_before, gt_before, eq_tot, gt_tot, sh);
    const int tie_budget = k - gt_tot;
    const int take = max(0, min(eq, tie_budget - eq_before));
    int pos, dummy, tot_sel, dummy2;
    block_exscan2<NT>(gt + take, 0, pos, dummy, tot_sel, dummy2, sh);
    int taken = 0;
    for (int i = i0; i < i1; i++) {
        const int key = skeys[i];
        bool s = key > thr;
        if (key == thr && taken < take) { s = true; taken++; }
        if (s) {
            out[pos] = map[i];
            if (out_l) out_l[pos] = i;
            pos++;
        }
    }
    below = __reduce_max_sync(0xffffffffu, below);
    __syncthreads();
    if (lane == 0) sh.warp_a[warp] = below;
    __syncthreads();
    if (tid == 0) {
        int m = -1;
        for (int wi = 0; wi < NT / 32; wi++) m = max(m, sh.warp_a[wi]);
        *n_sel = k;
        *kth = thr;
        *kplus1 = (eq_tot > tie_budget) ? thr : m;
    }
}

}  // namespace pt
