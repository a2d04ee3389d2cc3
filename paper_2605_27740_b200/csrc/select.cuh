// select.cuh -- block-wide top-k page selection over ordered u16 keys staged in shared
// memory; shared by the standalone K3 kernel (topk.cu) and the fused score+select tail
// (score.cu).
//
// Restates select.py:87-115 + _kernels_cy.pyx:46-126.  The reference finds the threshold
// key (the k-th largest) with two 8-bit radix histogram rounds; here the same key is found
// by a 16-step bisection over the key space with block-wide counts (each thread owns a
// contiguous segment of keys; SIMD u16 compares, no atomics -- scores cluster in one or two
// radix buckets, which makes histogram atomics contend).  Given the threshold:
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

// number of u16 keys >= t among this thread's words i = tid, tid + NT, ... (strided:
// bank-conflict free; the count is order independent).  Packed-pair compare without the
// emulated SIMD intrinsics: hi >= t and lo >= t tested on the two halves.
template <int NT>
__device__ __forceinline__ int count_ge(const uint32_t *w, int nw, uint32_t t) {
    int c = 0;
    for (int i = threadIdx.x; i < nw; i += NT) {
        const uint32_t x = w[i];
        c += ((x & 0xFFFFu) >= t) + ((x >> 16) >= t);
    }
    return c;
}

// Select for one unit.  `skeys` (shared, 16-byte aligned, room for P + 1 keys) holds the
// unit's P keys.  Writes out/out_l [k]; thread 0 writes n_sel, kth, kplus1.
template <int NT>
__device__ void select_block(uint16_t *skeys, int P, int k, const int32_t *__restrict__ map,
                             int32_t *__restrict__ out, int32_t *__restrict__ out_l,
                             int32_t *__restrict__ n_sel, int32_t *__restrict__ kth,
                             int32_t *__restrict__ kplus1, SelectShared<NT> &sh) {
    const int tid = threadIdx.x;
    if (P <= k) {  // _take_all
        int mn = 0xFFFF;
        for (int i = tid; i < P; i += NT) {
            out[i] = map[i];
            if (out_l) out_l[i] = i;
            mn = min(mn, (int)skeys[i]);
        }
        mn = __reduce_min_sync(0xffffffffu, mn);
        __syncthreads();
        if ((tid & 31) == 0) sh.warp_a[tid >> 5] = mn;
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
    // pad the key array to an even count with 0 (key 0 never counts for t >= 1 and is
    // excluded explicitly below), segments of whole 32-bit words
    if (tid == 0 && (P & 1)) skeys[P] = 0;
    __syncthreads();
    const uint32_t *w = reinterpret_cast<const uint32_t *>(skeys);
    const int nw = (P + 1) >> 1;
    const int wseg = (nw + NT - 1) / NT;
    const int w0 = min(tid * wseg, nw), w1 = min(w0 + wseg, nw);
    // bisection: thr = max t with #(keys >= t) >= k   (t = 0 always qualifies; the odd-P
    // padding key 0 never counts for the probed t >= 1)
    int lo = 0, hi = 0x10000;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        const int tot = block_sum<NT>(count_ge<NT>(w, nw, (uint32_t)mid), sh);
        if (tot >= k) lo = mid; else hi = mid;
    }
    const int thr = lo;
    // per-segment counts of > thr and == thr (in logical order: key index 2*word + half)
    const int i0 = min(2 * w0, P), i1 = min(2 * w1, P);
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
    if ((tid & 31) == 0) sh.warp_a[tid >> 5] = below;
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
