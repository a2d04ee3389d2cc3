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
// out/out_l [k]; thread 0 writes n_sel, kth, kplus1.  With `slist` (shared, k ints) the
// compaction emits logical ids there and the page-table translation runs as one parallel
// round of loads after it (instead of a dependent global load per selected page inside
// each thread's serial compaction loop); on return slist holds the selected ids in
// emission order -- logical, or physical with `slist_physical` (the fused attention
// kernel streams straight from that list).  `out`/`out_l` may then be null.
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
                             SelectShared<NT> &sh, int *slist = nullptr,
                             bool slist_physical = false, unsigned long long *tp = nullptr) {
    // tp (tuning aid): thread 0 stamps %globaltimer after each phase
    auto stamp = [&](int i) {
        if (tp && threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            tp[i] = t;
        }
    };
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    if (P <= k) {  // _take_all
        int mn = 0xFFFF;
        for (int i = tid; i < P; i += NT) {
            const int pid = (out || (slist && slist_physical)) ? __ldg(map + i) : 0;
            if (out) out[i] = pid;
            if (out_l) out_l[i] = i;
            if (slist) slist[i] = slist_physical ? pid : i;
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
    stamp(0);
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
    int thr = -1;
    stamp(1);
    // ---- fast path: the k-th largest key among the top 64 values below the maximum ----
    // Lane-private u16 counters (a 32 x 32 word grid per warp, lane = column, so increments
    // never conflict -- contended shared atomics on the few hot bins of clustered scores
    // cost ~10 us per unit), summed by 32 warp reductions; falls through when the top 64
    // values hold fewer than k keys.
    if constexpr ((NT / 32) * 1024 <= kSelectBins) {
        if (P / (NT / 32) < 65536 && R > 1) {
            uint32_t *hw = reinterpret_cast<uint32_t *>(bins) + warp * 1024;
#pragma unroll 8
            for (int r = 0; r < 32; r++) hw[r * 32 + lane] = 0u;
            for (int i = tid; i < nw; i += NT) {
                const uint32_t x = w[i];
                const int b0 = mx - (int)(x & 0xFFFF), b1 = mx - (int)(x >> 16);
                if (b0 < 64) hw[(b0 >> 1) * 32 + lane] += 1u << ((b0 & 1) * 16);
                if (b1 < 64) hw[(b1 >> 1) * 32 + lane] += 1u << ((b1 & 1) * 16);
            }
            if ((P & 1) && tid == 0) {
                const int b = mx - (int)skeys[P - 1];
                if (b < 64) hw[(b >> 1) * 32 + lane] += 1u << ((b & 1) * 16);
            }
            __syncwarp();
            uint32_t mine = 0u;  // lane r: this warp's counts of bins 2r (lo) and 2r+1 (hi)
#pragma unroll 8
            for (int r = 0; r < 32; r++) {
                const uint32_t v = __reduce_add_sync(0xffffffffu, hw[r * 32 + lane]);
                if (lane == r) mine = v;
            }
            __syncwarp();
            hw[lane] = mine;
            __syncthreads();
            if (warp == 0) {
                int c0 = 0, c1 = 0;
#pragma unroll
                for (int wi = 0; wi < NT / 32; wi++) {
                    const uint32_t v = reinterpret_cast<const uint32_t *>(bins)[wi * 1024 + lane];
                    c0 += (int)(v & 0xFFFFu);
                    c1 += (int)(v >> 16);
                }
                int inc = c0 + c1;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (lane >= o) inc += y;
                }
                const int pre = inc - c0 - c1;
                int t = -1;
                if (pre < k && pre + c0 >= k) t = mx - 2 * lane;
                else if (pre + c0 < k && inc >= k) t = mx - 2 * lane - 1;
                t = __reduce_max_sync(0xffffffffu, t);
                if (lane == 0) sh.warp_a[0] = t;
            }
            __syncthreads();
            thr = sh.warp_a[0];
            __syncthreads();
        }
    }
    if (thr >= 0) {
        // threshold found by the fast path
    } else if (R <= kSelectBins) {
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
    stamp(2);
    // ---- ordered compaction (logical order), warp-segmented ----
    // Warp w owns a contiguous run of key words; each step a warp reads 32 consecutive words
    // (64 keys, bank-conflict free) and ranks them with ballots, so positions and the
    // lowest-logical-index tie budget follow the logical order exactly.
    constexpr int NWARPS = NT / 32;
    const unsigned lt = (1u << lane) - 1u;
    const int nwt = (P + 1) >> 1;
    const int segw = (((nwt + NWARPS - 1) / NWARPS) + 31) & ~31;
    const int wb = min(warp * segw, nwt), we = min(wb + segw, nwt);
    int gt = 0, eq = 0, below = -1;
    for (int i = wb + lane; i < we; i += 32) {
        const uint32_t x = w[i];
        const int k0 = x & 0xFFFF, k1 = x >> 16;
        const bool v1 = 2 * i + 1 < P;
        gt += (k0 > thr) + (v1 && k1 > thr);
        eq += (k0 == thr) + (v1 && k1 == thr);
        if (k0 < thr) below = max(below, k0);
        if (v1 && k1 < thr) below = max(below, k1);
    }
    gt = __reduce_add_sync(0xffffffffu, gt);
    eq = __reduce_add_sync(0xffffffffu, eq);
    __syncthreads();
    if (lane == 0) { sh.warp_a[warp] = gt; sh.warp_b[warp] = eq; }
    __syncthreads();
    int gt_before = 0, eq_before = 0, gt_tot = 0, eq_tot = 0;
#pragma unroll
    for (int wi = 0; wi < NWARPS; wi++) {
        const int a2 = sh.warp_a[wi], b2 = sh.warp_b[wi];
        if (wi < warp) { gt_before += a2; eq_before += b2; }
        gt_tot += a2;
        eq_tot += b2;
    }
    const int tie_budget = k - gt_tot;  // in [1, eq_tot]: thr is the k-th largest key
    int run_sel = gt_before + min(eq_before, tie_budget);
    int run_eq = eq_before;
    for (int base = wb; base < we; base += 32) {
        const int i = base + lane;
        const bool v0 = i < we, v1 = v0 && 2 * i + 1 < P;
        const uint32_t x = v0 ? w[i] : 0u;
        const int k0 = x & 0xFFFF, k1 = x >> 16;
        const bool e0 = v0 && k0 == thr, e1 = v1 && k1 == thr;
        const unsigned be0 = __ballot_sync(0xffffffffu, e0), be1 = __ballot_sync(0xffffffffu, e1);
        const int t0 = run_eq + __popc(be0 & lt) + __popc(be1 & lt);  // ties before key 2i
        const bool s0 = (v0 && k0 > thr) || (e0 && t0 < tie_budget);
        const bool s1 = (v1 && k1 > thr) || (e1 && t0 + (int)e0 < tie_budget);
        const unsigned bs0 = __ballot_sync(0xffffffffu, s0), bs1 = __ballot_sync(0xffffffffu, s1);
        const int p0 = run_sel + __popc(bs0 & lt) + __popc(bs1 & lt);
        if (s0 || s1) {
            const int p1 = p0 + (int)s0;
            if (slist) {
                if (s0) slist[p0] = 2 * i;
                if (s1) slist[p1] = 2 * i + 1;
            } else {
                if (s0) { out[p0] = map[2 * i]; if (out_l) out_l[p0] = 2 * i; }
                if (s1) { out[p1] = map[2 * i + 1]; if (out_l) out_l[p1] = 2 * i + 1; }
            }
        }
        run_eq += __popc(be0) + __popc(be1);
        run_sel += __popc(bs0) + __popc(bs1);
    }
    stamp(3);
    if (slist) {
        __syncthreads();
        for (int t = tid; t < k; t += NT) {
            const int li = slist[t];
            const int pid = __ldg(map + li);
            if (out) out[t] = pid;
            if (out_l) out_l[t] = li;
            if (slist_physical) slist[t] = pid;
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

// ---------------------------------------------------------------------------
// Fast block selection over keys staged in shared memory (the fused select+attend prologue).
//
// Keys are processed as u16x2 words with the SIMD video instructions (VIMNMX/VSET-style
// __vcmpgeu2 / __vmaxu2): 8 keys per 16-byte shared load, ~1.5 instructions per key per pass.
// 1. threshold thr (the k-th largest key):
//    - with the scoring kernel's per-32-page tile maxima (>= k tiles): L = the k-th largest
//      tile maximum is a lower bound for thr (k distinct tiles each hold a key >= L); for
//      decode-step scores only ~1-3 % of the keys reach it.  One pass appends the keys >= L
//      to a candidate list in ascending logical order; thr = the k-th largest candidate
//      (64-bin histogram over [L, max], or bisection over the candidates);
//    - otherwise (no tile maxima, fewer tiles than k, or too many candidates): bisection over
//      [min, max] with block-wide counts (exact for any key distribution);
// 2. ordered compaction: keys > thr plus the first (k - #>thr) keys == thr in ascending
//    logical index -- the reference's rule -- over the candidate list when there is one, else
//    over all keys (one block scan per round of NT key vectors); physical ids by one parallel
//    round of page-table loads.
// Emission order is ascending logical (the same list as select_block).  Returns false only
// for the take-all case (P <= k) and P > 65536 (the caller runs select_block).
// ---------------------------------------------------------------------------
constexpr int kCandMax = 2048;

template <int NT>
struct SelectCandShared {
    uint32_t red[2][NT / 32][2];
    int bins[64];
    int below, thr, gt, eq;
    int hist[256];  // radix rounds (no tile-maximum bound)
    uint32_t cand[kCandMax];
};

// Bounded mode (attend_fused.cu with pt_score_bounded's key intervals): skeys holds the
// interval's lower keys, `resolve(L)` (block-wide) replaces the key of every page whose
// interval reaches L by its exact key and returns the largest key it wrote (or -1), and L is
// the kL-th (= k + 1-th) largest tile maximum -- so the k + 1 largest exact keys all lie in
// the candidate list and everything below it is strictly smaller.
struct NoResolve {
    __device__ int operator()(int) const { return -1; }
};
struct NoResolveCands {
    __device__ void operator()(int, int, int) const {}
};

template <int NT, class Resolve = NoResolve, class ResolveCands = NoResolveCands>
__device__ bool select_cand(const uint16_t *__restrict__ skeys, const uint16_t *__restrict__ tmax_g,
                            int P, int k, const int32_t *__restrict__ map,
                            int32_t *__restrict__ out, int32_t *__restrict__ out_l,
                            int32_t *__restrict__ n_sel, int32_t *__restrict__ kth,
                            int32_t *__restrict__ kplus1, SelectCandShared<NT> &sh, int *slist,
                            bool slist_physical, unsigned long long *tp = nullptr,
                            bool tmax_shared = false, int kL = 0,
                            const Resolve &resolve = Resolve(), const uint16_t *shi = nullptr,
                            uint16_t *candhi = nullptr,
                            const ResolveCands &resolve_cands = ResolveCands(),
                            int *defer = nullptr, bool tclk = false) {
    constexpr int NWP = NT / 32;
    constexpr int MAXT = 8;  // tile maxima per thread: ceil(P / 32) <= NT * MAXT
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (P <= k || P > 65536) return false;
    const int kl = kL > 0 ? kL : k;
    auto stamp = [&](int i) {
        if (tp && tid == 0) {
            unsigned long long t;
            if (tclk) asm volatile("mov.u64 %0, %clock64;" : "=l"(t));
            else asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            tp[i] = t;
        }
    };
    const uint4 *s4 = reinterpret_cast<const uint4 *>(skeys);
    const int nvec = (P + 7) >> 3;
    const int tailn = P - (nvec - 1) * 8;  // valid keys in the last vector (1..8)
    // per-word validity masks of vector v (only the last one can be partial)
    auto vmask = [&](int v, uint32_t (&m)[4]) {
#pragma unroll
        for (int w = 0; w < 4; w++) {
            const int nk = v < nvec - 1 ? 8 : tailn;
            const int lo = 2 * w, hi = 2 * w + 1;
            m[w] = (lo < nk ? 0x0000FFFFu : 0u) | (hi < nk ? 0xFFFF0000u : 0u);
        }
    };
    auto words = [](const uint4 &x, uint32_t (&w)[4]) { w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w; };
    // count of valid keys >= t (t16 = t * 0x10001) in vector v
    auto count_ge = [&](const uint4 &x, int v, uint32_t t16) -> int {
        uint32_t w[4], m[4];
        words(x, w);
        vmask(v, m);
        int c = 0;
#pragma unroll
        for (int q = 0; q < 4; q++) c += __popc(__vcmpgeu2(w[q], t16) & m[q]);
        return c >> 4;
    };
    auto block_sum = [&](int v) -> int {
        v = __reduce_add_sync(0xffffffffu, v);
        __syncthreads();
        if (lane == 0) sh.red[0][warp][0] = (uint32_t)v;
        __syncthreads();
        int t = 0;
#pragma unroll
        for (int w = 0; w < NWP; w++) t += (int)sh.red[0][w][0];
        return t;
    };
    auto block_max = [&](int v) -> int {
        v = __reduce_max_sync(0xffffffffu, v);
        __syncthreads();
        if (lane == 0) sh.red[0][warp][1] = (uint32_t)v;
        __syncthreads();
        int t = -1;
#pragma unroll
        for (int w = 0; w < NWP; w++) t = max(t, (int)sh.red[0][w][1]);
        return t;
    };
    const int ntiles = (P + 31) >> 5;
    const bool use_tiles = tmax_g != nullptr && ntiles >= kl && ntiles <= NT * MAXT;
    int tm[MAXT];
#pragma unroll
    for (int i = 0; i < MAXT; i++) {
        const int t = tid + i * NT;
        tm[i] = (use_tiles && t < ntiles) ? (int)(tmax_shared ? tmax_g[t] : __ldcg(tmax_g + t)) : -1;
    }
    if (tid < 64) sh.bins[tid] = 0;
    if (tid == 0) { sh.below = -1; sh.eq = -1; }
    int mx, mn = 0, L = -1;
    if (use_tiles) {
        int m = -1;
#pragma unroll
        for (int i = 0; i < MAXT; i++) m = max(m, tm[i]);
        mx = block_max(m);  // the largest tile maximum is the largest key
        auto round8 = [&](int lo, int shift, int (&tot)[8]) {
            unsigned long long c = 0ull;
#pragma unroll
            for (int i = 0; i < MAXT; i++) {
                const int d = mx - tm[i] - lo, b = d >> shift;
                if (tm[i] >= 0 && d >= 0 && b < 8) c += 1ull << (8 * b);
            }
            __syncthreads();
#pragma unroll
            for (int b = 0; b < 8; b++) {
                const int x = __reduce_add_sync(0xffffffffu, (uint32_t)((c >> (8 * b)) & 0xFFu));
                if (lane == 0) sh.bins[b * NWP + warp] = x;
            }
            __syncthreads();
#pragma unroll
            for (int b = 0; b < 8; b++) {
                int t = 0;
#pragma unroll
                for (int w = 0; w < NWP; w++) t += sh.bins[b * NWP + w];
                tot[b] = t;
            }
        };
        static_assert(8 * (NT / 32) <= 64, "bins scratch");
        int ta[8], tb[8];
        round8(0, 3, ta);
        int ia = -1, cum = 0, before = 0;
#pragma unroll
        for (int b = 0; b < 8; b++) {
            if (ia < 0 && cum + ta[b] >= kl) { ia = b; before = cum; }
            cum += ta[b];
        }
        if (ia >= 0) {
            round8(8 * ia, 0, tb);
            int c2 = before, ib = 7;
            bool done = false;
#pragma unroll
            for (int b = 0; b < 8; b++) {
                if (!done && c2 + tb[b] >= kl) { ib = b; done = true; }
                c2 += tb[b];
            }
            L = mx - (8 * ia + ib);
        }
        __syncthreads();
        if (tid < 64) sh.bins[tid] = 0;
        // bounded mode: the candidates are resolved after the candidate pass (only those
        // meeting the threshold bracket); without tile-maximum bound every uncertain key now
        if (!shi || L < 0) mx = max(mx, resolve(L));
    } else {
        resolve(-1);
        int m = -1, n = 0xFFFF;
        for (int v = tid; v < nvec; v += NT) {
            uint32_t w[4], mk[4];
            words(s4[v], w);
            vmask(v, mk);
            uint32_t a = 0u, b = 0xFFFFFFFFu;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                a = __vmaxu2(a, w[q] & mk[q]);
                b = __vminu2(b, w[q] | ~mk[q]);
            }
            m = max(m, (int)max(a & 0xFFFFu, a >> 16));
            n = min(n, (int)min(b & 0xFFFFu, b >> 16));
        }
        mx = block_max(m);
        mn = 0xFFFF - block_max(0xFFFF - n);
    }
    stamp(0);
    int thr = -1, gt_tot = 0, eq_tot = 0, C = -1;
    if (L >= 0) {
        // ---- candidates >= L in logical order: each round a thread owns VPT consecutive
        // key vectors (so thread order is logical order) and one block scan ranks them ----
        constexpr int VPT = 4;
        const uint32_t L16 = (uint32_t)L * 0x10001u;
        int run = 0, below = -1, par = 0, mhi = -1;
        for (int v0 = 0; v0 < nvec; v0 += NT * VPT, par ^= 1) {
            const int vt = v0 + tid * VPT;
            uint4 x[VPT], y[VPT];
            int cv[VPT];
            int c = 0;
#pragma unroll
            for (int j = 0; j < VPT; j++) {
                const int v = vt + j;
                x[j] = make_uint4(0u, 0u, 0u, 0u);
                y[j] = x[j];
                cv[j] = 0;
                if (v < nvec) {
                    x[j] = s4[v];
                    y[j] = shi ? reinterpret_cast<const uint4 *>(shi)[v] : x[j];
                    uint32_t w[4], wh[4], mk[4];
                    words(x[j], w);
                    words(y[j], wh);
                    vmask(v, mk);
                    uint32_t bl = 0u;
                    bool any_below = false;
                    int cc = 0;
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const uint32_t ge = __vcmpgeu2(wh[q], L16);  // bounded: the upper key
                        cc += __popc(ge & mk[q]);
                        const uint32_t lt = ~ge & mk[q];
                        any_below |= lt != 0u;
                        bl = __vmaxu2(bl, w[q] & lt);
                    }
                    cv[j] = cc >> 4;
                    c += cv[j];
                    if (any_below) below = max(below, (int)max(bl & 0xFFFFu, bl >> 16));
                }
            }
            int inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) sh.red[par][warp][0] = (uint32_t)inc;
            __syncthreads();
            int pos = run + inc - c;
#pragma unroll
            for (int w = 0; w < NWP; w++) {
                const int t = (int)sh.red[par][w][0];
                if (w < warp) pos += t;
                run += t;
            }
            if (c) {
                // the vector's candidates as an 8-bit mask, appended by a loop over its set bits
                // (a short loop, not 8 unrolled copies: this code runs once per CTA, so its
                // instruction footprint is most of its cost)
#pragma unroll
                for (int j = 0; j < VPT; j++) {
                    if (!cv[j]) continue;
                    const int v = vt + j;
                    uint32_t wh[4], mk[4];
                    words(y[j], wh);
                    vmask(v, mk);
                    uint32_t bits = 0u;
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const uint32_t ge = __vcmpgeu2(wh[q], L16) & mk[q];
                        bits |= ((ge & 1u) | ((ge >> 15) & 2u)) << (2 * q);
                    }
                    const uint64_t lo64 = ((uint64_t)x[j].y << 32) | x[j].x, lo64b = ((uint64_t)x[j].w << 32) | x[j].z;
                    const uint64_t hi64 = ((uint64_t)y[j].y << 32) | y[j].x, hi64b = ((uint64_t)y[j].w << 32) | y[j].z;
                    for (; bits; bits &= bits - 1u) {
                        const int e = __ffs(bits) - 1;
                        const int sft = 16 * (e & 3);
                        const int key = (int)(((e < 4 ? lo64 : lo64b) >> sft) & 0xFFFFu);
                        const int kh = (int)(((e < 4 ? hi64 : hi64b) >> sft) & 0xFFFFu);
                        if (pos < kCandMax) {
                            sh.cand[pos] = ((uint32_t)key << 16) | (uint32_t)(v * 8 + e);
                            if (candhi) candhi[pos] = (uint16_t)kh;
                        }
                        pos++;
                        mhi = max(mhi, kh);
                    }
                }
            }
        }
        below = __reduce_max_sync(0xffffffffu, below);
        mhi = __reduce_max_sync(0xffffffffu, mhi);
        if (lane == 0) { atomicMax(&sh.below, below); atomicMax(&sh.eq, mhi); }  // eq: max upper key
        __syncthreads();
        if (run <= kCandMax) C = run;  // else: too many keys tie at L -- bisection below
    }
    if (shi && L >= 0) {
        stamp(10);
        if (C >= 0) {
            // bounded mode, threshold bracket over the candidates: A = the (k+1)-th largest
            // lower key <= the exact (k+1)-th key, B = the k-th largest upper key >= the exact
            // threshold.  Only uncertain candidates whose interval meets [A, B] need their exact
            // key: the others are certainly above the threshold (lower key > B) or certainly
            // below the (k+1)-th key (upper key < A), so their counts, ties and kplus1 are
            // decided either way.
            const int mxh = sh.eq;  // the largest candidate upper key (candidate pass)
            stamp(11);
            int A = L, B = mxh;
            if (mxh - L < 64) {
                // both ranks from one pass: upper keys -> bins (B = k-th largest), lower keys
                // reaching L -> hist (A = (k+1)-th largest); warps 0 and 1 scan in parallel
                if (tid < 64) { sh.bins[tid] = 0; sh.hist[tid] = 0; }
                __syncthreads();
                for (int i = tid; i < C; i += NT) {
                    atomicAdd(&sh.bins[mxh - (int)candhi[i]], 1);
                    const int lo = (int)(sh.cand[i] >> 16);
                    if (lo >= L) atomicAdd(&sh.hist[mxh - lo], 1);
                }
                __syncthreads();
                if (warp < 2) {
                    const int *hb = warp == 0 ? sh.bins : sh.hist;
                    const int rank = warp == 0 ? k : k + 1;
                    const int c0 = hb[2 * lane], c1 = hb[2 * lane + 1];
                    int incl = c0 + c1;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y2 = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y2;
                    }
                    const int pre = incl - c0 - c1;
                    int bb = 999;
                    if (pre < rank && pre + c0 >= rank) bb = 2 * lane;
                    else if (pre + c0 < rank && incl >= rank) bb = 2 * lane + 1;
                    bb = __reduce_min_sync(0xffffffffu, bb);
                    if (lane == 0) sh.red[1][warp][0] = (uint32_t)(bb < 999 ? bb : 63);
                }
                __syncthreads();
                B = mxh - (int)sh.red[1][0][0];
                A = mxh - (int)sh.red[1][1][0];
                stamp(12);
                stamp(13);
                __syncthreads();
                if (tid < 64) sh.bins[tid] = 0;
            }
            if (defer) {
                // the caller finishes the selection itself (attend_fused.cu: the certainly
                // selected pages -- lower key > B -- stream while 4 warps resolve the bracket)
                if (tid == 0) {
                    defer[0] = 1; defer[1] = C; defer[2] = L; defer[3] = A; defer[4] = B;
                    defer[5] = sh.below;
                }
                __syncthreads();
                return true;
            }
            resolve_cands(C, A, B);
            int m2 = -1;
            for (int i = tid; i < C; i += NT) m2 = max(m2, (int)(sh.cand[i] >> 16));
            mx = max(mx, block_max(m2));
        } else {
            mx = max(mx, resolve(L));  // candidate overflow: resolve the key array
        }
    }
    stamp(1);
    if (C >= 0) {
        // ---- thr = the k-th largest candidate ----
        if (mx - L < 64) {
            // (bounded mode: candidates whose key ended below L are below the threshold)
            for (int i = tid; i < C; i += NT) {
                const int key = (int)(sh.cand[i] >> 16);
                if (key >= L) atomicAdd(&sh.bins[mx - key], 1);
            }
            __syncthreads();
            if (warp == 0) {
                const int c0 = sh.bins[2 * lane], c1 = sh.bins[2 * lane + 1];
                int incl = c0 + c1;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const int pre = incl - c0 - c1;
                int b = -1, g = 0, q = 0;
                if (pre < k && pre + c0 >= k) { b = 2 * lane; g = pre; q = c0; }
                else if (pre + c0 < k && incl >= k) { b = 2 * lane + 1; g = pre + c0; q = c1; }
                const unsigned hit = __ballot_sync(0xffffffffu, b >= 0);
                const int src = __ffs(hit) - 1;
                const int bt = __shfl_sync(0xffffffffu, b, src);
                const int nb = (c0 > 0 && 2 * lane > bt) ? 2 * lane
                             : (c1 > 0 && 2 * lane + 1 > bt) ? 2 * lane + 1 : 999;
                const int nbm = __reduce_min_sync(0xffffffffu, nb);
                if (lane == src) {
                    sh.thr = mx - b;
                    sh.gt = g;
                    sh.eq = q;
                    if (nbm < 999) sh.below = mx - nbm;  // a candidate lies below thr
                }
            }
            __syncthreads();
            thr = sh.thr;
            gt_tot = sh.gt;
            eq_tot = sh.eq;
        } else {
            int lo = L, hi = mx + 1;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                int c = 0;
                for (int i = tid; i < C; i += NT) c += (int)(sh.cand[i] >> 16) >= mid;
                if (block_sum(c) >= k) lo = mid; else hi = mid;
            }
            thr = lo;
            int g = 0, q = 0, bl = -1;
            for (int i = tid; i < C; i += NT) {
                const int key = (int)(sh.cand[i] >> 16);
                g += key > thr;
                q += key == thr;
                if (key < thr) bl = max(bl, key);
            }
            gt_tot = block_sum(g);
            eq_tot = block_sum(q);
            bl = __reduce_max_sync(0xffffffffu, bl);
            if (lane == 0) atomicMax(&sh.below, bl);
            __syncthreads();
        }
    } else {
        // ---- thr = max t with #(keys >= t) >= k ----
        int lo = L >= 0 ? L : mn, hi = mx + 1;
        if (L < 0 && hi - lo > 64) {
            // the full key range: two 8-bit radix rounds (select.py:87-115's scheme) instead of
            // ~16 bisection passes -- the high byte's bucket holding the k-th largest key, then
            // the low byte within it (shared-memory histograms, one warp scans 256 bins)
            auto radix_round = [&](int shift, int hi_byte, int rank) -> int {
                for (int i = tid; i < 256; i += NT) sh.hist[i] = 0;
                __syncthreads();
                for (int v = tid; v < nvec; v += NT) {
                    uint32_t w[4];
                    words(s4[v], w);
#pragma unroll
                    for (int e = 0; e < 8; e++) {
                        const int key = (e & 1) ? (int)(w[e >> 1] >> 16) : (int)(w[e >> 1] & 0xFFFFu);
                        if (v * 8 + e < P && (shift == 8 || (key >> 8) == hi_byte))
                            atomicAdd(&sh.hist[(key >> shift) & 0xFF], 1);
                    }
                }
                __syncthreads();
                if (warp == 0) {  // lane l: bins 255 - 8 l .. 248 - 8 l (descending key order)
                    int c8[8], sum = 0;
#pragma unroll
                    for (int j = 0; j < 8; j++) { c8[j] = sh.hist[255 - 8 * lane - j]; sum += c8[j]; }
                    int incl = sum;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    int cum = incl - sum, b = -1, before = 0;
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        if (b < 0 && cum + c8[j] >= rank) { b = 255 - 8 * lane - j; before = cum; }
                        cum += c8[j];
                    }
                    const unsigned hit = __ballot_sync(0xffffffffu, b >= 0);
                    const int src = __ffs(hit) - 1;
                    if (lane == src) { sh.thr = b; sh.gt = before; }
                }
                __syncthreads();
                return sh.thr;
            };
            const int hb = radix_round(8, 0, k);
            const int above = sh.gt;  // keys in higher buckets
            __syncthreads();
            const int lb = radix_round(0, hb, k - above);
            lo = (hb << 8) | lb;
            hi = lo + 1;
        }
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            const uint32_t m16 = (uint32_t)mid * 0x10001u;
            int c = 0;
            for (int v = tid; v < nvec; v += NT) c += count_ge(s4[v], v, m16);
            if (block_sum(c) >= k) lo = mid; else hi = mid;
        }
        thr = lo;
        const uint32_t t16 = (uint32_t)thr * 0x10001u;
        const uint32_t t1 = (uint32_t)(thr + 1) * 0x10001u;
        int g = 0, ge = 0, bl = -1;
        for (int v = tid; v < nvec; v += NT) {
            const uint4 x = s4[v];
            g += thr < 0xFFFF ? count_ge(x, v, t1) : 0;
            ge += count_ge(x, v, t16);
            uint32_t w[4], mk[4];
            words(x, w);
            vmask(v, mk);
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint32_t lt = ~__vcmpgeu2(w[q], t16) & mk[q];
                if (lt) {
                    const uint32_t z = w[q] & lt;
                    if (lt & 0xFFFFu) bl = max(bl, (int)(z & 0xFFFFu));
                    if (lt >> 16) bl = max(bl, (int)(z >> 16));
                }
            }
        }
        gt_tot = block_sum(g);
        eq_tot = block_sum(ge) - gt_tot;
        bl = block_max(bl);
        if (tid == 0) sh.below = bl;
        __syncthreads();
    }
    const int budget = k - gt_tot;  // in [1, eq_tot]
    stamp(2);
    if (C >= 0) {
        // ---- ordered compaction of the (logically ordered) candidates ----
        const int cs = (C + NT - 1) / NT;
        const int i0 = min(tid * cs, C), i1 = min(i0 + cs, C);
        int g = 0, q = 0;
        for (int i = i0; i < i1; i++) {
            const int key = (int)(sh.cand[i] >> 16);
            g += key > thr;
            q += key == thr;
        }
        int ig = g, iq = q;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int yg = __shfl_up_sync(0xffffffffu, ig, o);
            const int yq = __shfl_up_sync(0xffffffffu, iq, o);
            if (lane >= o) { ig += yg; iq += yq; }
        }
        __syncthreads();
        if (lane == 31) { sh.red[1][warp][0] = (uint32_t)ig; sh.red[1][warp][1] = (uint32_t)iq; }
        __syncthreads();
        int gb = ig - g, qb = iq - q;
#pragma unroll
        for (int w = 0; w < NWP; w++)
            if (w < warp) { gb += (int)sh.red[1][w][0]; qb += (int)sh.red[1][w][1]; }
        int pos = gb + min(qb, budget);
        int seen = qb;
        for (int i = i0; i < i1; i++) {
            const uint32_t c = sh.cand[i];
            const int key = (int)(c >> 16), idx = (int)(c & 0xFFFFu);
            bool sel = key > thr;
            if (key == thr) { sel = seen < budget; seen++; }
            if (sel) {
                if (slist) slist[pos] = idx;
                else { out[pos] = map[idx]; if (out_l) out_l[pos] = idx; }
                pos++;
            }
        }
    } else {
        // ---- ordered compaction over all keys: per round of 4 NT vectors, a block scan of
        // (keys > thr, keys == thr) gives each vector's output position and tie rank ----
        const uint32_t t16 = (uint32_t)thr * 0x10001u;
        const uint32_t t1 = (uint32_t)min(thr + 1, 0xFFFF) * 0x10001u;
        int run_g = 0, run_q = 0, par = 0;
        constexpr int VPT = 4;  // consecutive vectors per thread per round (one scan each)
        for (int v0 = 0; v0 < nvec; v0 += NT * VPT, par ^= 1) {
            const int vt = v0 + tid * VPT;
            uint4 x[VPT];
            int g = 0, q = 0;
#pragma unroll
            for (int j = 0; j < VPT; j++) {
                const int v = vt + j;
                x[j] = make_uint4(0u, 0u, 0u, 0u);
                if (v < nvec) {
                    x[j] = s4[v];
                    const int ge = count_ge(x[j], v, t16);
                    const int gj = thr < 0xFFFF ? count_ge(x[j], v, t1) : 0;
                    g += gj;
                    q += ge - gj;
                }
            }
            const int pk = g | (q << 16);
            int inc = pk;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) sh.red[par][warp][0] = (uint32_t)inc;
            __syncthreads();
            int pre = inc - pk;
            int tot = 0;
#pragma unroll
            for (int w = 0; w < NWP; w++) {
                const int t = (int)sh.red[par][w][0];
                if (w < warp) pre += t;
                tot += t;
            }
            if (g | q) {
                int gpos = run_g + (pre & 0xFFFF), seen = run_q + (pre >> 16);
                int pos = gpos + min(seen, budget);
#pragma unroll
                for (int j = 0; j < VPT; j++) {
                    const int v = vt + j;
                    if (v >= nvec) break;
                    uint32_t w[4];
                    words(x[j], w);
#pragma unroll
                    for (int e = 0; e < 8; e++) {
                        const int key = (e & 1) ? (int)(w[e >> 1] >> 16) : (int)(w[e >> 1] & 0xFFFFu);
                        if (v * 8 + e >= P || key < thr) continue;
                        bool sel = key > thr;
                        if (key == thr) { sel = seen < budget; seen++; }
                        if (sel) {
                            if (slist) slist[pos] = v * 8 + e;
                            else { out[pos] = map[v * 8 + e]; if (out_l) out_l[pos] = v * 8 + e; }
                            pos++;
                        }
                    }
                }
            }
            run_g += tot & 0xFFFF;
            run_q += tot >> 16;
        }
    }
    stamp(3);
    if (slist) {
        __syncthreads();
        for (int t = tid; t < k; t += NT) {
            const int li = slist[t];
            const int pid = __ldg(map + li);
            if (out) out[t] = pid;
            if (out_l) out_l[t] = li;
            if (slist_physical) slist[t] = pid;
        }
    }
    if (tid == 0) {
        *n_sel = k;
        *kth = thr;
        *kplus1 = (eq_tot > budget) ? thr : sh.below;
    }
    __syncthreads();
    return true;
}

// ---------------------------------------------------------------------------
// Warp-level selection (the warp-per-unit fused kernel: many short units, small k).
// One warp selects one unit whose P <= 256 * MAXV keys sit in registers (lane l holds the
// 16-byte key vectors l, l+32, ...).  Threshold = bisection over [min, max] with warp-wide
// counts (exact for any key distribution, ~log2(range) rounds); ordered compaction per key
// vector in logical order (ballot/scan ranks), ties by ascending logical index -- the
// reference's rule; logical ids land in `ids` (warp-private shared memory) and are translated
// to physical ids in one parallel round.  Same outputs as select_block.
// ---------------------------------------------------------------------------
// Bounded mode (pt_score_bounded's key intervals; keys_g = lower keys): hi_g = the upper keys
// and exact(p) = the exact key of logical page p.  Before selecting, the warp computes the
// bracket A = the (k+1)-th largest lower key, B = the k-th largest upper key and replaces the
// lower key of every page whose interval is not one key and meets [A, B] (every uncertain page
// when P <= k) by its exact key -- the same argument as select_cand's bounded mode: pages
// above B are selected and pages below A are below the (k+1)-th key whatever their exact keys.
struct NoExactKey {
    __device__ int operator()(int) const { return 0; }
};
struct NoPrefetch {
    __device__ void operator()(int) const {}
};

template <int MAXV, class ExactKey = NoExactKey, class PrefetchRow = NoPrefetch>
__device__ void select_warp(const uint16_t *__restrict__ keys_g, int P, int k,
                            const int32_t *__restrict__ map, int32_t *__restrict__ out,
                            int32_t *__restrict__ out_l, int32_t *__restrict__ n_sel,
                            int32_t *__restrict__ kth, int32_t *__restrict__ kplus1, int *ids,
                            const uint16_t *__restrict__ hi_g = nullptr,
                            const ExactKey &exact = ExactKey(), int *scratch = nullptr,
                            int scratch_cap = 0, const uint16_t *__restrict__ tmax_g = nullptr,
                            unsigned long long *tp = nullptr,
                            const PrefetchRow &prefetch = PrefetchRow()) {
    // tuning aid: %clock64 phase stamps tp[i] (lane 0)
    auto sw_stamp = [&](int i) {
        if (tp && (threadIdx.x & 31) == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %clock64;" : "=l"(t));
            tp[i] = t;
        }
    };
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const uint4 *k4 = reinterpret_cast<const uint4 *>(keys_g);
    uint4 v[MAXV];
#pragma unroll
    for (int j = 0; j < MAXV; j++) {
        const int base = (lane + 32 * j) * 8;
        v[j] = base < P ? __ldcg(k4 + lane + 32 * j) : make_uint4(0u, 0u, 0u, 0u);
    }
    // the scorer's per-32-page tile maxima (of the lower keys): Lt = the (k+1)-th largest is
    // a lower bound of the threshold, of the (k+1)-th largest key and (bounded) of A and B --
    // k + 1 distinct tiles each hold a page whose (lower) key reaches it -- so every bisection
    // below starts from [Lt, max] instead of [min, max] (up to 64 tiles: P <= 2048)
    const int ntl = (P + 31) >> 5;
    const bool use_tm = tmax_g != nullptr && P > k && ntl >= k + 1 && ntl <= 64;
    int tm0 = -1, tm1 = -1;
    if (use_tm) {
        if (lane < ntl) tm0 = (int)__ldcg(tmax_g + lane);
        if (lane + 32 < ntl) tm1 = (int)__ldcg(tmax_g + lane + 32);
    }
    auto keyof = [&](const uint4 &x, int e) -> int {
        const uint32_t w = e < 2 ? x.x : e < 4 ? x.y : e < 6 ? x.z : x.w;
        return (e & 1) ? (int)(w >> 16) : (int)(w & 0xFFFFu);
    };
    // keys past P read as 0 (below every real key: the ordered encoding of a finite or
    // infinite bf16 score is >= 0x7F), so the bisection counts below need no validity mask
    auto zero_tail = [&](uint4 (&a)[MAXV]) {
#pragma unroll
        for (int j = 0; j < MAXV; j++) {
            const int base = (lane + 32 * j) * 8;
            if (base < P && base + 8 > P) {
                const int nk = P - base;  // 1..7 valid keys
                uint32_t w[4] = {a[j].x, a[j].y, a[j].z, a[j].w};
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const uint32_t m = (2 * q < nk ? 0x0000FFFFu : 0u) | (2 * q + 1 < nk ? 0xFFFF0000u : 0u);
                    w[q] &= m;
                }
                a[j] = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
    };
    // #keys >= t in this lane's vectors (t >= 1), two u16 keys per SIMD compare
    auto cnt_ge = [&](const uint4 (&a)[MAXV], int t) -> int {
        const uint32_t t16 = (uint32_t)t * 0x10001u;
        int c = 0;
#pragma unroll
        for (int j = 0; j < MAXV; j++) {
            c += __popc(__vcmpgeu2(a[j].x, t16)) + __popc(__vcmpgeu2(a[j].y, t16)) +
                 __popc(__vcmpgeu2(a[j].z, t16)) + __popc(__vcmpgeu2(a[j].w, t16));
        }
        return c >> 4;
    };
    // min (over the non-zero = real keys) and max of this lane's keys, two per SIMD op
    auto minmax = [&](const uint4 (&a)[MAXV], int &mn_, int &mx_) {
        uint32_t lo = 0xFFFFFFFFu, hi = 0u;
#pragma unroll
        for (int j = 0; j < MAXV; j++) {
            const uint32_t w[4] = {a[j].x, a[j].y, a[j].z, a[j].w};
#pragma unroll
            for (int q = 0; q < 4; q++) {
                hi = __vmaxu2(hi, w[q]);
                lo = __vminu2(lo, w[q] | __vcmpeq2(w[q], 0u));
            }
        }
        mn_ = (int)min(lo & 0xFFFFu, lo >> 16);
        mx_ = (int)max(hi & 0xFFFFu, hi >> 16);
    };
    zero_tail(v);
    sw_stamp(6);
    int Lt = -1;
    if (use_tm) {
        int lo2 = __reduce_min_sync(0xffffffffu, (unsigned)(tm0 < 0 ? 0xFFFF : min(tm0, tm1 < 0 ? 0xFFFF : tm1)));
        int hi2 = __reduce_max_sync(0xffffffffu, (unsigned)max(max(tm0, tm1), 0)) + 1;
        while (hi2 - lo2 > 1) {
            const int mid = (lo2 + hi2) >> 1;
            const int c = __reduce_add_sync(0xffffffffu, (unsigned)((tm0 >= mid) + (tm1 >= mid)));
            if (c >= k + 1) lo2 = mid; else hi2 = mid;
        }
        Lt = lo2;
    }
    sw_stamp(7);
    int bracket_lo = -1, bracket_hi = -1;  // bounded: the threshold lies in [A, B]
    if (hi_g) {
        const uint4 *h4 = reinterpret_cast<const uint4 *>(hi_g);
        uint4 hv[MAXV];
#pragma unroll
        for (int j = 0; j < MAXV; j++) {
            const int base = (lane + 32 * j) * 8;
            hv[j] = base < P ? __ldcg(h4 + lane + 32 * j) : make_uint4(0u, 0u, 0u, 0u);
        }
        zero_tail(hv);
        // A = the (k+1)-th largest lower key, B = the k-th largest upper key: one bisection
        // pass per round counting both arrays against their own midpoints
        int amn, amx, bmn, bmx;
        minmax(v, amn, amx);
        minmax(hv, bmn, bmx);
        int alo = __reduce_min_sync(0xffffffffu, amn), ahi = __reduce_max_sync(0xffffffffu, amx) + 1;
        int blo = __reduce_min_sync(0xffffffffu, bmn), bhi = __reduce_max_sync(0xffffffffu, bmx) + 1;
        alo = max(alo, Lt);  // Lt <= A <= B (Lt < 0 without tile maxima)
        blo = max(blo, Lt);
        if (P > k) {
            while (ahi - alo > 1 || bhi - blo > 1) {
                const int am = (alo + ahi) >> 1, bm = (blo + bhi) >> 1;
                // am, bm >= 1: the zeroed keys past P are never counted
                const int ca = __reduce_add_sync(0xffffffffu, (unsigned)cnt_ge(v, max(am, 1)));
                const int cb = __reduce_add_sync(0xffffffffu, (unsigned)cnt_ge(hv, max(bm, 1)));
                if (ahi - alo > 1) { if (ca >= k + 1) alo = am; else ahi = am; }
                if (bhi - blo > 1) { if (cb >= k) blo = bm; else bhi = bm; }
            }
        }
        const int A = P > k ? alo : 0, B = P > k ? blo : 0xFFFF;
        bracket_lo = A;
        bracket_hi = B;
    sw_stamp(8);
        // the bracket pages, compacted (lane-major) into the warp's scratch list in rounds of
        // scratch_cap, resolved one lane per page, written back into the lower keys
        // bit 8 j + e: page (lane + 32 j) * 8 + e needs its exact key -- interval not one key
        // and meeting [A, B] (the zeroed keys past P have lo == hi); two keys per SIMD compare
        uint64_t fl = 0ull;
        const uint32_t A16 = (uint32_t)A * 0x10001u, B16 = (uint32_t)min(B, 0xFFFF) * 0x10001u;
#pragma unroll
        for (int j = 0; j < MAXV; j++) {
            const uint32_t lw[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
            const uint32_t hw[4] = {hv[j].x, hv[j].y, hv[j].z, hv[j].w};
            uint32_t m = 0u;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const uint32_t f = ~__vcmpeq2(lw[q], hw[q]) & __vcmpgeu2(hw[q], A16) & __vcmpleu2(lw[q], B16);
                m |= ((f & 1u) | ((f >> 15) & 2u)) << (2 * q);
            }
            fl |= (uint64_t)m << (8 * j);
        }
        const int nf = __popcll(fl);
        int incl = nf;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int first = incl - nf, total = __shfl_sync(0xffffffffu, incl, 31);
        for (int r0 = 0; r0 < total; r0 += scratch_cap) {
            int rk = first;
            uint64_t f = fl;
            while (f) {  // list this lane's bracket pages with ranks in [r0, r0 + cap)
                const int b = __ffsll((long long)f) - 1;
                f &= f - 1;
                if (rk >= r0 && rk < r0 + scratch_cap) scratch[rk - r0] = (lane + 32 * (b >> 3)) * 8 + (b & 7);
                rk++;
            }
            __syncwarp();
            const int nr = min(scratch_cap, total - r0);
            // every row of the round requested before the first (latency-bound) exact sum
            for (int i = lane; i < nr; i += 32) prefetch(scratch[i]);
            for (int i = lane; i < nr; i += 32) scratch[i] = exact(scratch[i]);
            __syncwarp();
            rk = first;
            f = fl;
            while (f) {
                const int b = __ffsll((long long)f) - 1;
                f &= f - 1;
                if (rk >= r0 && rk < r0 + scratch_cap) {
                    const uint32_t x = (uint32_t)scratch[rk - r0];
                    const int j = b >> 3, e = b & 7;
#pragma unroll
                    for (int jj = 0; jj < MAXV; jj++) {
                        if (jj != j) continue;
                        uint32_t w[4] = {v[jj].x, v[jj].y, v[jj].z, v[jj].w};
                        w[e >> 1] = (e & 1) ? ((w[e >> 1] & 0xFFFFu) | (x << 16)) : ((w[e >> 1] & 0xFFFF0000u) | x);
                        v[jj] = make_uint4(w[0], w[1], w[2], w[3]);
                    }
                }
                rk++;
            }
            __syncwarp();
        }
    }
    sw_stamp(9);
    int mn, mx;
    minmax(v, mn, mx);
    mn = __reduce_min_sync(0xffffffffu, mn);
    sw_stamp(11);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (P <= k) {  // _take_all (select.py:75-84)
        for (int i = lane; i < P; i += 32) {
            const int pid = __ldg(map + i);
            ids[i] = pid;
            if (out) out[i] = pid;
            if (out_l) out_l[i] = i;
        }
        if (lane == 0) { *n_sel = P; *kth = mn; *kplus1 = -1; }
        __syncwarp();
        return;
    }
    auto count_ge = [&](int t) -> int {
        return __reduce_add_sync(0xffffffffu, (unsigned)cnt_ge(v, max(t, 1)));
    };
    // thr = max t with #(keys >= t) >= k (bounded: within the bracket [A, B])
    int lo = max(mn, Lt), hi = mx + 1;  // Lt <= thr
    if (bracket_lo >= 0) { lo = max(lo, bracket_lo); hi = min(hi, bracket_hi + 1); }
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (count_ge(mid) >= k) lo = mid; else hi = mid;
    }
    const int thr = lo;
    sw_stamp(12);
    // counts and the ordered compaction on u16x2 SIMD compares (the keys past P are 0: never
    // > or == thr, and below 0 means no key below thr); short loops, not per-key unrolled code
    // -- this runs once per warp, so its instruction footprint is its cost
    const uint32_t t16 = (uint32_t)thr * 0x10001u;
    auto pack2 = [](uint32_t m) -> uint32_t { return (m & 1u) | ((m >> 15) & 2u); };
    int gt = 0, eq = 0, below = -1;
    {
        uint32_t blw = 0u;
#pragma unroll
        for (int j = 0; j < MAXV; j++) {
            const uint32_t w[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
            for (int q = 0; q < 4; q++) {
                gt += __popc(__vcmpgtu2(w[q], t16));
                eq += __popc(__vcmpeq2(w[q], t16));
                blw = __vmaxu2(blw, w[q] & ~__vcmpgeu2(w[q], t16));
            }
        }
        gt >>= 4;
        eq >>= 4;
        const int b = (int)max(blw & 0xFFFFu, blw >> 16);
        below = b > 0 ? b : -1;
    }
    const int gt_tot = __reduce_add_sync(0xffffffffu, gt);
    const int eq_tot = __reduce_add_sync(0xffffffffu, eq);
    below = (int)__reduce_max_sync(0xffffffffu, (unsigned)(below + 1)) - 1;
    const int budget = k - gt_tot;
    sw_stamp(13);
    // ordered compaction in one sweep: per (lane, vector j) 8-bit masks of the keys > thr and
    // == thr; the ties a vector may take and every vector's output offset come from warp scans
    // of per-j counts packed in 16-bit fields (4 vectors per 64-bit word) -- a handful of
    // shuffles for all j instead of two dependent scans per j
    static_assert(MAXV <= 8, "packed per-vector counts");
    uint64_t gmp = 0ull, emp = 0ull;   // byte j: the vector's > / == masks
    uint64_t ec[2] = {0ull, 0ull};     // 16-bit field j: #(== thr) in vector j
#pragma unroll
    for (int j = 0; j < MAXV; j++) {
        const uint32_t w[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
        uint32_t gm = 0u, em = 0u;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            gm |= pack2(__vcmpgtu2(w[q], t16)) << (2 * q);
            em |= pack2(__vcmpeq2(w[q], t16)) << (2 * q);
        }
        gmp |= (uint64_t)gm << (8 * j);
        emp |= (uint64_t)em << (8 * j);
        ec[j >> 2] |= (uint64_t)__popc(em) << (16 * (j & 3));
    }
    auto scan64 = [&](uint64_t x) -> uint64_t {  // inclusive, field-wise (no field overflows)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        return x;
    };
    auto f16 = [](uint64_t x, int j) -> int { return (int)((x >> (16 * (j & 3))) & 0xFFFFull); };
    uint64_t sc[2] = {0ull, 0ull};  // 16-bit field j: keys this vector selects
    uint64_t keepp = 0ull;          // byte j: the ties vector j takes
    {
        const uint64_t ei0 = scan64(ec[0]), ei1 = scan64(ec[1]);
        const uint64_t et0 = __shfl_sync(0xffffffffu, ei0, 31), et1 = __shfl_sync(0xffffffffu, ei1, 31);
        int before_j = 0;  // ties in vectors j' < j over all lanes
#pragma unroll
        for (int j = 0; j < MAXV; j++) {
            const uint64_t inc = j < 4 ? ei0 : ei1, tot = j < 4 ? et0 : et1, own = ec[j >> 2];
            const int mine = f16(own, j);
            const int before = before_j + f16(inc, j) - mine;
            int allow = min(max(budget - before, 0), mine);
            uint32_t e2 = (uint32_t)((emp >> (8 * j)) & 0xFFu), keep = 0u;
            for (; allow > 0; allow--) {
                keep |= e2 & (0u - e2);
                e2 &= e2 - 1u;
            }
            keepp |= (uint64_t)keep << (8 * j);
            const int cnt = __popc((uint32_t)((gmp >> (8 * j)) & 0xFFu)) + __popc(keep);
            sc[j >> 2] |= (uint64_t)cnt << (16 * (j & 3));
            before_j += f16(tot, j);
        }
    }
    {
        const uint64_t si0 = scan64(sc[0]), si1 = scan64(sc[1]);
        const uint64_t st0 = __shfl_sync(0xffffffffu, si0, 31), st1 = __shfl_sync(0xffffffffu, si1, 31);
        int base_j = 0;  // selected keys in vectors j' < j over all lanes
#pragma unroll
        for (int j = 0; j < MAXV; j++) {
            const uint64_t inc = j < 4 ? si0 : si1, tot = j < 4 ? st0 : st1, own = sc[j >> 2];
            uint32_t m = (uint32_t)(((gmp | keepp) >> (8 * j)) & 0xFFu);
            int pos = base_j + f16(inc, j) - f16(own, j);
            const int base = (lane + 32 * j) * 8;
            for (; m; m &= m - 1u) ids[pos++] = base + __ffs(m) - 1;
            base_j += f16(tot, j);
        }
    }
    (void)lt;
    sw_stamp(14);
    __syncwarp();
    for (int t = lane; t < k; t += 32) {
        const int li = ids[t];
        const int pid = __ldg(map + li);
        ids[t] = pid;
        if (out) out[t] = pid;
        if (out_l) out_l[t] = li;
    }
    if (lane == 0) {
        *n_sel = k;
        *kth = thr;
        *kplus1 = (eq_tot > budget) ? thr : below;
    }
    __syncwarp();
}

}  // namespace pt
