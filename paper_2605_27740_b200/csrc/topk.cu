// topk.cu -- K3: per-unit top-k page selection over ordered u16 score keys.
//
// Restates select.py:87-115 radix_topk with _kernels_cy.pyx:46-126 radix_select_desc:
//   pass 1  256-bin histogram of the high byte; hi = bucket holding the k-th largest
//   pass 2  256-bin histogram of the low byte inside bucket hi; lo likewise;
//           threshold = hi<<8 | lo, tie_budget = need - above2
//   pass 3  keys > threshold, plus the first tie_budget keys == threshold in ASCENDING
//           LOGICAL INDEX (the reference's tie rule), found with a
//           block-wide ordered compaction (exclusive scans over per-thread segments)
//   kplus1 = threshold if ties are left over, else the max key below the threshold
//   P <= k -> every page (select.py:100-101, _take_all :75-84), kth = min key.
// The logical->physical translation (select.py:108-110) happens in the epilogue.
// Integer work: the result is bit-identical to the reference (ids as a set; emitted in
// ascending logical order).
//
// One CTA per unit; the unit's keys are staged once in shared memory (<= ~200 KB,
// i.e. P <= ~100K pages); histograms use warp-aggregated shared atomics
// (__match_any_sync) because scores cluster in very few buckets.
#include "common.cuh"

namespace pt {

constexpr int kTopkThreads = 512;
constexpr int kTopkWarps = kTopkThreads / 32;

struct TopkShared {
    int hist[256];
    int warp_a[kTopkWarps];
    int warp_b[kTopkWarps];
    int bcast[8];
};

// block-wide exclusive scan of two counters; returns totals via out params
__device__ __forceinline__ void block_exscan2(int a, int b, int &ea, int &eb, int &ta, int &tb,
                                              TopkShared &sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int ia = a, ib = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int xa = __shfl_up_sync(0xffffffffu, ia, o);
        int xb = __shfl_up_sync(0xffffffffu, ib, o);
        if (lane >= o) { ia += xa; ib += xb; }
    }
    if (lane == 31) { sh.warp_a[warp] = ia; sh.warp_b[warp] = ib; }
    __syncthreads();
    int pa = 0, pb = 0, sa = 0, sb = 0;
#pragma unroll
    for (int w = 0; w < kTopkWarps; w++) {
        const int wa = sh.warp_a[w], wb = sh.warp_b[w];
        if (w < warp) { pa += wa; pb += wb; }
        sa += wa;
        sb += wb;
    }
    ea = pa + ia - a;
    eb = pb + ib - b;
    ta = sa;
    tb = sb;
    __syncthreads();
}

// Find, scanning buckets from 255 down, the first bucket b where the cumulative count
// (of buckets >= b) reaches `need`; returns b and the count strictly above it.
__device__ __forceinline__ void find_bucket(const int *hist, int need, int &bucket, int &above,
                                            TopkShared &sh) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // threads 0..255 hold buckets in DESCENDING order: t -> bucket 255 - t
    int c = tid < 256 ? hist[255 - tid] : 0;
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int x = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += x;
    }
    if (lane == 31) sh.warp_a[warp] = inc;
    __syncthreads();
    int pre = 0;
    for (int w = 0; w < warp; w++) pre += sh.warp_a[w];
    inc += pre;
    if (tid < 256) {
        const int exc = inc - c;
        if (inc >= need && exc < need) {  // unique crossing point
            sh.bcast[0] = 255 - tid;
            sh.bcast[1] = exc;
        }
    }
    __syncthreads();
    bucket = sh.bcast[0];
    above = sh.bcast[1];
    __syncthreads();
}

__device__ __forceinline__ void hist_add(int *hist, int bin, bool valid) {
    // warp-aggregated shared-memory histogram update
    const unsigned active = __ballot_sync(0xffffffffu, valid);
    if (valid) {
        const unsigned peers = __match_any_sync(active, bin);
        const int leader = __ffs(peers) - 1;
        if ((threadIdx.x & 31) == leader) atomicAdd(&hist[bin], __popc(peers));
    }
}

__global__ void __launch_bounds__(kTopkThreads)
    k_topk(const uint16_t *__restrict__ keys_g, const int32_t *__restrict__ seq_len,
           const int32_t *__restrict__ page_table, int S, int Pmax, int k,
           int32_t *__restrict__ sel, int32_t *__restrict__ sel_logical,
           int32_t *__restrict__ n_sel, int32_t *__restrict__ kth, int32_t *__restrict__ kplus1) {
    extern __shared__ __align__(16) uint16_t skeys[];
    __shared__ TopkShared sh;
    const int64_t u = blockIdx.x;
    const int tid = threadIdx.x;
    const int n = seq_len[u];
    const int P = (n + S - 1) / S;
    const int32_t *map = page_table + u * Pmax;
    int32_t *out = sel + u * (int64_t)k;
    int32_t *out_l = sel_logical ? sel_logical + u * (int64_t)k : nullptr;
    if (P == 0) {
        if (tid == 0) { n_sel[u] = 0; kth[u] = 0; kplus1[u] = -1; }
        return;
    }
    // stage keys (row base is 64-byte aligned since Pmax % 32 == 0)
    const uint16_t *src = keys_g + u * (int64_t)Pmax;
    const int nvec = (P + 7) / 8;
    for (int i = tid; i < nvec; i += kTopkThreads)
        reinterpret_cast<uint4 *>(skeys)[i] = __ldg(reinterpret_cast<const uint4 *>(src) + i);
    for (int i = tid; i < 256; i += kTopkThreads) sh.hist[i] = 0;
    __syncthreads();

    if (P <= k) {  // _take_all
        int mn = 0xFFFF;
        for (int i = tid; i < P; i += kTopkThreads) {
            out[i] = map[i];
            if (out_l) out_l[i] = i;
            mn = min(mn, (int)skeys[i]);
        }
        mn = __reduce_min_sync(0xffffffffu, mn);
        if ((tid & 31) == 0) sh.warp_a[tid >> 5] = mn;
        __syncthreads();
        if (tid == 0) {
            int m = 0xFFFF;
            for (int w = 0; w < kTopkWarps; w++) m = min(m, sh.warp_a[w]);
            n_sel[u] = P;
            kth[u] = m;
            kplus1[u] = -1;
        }
        return;
    }

    // pass 1: high-byte histogram
    for (int base = 0; base < P; base += kTopkThreads) {
        const int i = base + tid;
        const bool v = i < P;
        hist_add(sh.hist, v ? (skeys[i] >> 8) : 0, v);
    }
    __syncthreads();
    int hi, above;
    find_bucket(sh.hist, k, hi, above, sh);
    const int need = k - above;
    for (int i = tid; i < 256; i += kTopkThreads) sh.hist[i] = 0;
    __syncthreads();
    // pass 2: low-byte histogram inside bucket hi
    for (int base = 0; base < P; base += kTopkThreads) {
        const int i = base + tid;
        const bool v = i < P && (skeys[i] >> 8) == hi;
        hist_add(sh.hist, v ? (skeys[i] & 0xFF) : 0, v);
    }
    __syncthreads();
    int lo, above2;
    find_bucket(sh.hist, need, lo, above2, sh);
    const int tie_budget = need - above2;
    const int leftover = sh.hist[lo] - tie_budget;
    const int thr = (hi << 8) | lo;

    // pass 3: ordered compaction over contiguous per-thread segments
    const int seg = (((P + kTopkThreads - 1) / kTopkThreads) + 7) & ~7;
    const int b0 = min(tid * seg, P), b1 = min(b0 + seg, P);
    int gt = 0, eq = 0, below_max = -1;
    for (int i = b0; i < b1; i++) {
        const int key = skeys[i];
        gt += key > thr;
        eq += key == thr;
        if (key < thr) below_max = max(below_max, key);
    }
    int eq_before, dummy_e, eq_tot, dummy_t;
    block_exscan2(eq, 0, eq_before, dummy_e, eq_tot, dummy_t, sh);
    const int take = max(0, min(eq, tie_budget - eq_before));
    int pos, dummy2, tot_sel, dummy3;
    block_exscan2(gt + take, 0, pos, dummy2, tot_sel, dummy3, sh);
    int taken = 0;
    for (int i = b0; i < b1; i++) {
        const int key = skeys[i];
        bool s = key > thr;
        if (key == thr && taken < take) { s = true; taken++; }
        if (s) {
            out[pos] = map[i];
            if (out_l) out_l[pos] = i;
            pos++;
        }
    }
    // kplus1: max key strictly below the threshold
    below_max = __reduce_max_sync(0xffffffffu, below_max);
    if ((tid & 31) == 0) sh.warp_a[tid >> 5] = below_max;
    __syncthreads();
    if (tid == 0) {
        int m = -1;
        for (int w = 0; w < kTopkWarps; w++) m = max(m, sh.warp_a[w]);
        n_sel[u] = k;
        kth[u] = thr;
        kplus1[u] = leftover > 0 ? thr : m;
    }
}

}  // namespace pt

using namespace pt;

static size_t topk_smem_bytes(int Pmax) { return (size_t)((Pmax + 7) / 8) * 16; }

extern "C" int pt_topk(const uint16_t *keys, const int32_t *seq_len, const int32_t *page_table,
                       int U, int S, int Pmax, int k, int32_t *sel, int32_t *sel_logical,
                       int32_t *n_sel, int32_t *kth, int32_t *kplus1, void *stream) {
    if (!keys || !seq_len || !page_table || !sel || !n_sel || !kth || !kplus1 || U < 0 || S < 1 ||
        Pmax % 32)
        return PT_ERR_INVALID;
    if (k < 1) return PT_ERR_K;
    if (U == 0) return PT_OK;
    const size_t smem = topk_smem_bytes(Pmax);
    if (smem > 200 * 1024) return PT_ERR_UNSUPPORTED;
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        PT_CUDA_TRY(cudaFuncSetAttribute(k_topk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    k_topk<<<U, kTopkThreads, smem, (cudaStream_t)stream>>>(keys, seq_len, page_table, S, Pmax, k, sel,
                                                           sel_logical, n_sel, kth, kplus1);
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}
