// common.cuh -- shared device helpers for the pagetopk B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pagetopk_b200.h"

namespace pt {

// ---------------------------------------------------------------------------
// element access: the KV pool and the page means are bf16 or f32
// ---------------------------------------------------------------------------
__device__ __forceinline__ float bf16_bits_to_f32(uint32_t b) { return __uint_as_float(b << 16); }
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

template <int DT>
__device__ __forceinline__ float load_elem(const void *base, int64_t i) {
    if constexpr (DT == PT_F32) {
        return static_cast<const float *>(base)[i];
    } else {
        return bf16_bits_to_f32(static_cast<const uint16_t *>(base)[i]);
    }
}

// Stage n contiguous elements (rows of length D) from global memory into shared f32 with
// row stride ld, widening bf16.  Each thread issues up to MAXC 16-byte loads before its
// first shared store, so a thread's share arrives in one memory round instead of one round
// per loop iteration (the compiler does not hoist loads across the stores of a runtime-trip
// loop).  Falls back to element loads when rows are not 16-byte multiples.
template <int DT, int MAXC>
__device__ __forceinline__ void stage_rows_f32(float *dst, int ld, const void *src, int n, int D,
                                               int t, int nt) {
    constexpr int ES = DT == PT_F32 ? 4 : 2;
    constexpr int EPC = 16 / ES;
    if ((D * ES) % 16 != 0 || (reinterpret_cast<uintptr_t>(src) & 15) != 0) {
        for (int i = t; i < n; i += nt) dst[(i / D) * ld + (i % D)] = load_elem<DT>(src, i);
        return;
    }
    const int C = n / EPC;
    const uint4 *s4 = static_cast<const uint4 *>(src);
    for (int c0 = t; c0 < C; c0 += MAXC * nt) {
        uint4 v[MAXC];
#pragma unroll
        for (int j = 0; j < MAXC; j++) {
            const int c = c0 + j * nt;
            if (c < C) v[j] = __ldg(s4 + c);
        }
#pragma unroll
        for (int j = 0; j < MAXC; j++) {
            const int c = c0 + j * nt;
            if (c >= C) break;
            const int e = c * EPC, r = e / D, col = e - r * D;
            float *o = dst + r * ld + col;
            if constexpr (DT == PT_F32) {
                o[0] = __uint_as_float(v[j].x); o[1] = __uint_as_float(v[j].y);
                o[2] = __uint_as_float(v[j].z); o[3] = __uint_as_float(v[j].w);
            } else {
                const uint32_t w[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    o[2 * q] = __uint_as_float(w[q] << 16);
                    o[2 * q + 1] = __uint_as_float(w[q] & 0xFFFF0000u);
                }
            }
        }
    }
}

// bf16.py:18-33 -- round to nearest even, NaN quieted (identical to __float2bfloat16_rn
// for non-NaN inputs; written out so the NaN payload rule matches the reference).
__device__ __forceinline__ uint16_t f32_to_bf16_rne(float x) {
    uint32_t b = __float_as_uint(x);
    if (x != x) return (uint16_t)((b >> 16) | 0x0040u);
    return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}

// select.py:51-57 -- order-preserving key of a bf16 pattern
__device__ __forceinline__ uint16_t encode_ordered(uint16_t b) {
    return (b & 0x8000u) ? (uint16_t)~b : (uint16_t)(b | 0x8000u);
}

template <int DT>
__device__ __forceinline__ void store_elem(void *base, int64_t i, float v) {
    if constexpr (DT == PT_F32) {
        static_cast<float *>(base)[i] = v;
    } else {
        static_cast<uint16_t *>(base)[i] = f32_to_bf16_rne(v);
    }
}

// Means are kept in a page-interleaved tile layout so that one thread can walk one
// page's mean vector in the reference's sequential d order while every warp-wide
// load is a contiguous 512-byte, 128-bit-per-lane access:
//   means[u][p / 32][d / V][p % 32][d % V],  V = 16 bytes / sizeof(elem)
// Pmax is a multiple of 32.
template <int DT>
struct StatsTile {
    static constexpr int V = DT == PT_F32 ? 4 : 8;
};

__host__ __device__ __forceinline__ int64_t mean_offset(int64_t u, int64_t p, int d, int D,
                                                        int64_t Pmax, int V) {
    return u * Pmax * D + (p >> 5) * 32 * D + (int64_t)(d / V) * 32 * V + (p & 31) * V + (d % V);
}

// ---------------------------------------------------------------------------
// async bulk copy (TMA 1-D) + mbarrier helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// global -> shared bulk copy, completion counted on an mbarrier (SASS: UBLKCP)
// L2 evict-first policy for data read exactly once per step (the page means): keeps the
// step's small re-read outputs (keys, tile maxima, page tables) resident in L2
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_evict_normal_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void *smem_dst, const void *gmem_src, uint32_t bytes,
                                              uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *smem_dst, const void *gmem_src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// numpy pairwise_sum over n float64 values x(0..n-1), run by ONE thread
// (numpy/_core/src/umath/loops_utils.h.src; a 1-D np.sum is 0.0 + pairwise(x, n),
// identity-initialised -- pinned against numpy in tests/test_oracle_golden.py).
// X is any accessor `double operator()(int i)`.
template <class X>
__device__ __noinline__ double np_pairwise_leaf(const X &x, int off, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; i++) res = __dadd_rn(res, x(off + i));
        return res;
    }
    double r[8];
    int i;
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = x(off + j);
    for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], x(off + i + j));
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; i++) res = __dadd_rn(res, x(off + i));
    return res;
}

template <int DEPTH, class X>
__device__ __noinline__ double np_pairwise(const X &x, int off, int n) {
    if constexpr (DEPTH == 0) {
        return np_pairwise_leaf(x, off, n);  // caller guarantees n <= 128 * 2^DEPTH
    } else {
        if (n <= 128) return np_pairwise_leaf(x, off, n);
        int n2 = n / 2;
        n2 -= n2 % 8;
        return __dadd_rn(np_pairwise<DEPTH - 1>(x, off, n2),
                         np_pairwise<DEPTH - 1>(x, off + n2, n - n2));
    }
}

// np.sum of n <= 2048 float64 values
template <class X>
__device__ __forceinline__ double np_sum(const X &x, int n) {
    return __dadd_rn(0.0, np_pairwise<4>(x, 0, n));
}

struct DoubleArray {
    const double *a;
    __device__ __forceinline__ double operator()(int i) const { return a[i]; }
};
// np.sum of n float64 values in shared memory, by a whole warp (result valid in lane 0):
// numpy's leaf keeps 8 running sums r[j] over x[j], x[j+8], ...; here lane j (and lane 8 + j
// for the second half when n > 128 splits once) runs r[j], and the fixed combine tree
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) is done by shuffles -- the same operations in the
// same order as np_sum.  Other n (not a multiple of 8, or > 256) take the one-thread np_sum.
__device__ __forceinline__ double np_sum_warp(const double *x, int n, int lane) {
    if (n % 8 != 0 || n > 256 || n < 8) {
        double v = 0.0;
        if (lane == 0) v = np_sum(DoubleArray{x}, n);
        return v;
    }
    int off = 0, len = n;
    if (n > 128) {
        int n2 = n / 2;
        n2 -= n2 % 8;
        if (lane < 8) len = n2; else { off = n2; len = n - n2; }
    }
    const int j = lane & 7;
    double r = 0.0;
    if (lane < 16) {
        r = x[off + j];
        for (int i = 8; i < len; i += 8) r = __dadd_rn(r, x[off + i + j]);
    }
    const double a = __dadd_rn(r, __shfl_down_sync(0xffffffffu, r, 1));  // lanes 0,2,4,6: r0+r1, ...
    const double b = __dadd_rn(a, __shfl_down_sync(0xffffffffu, a, 2));  // lanes 0,4
    const double c = __dadd_rn(b, __shfl_down_sync(0xffffffffu, b, 4));  // lane 0 (and 8)
    const double hi = __shfl_down_sync(0xffffffffu, c, 8);
    return __dadd_rn(0.0, n > 128 ? __dadd_rn(c, hi) : c);
}

// ---------------------------------------------------------------------------
// bf16 mirror of the f32 page means (bounded scoring).
// Every stats writer that is given a mirror also stores m~ = bf16_rne(m) (tile layout,
// V = 8) and err_p = ||m~ - m|| + kMirrorAccSlack(D) * (||m|| + ||m~||), rounded up.  Then for
// any query q: |dot_ref(q, m) - dot_mirror(q, m~)| <= ||q|| * err_p, where dot_ref is the
// reference's sequential f32 dot (error <= gamma_D ||q|| ||m||) and dot_mirror is the
// scorer's bf16 x bf16 tensor-core dot (exact products, f32 accumulation; its accumulation
// error is bounded with 64x the RN gamma_D -- tests/test_gpu_bounded.py measures it).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ double mirror_acc_slack(int D) { return (double)(D + 2) * 0x1p-18; }

// The mirror block (one caller allocation of pt_mirror_bytes(U, Pmax, D) bytes):
//   tiles: bf16 means in the page-interleaved layout (V = 8)  [U][Pmax/32][D/8][32][8]
//   rows : the same f32 means row-major (one 4D-byte row per page: the selection's resolve
//          step fetches a page's exact mean with ONE bulk copy)  [U][Pmax][D]
//   err  : the per-page error bound                                [U][Pmax]
struct MirrorView {
    uint16_t *tiles;
    float *rows;
    float *err;
};
__host__ __device__ __forceinline__ size_t mirror_align(size_t x) { return (x + 255) & ~(size_t)255; }
__host__ __device__ __forceinline__ size_t mirror_bytes(int U, int Pmax, int D) {
    const size_t n = (size_t)U * Pmax;
    return mirror_align(n * D * 2) + mirror_align(n * D * 4) + n * 4;
}
__host__ __device__ __forceinline__ MirrorView mirror_view(const void *base, int U, int Pmax, int D) {
    MirrorView v{nullptr, nullptr, nullptr};
    if (!base) return v;
    char *b = static_cast<char *>(const_cast<void *>(base));
    const size_t n = (size_t)U * Pmax;
    v.tiles = reinterpret_cast<uint16_t *>(b);
    v.rows = reinterpret_cast<float *>(b + mirror_align(n * D * 2));
    v.err = reinterpret_cast<float *>(b + mirror_align(n * D * 2) + mirror_align(n * D * 4));
    return v;
}

template <int DJ>
__device__ __forceinline__ void store_mirror(const double (&mean)[DJ], int D, int64_t u, int64_t p,
                                             int64_t Pmax, const MirrorView &mv, int lane) {
    double dd = 0.0, mm = 0.0, tt = 0.0;
#pragma unroll
    for (int j = 0; j < DJ; j++) {
        const int d = lane + 32 * j;
        if (d < D) {
            const float m = __double2float_rn(mean[j]);
            const uint16_t b = f32_to_bf16_rne(m);
            const double mt = (double)bf16_bits_to_f32(b), m64 = (double)m;
            mv.tiles[mean_offset(u, p, d, D, Pmax, 8)] = b;
            mv.rows[(u * Pmax + p) * D + d] = m;
            const double e = mt - m64;  // exact: m~ and m are f32 within a factor 2
            dd = fma(e, e, dd);
            mm = fma(m64, m64, mm);
            tt = fma(mt, mt, tt);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dd += __shfl_xor_sync(0xffffffffu, dd, o);
        mm += __shfl_xor_sync(0xffffffffu, mm, o);
        tt += __shfl_xor_sync(0xffffffffu, tt, o);
    }
    if (lane == 0) {
        // f64 rounding of the sums / roots: relative 1e-14, covered by the (1 + 2^-30) factor;
        // the absolute term covers subnormal products
        const double e = (sqrt(dd) + mirror_acc_slack(D) * (sqrt(mm) + sqrt(tt))) * (1.0 + 0x1p-30) + 0x1p-120;
        mv.err[u * Pmax + p] = __double2float_ru(e);
    }
}

// squares of f32 values widened to f64: np.sum(f64(q)**2) (scoring.py:45)
struct SquaresOfF32 {
    const float *a;
    __device__ __forceinline__ double operator()(int i) const {
        const double v = (double)a[i];
        return __dmul_rn(v, v);
    }
};

}  // namespace pt

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL): the decode-step kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization so kernel N+1 is dispatched while
// kernel N drains (its CTAs are scheduled as SM resources free up and block in
// griddepcontrol.wait until N has completed and its writes are visible).  Every step
// kernel triggers its dependents first thing and waits before touching global memory, so
// only launch latency and on-chip set-up overlap -- no data race is possible.  A kernel
// launched without the attribute treats both instructions as no-ops.  PT_NO_PDL=1 turns
// the attribute off.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pt_pdl_enabled();  // capi.cu: false when PT_NO_PDL=1
int pt_num_sms();       // capi.cu: SM count of the current device (cached per device)

template <typename... KArgs, typename... Args>
static inline cudaError_t pt_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                    cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pt_pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

#define PT_CUDA_TRY(expr)                                                  \
    do {                                                                   \
        cudaError_t _e = (expr);                                           \
        if (_e != cudaSuccess) return PT_ERR_CUDA_BASE + (int)_e;          \
    } while (0)
