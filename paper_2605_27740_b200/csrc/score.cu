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
#include "common.cuh"

namespace pt {

constexpr int kScoreThreads = 256;
constexpr int kScoreMaxD = 512;

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
template <int QDT, int SDT, int G>
__global__ void __launch_bounds__(kScoreThreads)
    k_score(const void *__restrict__ q, const float *__restrict__ norms_in,
            const void *__restrict__ means, const float *__restrict__ stds,
            const int32_t *__restrict__ seq_len, int D, int S, int Pmax, float lam,
            uint16_t *__restrict__ keys, float *__restrict__ scores) {
    constexpr int V = MeanVec<SDT>::V;
    constexpr bool kExactProduct = (QDT == PT_BF16 && SDT == PT_BF16);
    __shared__ __align__(16) float qs[G][kScoreMaxD];
    __shared__ float lam_norm[G];
    const int64_t u = blockIdx.y;
    const int tid = threadIdx.x;
    const int n = seq_len[u];
    const int P = (n + S - 1) / S;
    const int64_t p0 = (int64_t)blockIdx.x * kScoreThreads;
    if (p0 >= P) return;

    for (int i = tid; i < G * D; i += kScoreThreads) {
        const int g = i / D, d = i % D;
        const float v = load_elem<QDT>(q, (u * G + g) * (int64_t)D + d);
        qs[g][d] = v;
    }
    __syncthreads();
    if (tid < G) {
        const float nrm = norms_in ? norms_in[u * G + tid]
                                   : __double2float_rn(__dsqrt_rn(np_sum(SquaresOfF32{qs[tid]}, D)));
        lam_norm[tid] = __fmul_rn(lam, nrm);
    }
    __syncthreads();

    const int64_t p = p0 + tid;
    if (p >= P) return;
    const char *mp = static_cast<const char *>(means) +
                     ((u * Pmax * D + (p >> 5) * 32 * (int64_t)D + (p & 31) * V) *
                      (SDT == PT_F32 ? 4 : 2));
    const int64_t chunk_stride = 32 * V * (SDT == PT_F32 ? 4 : 2);  // bytes between d-chunks
    float acc[G];
#pragma unroll
    for (int g = 0; g < G; g++) acc[g] = 0.0f;
    const int nchunk = D / V;
#pragma unroll 8
    for (int c = 0; c < nchunk; c++) {
        float m[V];
        MeanVec<SDT>::load(mp + c * chunk_stride, m);
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

template <int QDT, int SDT>
static int launch_score(const void *q, const float *norms, const void *means, const float *stds,
                        const int32_t *seq_len, int U, int G, int D, int S, int Pmax, float lam,
                        uint16_t *keys, float *scores, cudaStream_t st) {
    dim3 grid((Pmax + kScoreThreads - 1) / kScoreThreads, U);
#define PT_SCORE_CASE(G_)                                                                      \
    case G_:                                                                                   \
        k_score<QDT, SDT, G_><<<grid, kScoreThreads, 0, st>>>(q, norms, means, stds, seq_len, D, \
                                                              S, Pmax, lam, keys, scores);     \
        break;
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

extern "C" int pt_score(const void *q, int q_dtype, const float *norms, const void *means,
                        int stats_dtype, const float *stds, const int32_t *seq_len, int U, int G,
                        int D, int S, int Pmax, float lam, uint16_t *keys, float *scores,
                        void *stream) {
    if (!q || !means || !stds || !seq_len || !keys || U < 0 || S < 1 || Pmax % 32 || G < 1)
        return PT_ERR_INVALID;
    const int V = stats_dtype == PT_F32 ? 4 : 8;
    if (D < 1 || D > kScoreMaxD || D % V) return PT_ERR_UNSUPPORTED;
    if (U == 0) return PT_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (q_dtype == PT_F32 && stats_dtype == PT_F32)
        return launch_score<PT_F32, PT_F32>(q, norms, means, stds, seq_len, U, G, D, S, Pmax, lam, keys, scores, st);
    if (q_dtype == PT_BF16 && stats_dtype == PT_F32)
        return launch_score<PT_BF16, PT_F32>(q, norms, means, stds, seq_len, U, G, D, S, Pmax, lam, keys, scores, st);
    if (q_dtype == PT_BF16 && stats_dtype == PT_BF16)
        return launch_score<PT_BF16, PT_BF16>(q, norms, means, stds, seq_len, U, G, D, S, Pmax, lam, keys, scores, st);
    if (q_dtype == PT_F32 && stats_dtype == PT_BF16)
        return launch_score<PT_F32, PT_BF16>(q, norms, means, stds, seq_len, U, G, D, S, Pmax, lam, keys, scores, st);
    return PT_ERR_INVALID;
}

extern "C" int pt_tile_means(const float *src, int U, int P, int D, int Pmax, void *dst,
                             int stats_dtype, void *stream) {
    if (!src || !dst || U < 0 || P < 0 || P > Pmax || Pmax % 32) return PT_ERR_INVALID;
    if ((int64_t)U * P * D == 0) return PT_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int64_t total = (int64_t)U * P * D;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (stats_dtype == PT_F32) k_tile_means<PT_F32><<<blocks, 256, 0, st>>>(src, U, P, D, Pmax, dst);
    else if (stats_dtype == PT_BF16) k_tile_means<PT_BF16><<<blocks, 256, 0, st>>>(src, U, P, D, Pmax, dst);
    else return PT_ERR_INVALID;
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}
