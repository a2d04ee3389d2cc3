// topk.cu -- K3: per-unit top-k page selection (standalone kernel; see select.cuh).
//
// One CTA (128 threads) per unit stages the unit's keys once in shared memory and runs the
// block selection of select.cuh (histogram / bisection for the threshold key, ordered
// compaction for the lowest-logical-index tie rule, page-table translation in the epilogue).
// The decode engine normally runs the selection fused into the attention kernel
// (attend_fused.cu, pt_select_attend); this entry point is the C-ABI K3, the fallback
// outside the fused kernel's envelope, and the cross-check of the fused selection.
#include <stdlib.h>

#include "select.cuh"

namespace pt {

template <int kTopkThreads>
__global__ void __launch_bounds__(kTopkThreads)
    k_topk(const uint16_t *__restrict__ keys_g, const int32_t *__restrict__ seq_len,
           const int32_t *__restrict__ page_table, int S, int Pmax, int k,
           int32_t *__restrict__ sel, int32_t *__restrict__ sel_logical,
           int32_t *__restrict__ n_sel, int32_t *__restrict__ kth, int32_t *__restrict__ kplus1) {
    extern __shared__ __align__(16) uint16_t skeys[];
    __shared__ SelectShared<kTopkThreads> sh;
    __shared__ int bins[kSelectBins];
    const int64_t u = blockIdx.x;
    const int n = seq_len[u];
    const int P = (n + S - 1) / S;
    if (P == 0) {
        if (threadIdx.x == 0) { n_sel[u] = 0; kth[u] = 0; kplus1[u] = -1; }
        return;
    }
    const uint4 *src = reinterpret_cast<const uint4 *>(keys_g + u * (int64_t)Pmax);
    {  // all of a thread's 16-byte key loads in flight before its first shared store
        constexpr int kMax = 4;
        const int nv = (P + 7) / 8;
        for (int i0 = threadIdx.x; i0 < nv; i0 += kMax * kTopkThreads) {
            uint4 v[kMax];
#pragma unroll
            for (int j = 0; j < kMax; j++)
                if (i0 + j * kTopkThreads < nv) v[j] = __ldg(src + i0 + j * kTopkThreads);
#pragma unroll
            for (int j = 0; j < kMax; j++)
                if (i0 + j * kTopkThreads < nv) reinterpret_cast<uint4 *>(skeys)[i0 + j * kTopkThreads] = v[j];
        }
    }
    __syncthreads();
    select_block<kTopkThreads>(skeys, bins, P, k, page_table + u * Pmax, sel + u * (int64_t)k,
                               sel_logical ? sel_logical + u * (int64_t)k : nullptr, n_sel + u,
                               kth + u, kplus1 + u, sh,
                               reinterpret_cast<int *>(skeys + ((Pmax + 8) & ~7)));
}

}  // namespace pt

using namespace pt;

// keys (+1 pad key, 16-byte rounded) then the k-entry logical-id list
static size_t topk_smem_bytes(int Pmax, int k) { return (size_t)((Pmax + 8) / 8) * 16 + (size_t)k * 4; }

extern "C" int pt_topk(const uint16_t *keys, const int32_t *seq_len, const int32_t *page_table,
                       int U, int S, int Pmax, int k, int32_t *sel, int32_t *sel_logical,
                       int32_t *n_sel, int32_t *kth, int32_t *kplus1, void *stream) {
    if (!keys || !seq_len || !page_table || !sel || !n_sel || !kth || !kplus1 || U < 0 || S < 1 ||
        Pmax % 32)
        return PT_ERR_INVALID;
    if (k < 1) return PT_ERR_K;
    if (U == 0) return PT_OK;
    const size_t smem = topk_smem_bytes(Pmax, k);
    if (smem > 200 * 1024) return PT_ERR_UNSUPPORTED;
    // PT_TOPK_THREADS (128 / 256 / 512 / 1024) overrides the block size (tuning); 128 keeps
    // the conflict-free top-64 histogram of select_block in its 16 KB scratch
    const char *e = getenv("PT_TOPK_THREADS");
    const int nt = e ? atoi(e) : 128;
    cudaStream_t st = (cudaStream_t)stream;
#define PT_TOPK(NT_)                                                                           \
    if (nt == NT_) {                                                                           \
        static size_t configured = 0;                                                          \
        if (smem > configured) { /* static bins + dynamic keys may exceed 48 KB */              \
            PT_CUDA_TRY(cudaFuncSetAttribute(k_topk<NT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                             (int)smem));                                      \
            configured = smem;                                                                 \
        }                                                                                      \
        k_topk<NT_><<<U, NT_, smem, st>>>(keys, seq_len, page_table, S, Pmax, k, sel, sel_logical, \
                                          n_sel, kth, kplus1);                                 \
    } else
    PT_TOPK(256) PT_TOPK(512) PT_TOPK(1024) PT_TOPK(128)
#undef PT_TOPK
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}
