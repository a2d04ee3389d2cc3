// attend_mma.cu -- tensor-core (mma.sync + TMA) K4 instantiations for bf16 KV (attend.cuh).
#include "attend.cuh"

namespace pt {

template <int D, int MT>
static int launch_one(const CUtensorMap &tk, const CUtensorMap &tv, const AttnParams &prm, int U,
                      int nsplit, int NW, size_t smem, cudaStream_t st) {
    static size_t configured = 0;
    if (smem > configured) {
        PT_CUDA_TRY(cudaFuncSetAttribute(k_attend_mma<D, MT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    dim3 grid(nsplit, U);
    k_attend_mma<D, MT><<<grid, NW * 32, smem, st>>>(tk, tv, prm);
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}

int launch_attend_mma(const CUtensorMap &tk, const CUtensorMap &tv, const AttnParams &prm, int U,
                      int nsplit, int NW, size_t smem, cudaStream_t st) {
    const int D = prm.D, S = prm.S;
#define PT_MMA(D_, MT_) \
    if (D == D_ && S == 16 * MT_) return launch_one<D_, MT_>(tk, tv, prm, U, nsplit, NW, smem, st);
    PT_MMA(64, 1) PT_MMA(64, 2) PT_MMA(64, 4)
    PT_MMA(128, 1) PT_MMA(128, 2) PT_MMA(128, 4)
    PT_MMA(256, 1) PT_MMA(256, 2) PT_MMA(256, 4)
#undef PT_MMA
    return PT_ERR_UNSUPPORTED;
}

template <int D, int MT>
static int launch_stream_one(const CUtensorMap &tk, const CUtensorMap &tv, const StreamParams &p,
                             int grid, int NW, size_t smem, cudaStream_t st) {
    static size_t configured = 0;
    if (smem > configured) {
        PT_CUDA_TRY(cudaFuncSetAttribute(k_attend_stream<D, MT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    k_attend_stream<D, MT><<<grid, NW * 32, smem, st>>>(tk, tv, p);
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}

int launch_attend_stream(const CUtensorMap &tk, const CUtensorMap &tv, const StreamParams &p,
                         int D, int S, int grid, int NW, size_t smem, cudaStream_t st) {
#define PT_STR(D_, MT_) \
    if (D == D_ && S == 16 * MT_) return launch_stream_one<D_, MT_>(tk, tv, p, grid, NW, smem, st);
    PT_STR(64, 1) PT_STR(64, 2) PT_STR(64, 4)
    PT_STR(128, 1) PT_STR(128, 2) PT_STR(128, 4)
    PT_STR(256, 1) PT_STR(256, 2) PT_STR(256, 4)
#undef PT_STR
    return PT_ERR_UNSUPPORTED;
}

}  // namespace pt
