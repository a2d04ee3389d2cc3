// attend_simt_bf16.cu -- CUDA-core K4 instantiations for PT_BF16 KV (attend.cuh).
#include "attend.cuh"

namespace pt {

template <int GP, int DPL>
static int launch_one(const AttnParams &prm, int U, int nsplit, int NW, size_t smem,
                      cudaStream_t st) {
    static size_t configured = 0;
    if (smem > configured) {
        PT_CUDA_TRY(cudaFuncSetAttribute(k_attend<PT_BF16, GP, DPL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    dim3 grid(nsplit, U);
    k_attend<PT_BF16, GP, DPL><<<grid, NW * 32, smem, st>>>(prm);
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}

int launch_attend_simt_bf16(const AttnParams &prm, int gp, int dpl, int U, int nsplit, int NW,
                         size_t smem, cudaStream_t st) {
#define PT_ATT(GP_, DPL_) \
    if (gp == GP_ && dpl == DPL_) return launch_one<GP_, DPL_>(prm, U, nsplit, NW, smem, st);
    PT_ATT(1, 1) PT_ATT(1, 2) PT_ATT(1, 4) PT_ATT(1, 8)
    PT_ATT(2, 1) PT_ATT(2, 2) PT_ATT(2, 4) PT_ATT(2, 8)
    PT_ATT(4, 1) PT_ATT(4, 2) PT_ATT(4, 4) PT_ATT(4, 8)
    PT_ATT(8, 1) PT_ATT(8, 2) PT_ATT(8, 4) PT_ATT(8, 8)
#undef PT_ATT
    return PT_ERR_UNSUPPORTED;
}

}  // namespace pt
