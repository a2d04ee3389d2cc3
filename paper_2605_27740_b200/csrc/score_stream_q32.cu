// score_stream_q32.cu -- K2 streaming-kernel instantiations for PT_F32 queries.
#include "score_stream.cuh"

namespace pt {

template <int SDT, int G, int D, int NST, int CPSW>
static int ss_launch_n(const StreamScoreParams &sp, int ctas, cudaStream_t st) {
    using C = SSCfg<PT_F32, SDT, G, D, NST, CPSW>;
    const size_t smem = ss_hdr_bytes(sp.U) + (size_t)kSSWarps * C::PER_WARP;
    while (ctas > 1 && smem * ctas > 226 * 1024) ctas--;
    if (smem * ctas > 226 * 1024) return PT_ERR_UNSUPPORTED;
    static size_t configured = 0;
    if (smem > configured) {
        PT_CUDA_TRY(cudaFuncSetAttribute(k_score_stream<PT_F32, SDT, G, D, NST, CPSW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    PT_CUDA_TRY(pt_launch(k_score_stream<PT_F32, SDT, G, D, NST, CPSW>, dim3(pt_num_sms() * ctas), dim3(kSSWarps * 32),
                          smem, st, sp));
    return PT_OK;
}

template <int SDT, int G, int D>
static int ss_launch(const StreamScoreParams &sp, cudaStream_t st) {
    const int ctas = ss_ctas_per_sm(sp.Pmax);
    return ctas >= 3 ? ss_launch_n<SDT, G, D, 3, 8>(sp, ctas, st) : ss_launch_n<SDT, G, D, 2, 16>(sp, ctas, st);
}

template <int SDT, int D>
static int ss_g(const StreamScoreParams &sp, int G, cudaStream_t st) {
    switch (G) {
        case 1: return ss_launch<SDT, 1, D>(sp, st);
        case 2: return ss_launch<SDT, 2, D>(sp, st);
        case 3: return ss_launch<SDT, 3, D>(sp, st);
        case 4: return ss_launch<SDT, 4, D>(sp, st);
        case 5: return ss_launch<SDT, 5, D>(sp, st);
        case 6: return ss_launch<SDT, 6, D>(sp, st);
        case 7: return ss_launch<SDT, 7, D>(sp, st);
        case 8: return ss_launch<SDT, 8, D>(sp, st);
        default: return PT_ERR_UNSUPPORTED;
    }
}

int launch_score_stream_q32(const StreamScoreParams &sp, int sdt, int G, int D, cudaStream_t st) {
    if (sdt == PT_F32 && D == 128) return ss_g<PT_F32, 128>(sp, G, st);
    if (sdt == PT_F32 && D == 64) return ss_g<PT_F32, 64>(sp, G, st);
    if (sdt == PT_BF16 && D == 128) return ss_g<PT_BF16, 128>(sp, G, st);
    if (sdt == PT_BF16 && D == 64) return ss_g<PT_BF16, 64>(sp, G, st);
    return PT_ERR_UNSUPPORTED;
}

}  // namespace pt
