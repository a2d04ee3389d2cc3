// attend.cu -- host side of K4: pt_attend (path choice, split sizing, TMA tensor maps).
// Kernels: attend.cuh; instantiations: attend_mma.cu, attend_simt_{f32,bf16}.cu.
#include "attend.cuh"

namespace pt {
int launch_attend_mma(const CUtensorMap &tk, const CUtensorMap &tv, const AttnParams &prm, int U,
                      int nsplit, int NW, size_t smem, cudaStream_t st);
int launch_attend_stream(const CUtensorMap &tk, const CUtensorMap &tv, const StreamParams &p,
                         int D, int S, int grid, int NW, size_t smem, cudaStream_t st);
int launch_attend_simt_f32(const AttnParams &prm, int gp, int dpl, int U, int nsplit, int NW,
                           size_t smem, cudaStream_t st);
int launch_attend_simt_bf16(const AttnParams &prm, int gp, int dpl, int U, int nsplit, int NW,
                            size_t smem, cudaStream_t st);
}  // namespace pt

using namespace pt;

static int gp_of(int G) { return G <= 1 ? 1 : G <= 2 ? 2 : G <= 4 ? 4 : G <= 8 ? 8 : -1; }
static int dpl_of(int D) { return D <= 32 ? 1 : D <= 64 ? 2 : D <= 128 ? 4 : D <= 256 ? 8 : -1; }

extern "C" size_t pt_attend_workspace_bytes(int U, int G, int D, int sel_stride) {
    (void)sel_stride;
    return (size_t)U * kAttnMaxSplits * G * ((size_t)D + 2) * sizeof(float);
}

// ---------------------------------------------------------------------------
// TMA tensor maps over the KV pool ([num_phys_pages * S rows][D cols] bf16)
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

static bool make_pool_tmap(CUtensorMap *tm, const void *base, int D, int S, int64_t pages) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)pages * (cuuint64_t)S};
    cuuint64_t strides[1] = {(cuuint64_t)D * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)S};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims,
                     strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// shared with attend_fused.cu
bool pt_make_pool_tmap(CUtensorMap *m, const void *pool, int D, int S, int num_pages) {
    return make_pool_tmap(m, pool, D, S, num_pages);
}

// PT_ATTEND_SIMT=1 forces the CUDA-core kernel (used by the parity tests to pin both paths);
// PT_ATTEND_SPLIT=1 forces the (split, unit) grid instead of the streaming kernel;
// PT_ATTEND_NSTAGE / PT_ATTEND_CHUNK override the streaming ring depth / chunk size.
static bool simt_forced() {
    const char *e = getenv("PT_ATTEND_SIMT");
    return e && e[0] == '1';
}
static int env_int(const char *name, int dflt) {
    const char *e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}

extern "C" int pt_attend(const void *q, int q_dtype, const void *k_pool, const void *v_pool,
                         int kv_dtype, int num_phys_pages, const int32_t *sel, int sel_stride, const int32_t *n_sel,
                         const int32_t *page_table, const int32_t *seq_len, int U, int G, int D,
                         int S, int Pmax, const float *bias, float scale, float *out, float *lse,
                         void *workspace, size_t workspace_bytes, int32_t *tickets, int nsplit,
                         void *stream) {
    if (!q || !k_pool || !v_pool || !sel || !page_table || !seq_len || !out || !lse ||
        U < 0 || G < 1 || S < 1 || sel_stride < 1)
        return PT_ERR_INVALID;
    const int E = kv_dtype == PT_F32 ? 4 : 2;
    const bool mma = kv_dtype == PT_BF16 && G <= 8 && (D == 64 || D == 128 || D == 256) &&
                     (S == 16 || S == 32 || S == 64) && num_phys_pages > 0 && !simt_forced();
    // sparse selections on the tensor-core path: persistent streaming kernel (one wave of
    // warps, balanced contiguous ranges of the concatenated page lists)
    if (mma && n_sel != nullptr && U > 0 && U <= 8192 && env_int("PT_ATTEND_SPLIT", 0) == 0) {
        const int stage_bytes = 2 * S * D * 2;
        const int NW = 4;
        int nstage = env_int("PT_ATTEND_NSTAGE", 0);
        if (nstage <= 0) nstage = 3;
        const int ctas_per_sm = env_int("PT_ATTEND_CTAS", 2);
        const int grid = pt_num_sms() * ctas_per_sm;
        const int W = grid * NW;
        const long long pages_ub = (long long)U * sel_stride;  // bound; exact count on device
        int L = (int)((pages_ub + W - 1) / W);
        // at most kAttnMaxSplits partial slots per unit
        const int lmin = (sel_stride + kAttnMaxSplits - 3) / (kAttnMaxSplits - 2);
        if (L < lmin) L = lmin;
        if (L < 1) L = 1;
        const size_t smem = attn_stream_hdr(U, NW, L, nstage) + (size_t)NW * nstage * stage_bytes;
        if (L <= 4096 && smem <= 225 * 1024 &&
            workspace && tickets &&
            workspace_bytes >= pt_attend_workspace_bytes(U, G, D, sel_stride)) {
            CUtensorMap tk, tv;
            if (!make_pool_tmap(&tk, k_pool, D, S, num_phys_pages) ||
                !make_pool_tmap(&tv, v_pool, D, S, num_phys_pages))
                return PT_ERR_UNSUPPORTED;
            StreamParams sp;
            sp.q = q; sp.sel = sel; sp.n_sel = n_sel; sp.page_table = page_table;
            sp.seq_len = seq_len; sp.bias = bias; sp.out = out; sp.lse = lse;
            sp.ws = static_cast<float *>(workspace); sp.tickets = tickets;
            sp.q_dtype = q_dtype; sp.sel_stride = sel_stride; sp.U = U; sp.G = G;
            sp.Pmax = Pmax; sp.L = L; sp.maxparts = kAttnMaxSplits; sp.nstage = nstage;
            sp.scale = scale;
            return launch_attend_stream(tk, tv, sp, D, S, grid, NW, smem, (cudaStream_t)stream);
        }
    }
    if (!mma && (gp_of(G) < 0 || dpl_of(D) < 0 || (D * E) % 16 || D % dpl_of(D)))
        return PT_ERR_UNSUPPORTED;
    if (U == 0) return PT_OK;
    // warps per CTA and ring depth: keep >= 2 CTAs per SM where the page size allows
    const size_t stage = (size_t)2 * S * D * E;
    const int gpl = mma ? kMmaGP : gp_of(G);
    const int kMaxPps = 2048;  // bounds the per-warp page-id lists of the mma kernel (8 KB)
    auto smem_of = [&](int nw, int nst, int pps_) {
        const size_t ring = (size_t)nw * nst * stage;
        const size_t merge = (size_t)nw * gpl * (D + 2) * 4;
        const size_t hdr = mma ? attn_mma_hdr_bytes(nw, nst, pps_) : attn_hdr_bytes(nw, nst, gpl);
        return hdr + (ring > merge ? ring : merge);
    };
    int NW = 4, nstage = 3;
    while (smem_of(NW, nstage, kMaxPps) > 110 * 1024 && nstage > 2) nstage--;
    while (smem_of(NW, nstage, kMaxPps) > 110 * 1024 && NW > 2) NW--;
    while (smem_of(NW, nstage, kMaxPps) > 220 * 1024 && NW > 1) NW--;
    if (smem_of(NW, nstage, kMaxPps) > 220 * 1024) return PT_ERR_UNSUPPORTED;
    const int ctas_per_sm = smem_of(NW, nstage, kMaxPps) <= 110 * 1024 ? 2 : 1;
    if (nsplit <= 0) {
        // enough CTAs for ~4 waves of the resident slots
        const int target = pt_num_sms() * ctas_per_sm * 4;
        nsplit = (target + U - 1) / U;
    }
    const int max_useful = (sel_stride + NW - 1) / NW;
    if (nsplit > max_useful) nsplit = max_useful;
    if (nsplit > kAttnMaxSplits) nsplit = kAttnMaxSplits;
    const int min_split = (sel_stride + kMaxPps - 1) / kMaxPps;
    if (nsplit < min_split) nsplit = min_split;
    if (nsplit < 1) nsplit = 1;
    if (nsplit > kAttnMaxSplits) return PT_ERR_UNSUPPORTED;
    const int pps = (sel_stride + nsplit - 1) / nsplit;
    nsplit = (sel_stride + pps - 1) / pps;
    const size_t smem = smem_of(NW, nstage, pps);
    if (nsplit > 1) {
        if (!workspace || !tickets ||
            workspace_bytes < pt_attend_workspace_bytes(U, G, D, sel_stride))
            return PT_ERR_INVALID;
    }
    AttnParams prm;
    prm.q = q; prm.k_pool = k_pool; prm.v_pool = v_pool; prm.sel = sel; prm.n_sel = n_sel;
    prm.page_table = page_table; prm.seq_len = seq_len; prm.bias = bias; prm.out = out;
    prm.lse = lse; prm.ws = static_cast<float *>(workspace); prm.tickets = tickets;
    prm.q_dtype = q_dtype; prm.sel_stride = sel_stride; prm.G = G; prm.D = D; prm.S = S;
    prm.Pmax = Pmax; prm.pps = pps; prm.nstage = nstage; prm.maxs = kAttnMaxSplits;
    prm.scale = scale;
    cudaStream_t st = (cudaStream_t)stream;
    if (mma) {
        CUtensorMap tk, tv;
        if (!make_pool_tmap(&tk, k_pool, D, S, num_phys_pages) ||
            !make_pool_tmap(&tv, v_pool, D, S, num_phys_pages))
            return PT_ERR_UNSUPPORTED;
        return launch_attend_mma(tk, tv, prm, U, nsplit, NW, smem, st);
    }
    if (kv_dtype == PT_F32)
        return launch_attend_simt_f32(prm, gp_of(G), dpl_of(D), U, nsplit, NW, smem, st);
    if (kv_dtype == PT_BF16)
        return launch_attend_simt_bf16(prm, gp_of(G), dpl_of(D), U, nsplit, NW, smem, st);
    return PT_ERR_INVALID;
}
