// attend.cu -- K4: split-KV paged decode attention over the selected pages.
//
// Restates attention.py:94-107 sparse_attention (+ kvcache.py:266-280 gather and
// attention.py:57-75 _run_stream) and _kernels_cy.pyx:129-172 stream_attention:
//   o_g = softmax(q_g . K_sel^T * scale + bias) V_sel,   lse_g = m + log(l)
// for the G query heads of a unit sharing one selection (attention.py:137-146), with
// f32 accumulation and running-max rescaling.  Dense attention (attention.py:78-91,
// the speed-up denominator) is the same kernel with sel = the unit's page table.
//
// B200 structure:
//   * grid (split, unit); a CTA owns a contiguous slice of the unit's selected pages.
//   * each warp streams its pages through a private ring of shared-memory stages: lane 0
//     issues one cp.async.bulk (1-D TMA, SASS UBLKCP) per K page and per V page, completion
//     tracked by an mbarrier with expect_tx; the gather of kvcache.py:266-280 never
//     materialises -- pages go HBM -> SMEM once, shared by all G heads of the group.
//   * lane owns DPL contiguous dims; QK partials for a TB x GP tile (TB*GP = 32) are
//     reduced with a transposing butterfly so lane L ends with score (t = L/GP, g = L%GP).
//   * warps merge through shared memory; splits merge in the last-arriving CTA of the unit
//     (atomic ticket, self-resetting for CUDA-graph replay).
#include "common.cuh"

namespace pt {

constexpr int kAttnMaxSplits = 64;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

template <int DT, int DPL>
__device__ __forceinline__ void load_lane_row(const char *row, int d0, bool on, float (&x)[DPL]) {
    if (!on) {
#pragma unroll
        for (int j = 0; j < DPL; j++) x[j] = 0.f;
        return;
    }
    if constexpr (DT == PT_BF16) {
        const char *p = row + d0 * 2;
        if constexpr (DPL == 1) {
            x[0] = bf16_bits_to_f32(*reinterpret_cast<const uint16_t *>(p));
        } else if constexpr (DPL == 2) {
            uint32_t w = *reinterpret_cast<const uint32_t *>(p);
            x[0] = bf16_lo(w); x[1] = bf16_hi(w);
        } else if constexpr (DPL == 4) {
            uint2 w = *reinterpret_cast<const uint2 *>(p);
            x[0] = bf16_lo(w.x); x[1] = bf16_hi(w.x); x[2] = bf16_lo(w.y); x[3] = bf16_hi(w.y);
        } else {
            uint4 w = *reinterpret_cast<const uint4 *>(p);
            x[0] = bf16_lo(w.x); x[1] = bf16_hi(w.x); x[2] = bf16_lo(w.y); x[3] = bf16_hi(w.y);
            x[4] = bf16_lo(w.z); x[5] = bf16_hi(w.z); x[6] = bf16_lo(w.w); x[7] = bf16_hi(w.w);
        }
    } else {
        const float *p = reinterpret_cast<const float *>(row) + d0;
        if constexpr (DPL == 1) {
            x[0] = p[0];
        } else if constexpr (DPL == 2) {
            float2 w = *reinterpret_cast<const float2 *>(p);
            x[0] = w.x; x[1] = w.y;
        } else {
#pragma unroll
            for (int j = 0; j < DPL; j += 4) {
                float4 w = *reinterpret_cast<const float4 *>(p + j);
                x[j] = w.x; x[j + 1] = w.y; x[j + 2] = w.z; x[j + 3] = w.w;
            }
        }
    }
}

// Transposing butterfly: in: v[32] partial sums per lane (index i); out: lane L holds
// the full warp sum of index L.
__device__ __forceinline__ float butterfly_reduce32(float (&v)[32]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int half = 16; half >= 1; half >>= 1) {
        const bool up = lane & half;
#pragma unroll
        for (int i = 0; i < half; i++) {
            const float keep = up ? v[i + half] : v[i];
            const float send = up ? v[i] : v[i + half];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
        }
    }
    return v[0];
}

// bytes before the stage ring: mbarriers + per-warp broadcast scratch, 128-B aligned
__host__ __device__ __forceinline__ size_t attn_hdr_bytes(int NW, int nstage, int GP) {
    const size_t b = (size_t)NW * nstage * 8 + (size_t)NW * (32 + GP) * 4;
    return (b + 127) & ~(size_t)127;
}

struct AttnParams {
    const void *q;
    const void *k_pool;
    const void *v_pool;
    const int32_t *sel;
    const int32_t *n_sel;
    const int32_t *page_table;
    const int32_t *seq_len;
    const float *bias;
    float *out;
    float *lse;
    float *ws;
    int32_t *tickets;
    int q_dtype, sel_stride, G, D, S, Pmax, pps, nstage, maxs;
    float scale;
};

template <int DT, int GP, int DPL>
__global__ void __launch_bounds__(128) k_attend(const AttnParams prm) {
    constexpr int E = DT == PT_F32 ? 4 : 2;
    constexpr int TB = 32 / GP;  // tokens per sub-block
    extern __shared__ __align__(128) char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const int64_t u = blockIdx.y;
    const int s = blockIdx.x;
    const int D = prm.D, S = prm.S, G = prm.G;
    const int n = prm.seq_len[u];
    const int P = (n + S - 1) / S;
    const int ns = prm.n_sel ? prm.n_sel[u] : P;  // n_sel == NULL: dense over the page table
    const int first = s * prm.pps;
    if (first >= ns) return;
    const int last = min(first + prm.pps, ns);
    const int nsplit_u = (ns + prm.pps - 1) / prm.pps;
    const int tail_pid = prm.page_table[u * prm.Pmax + P - 1];
    const int tail_rows = n - (P - 1) * S;

    const uint32_t page_bytes = (uint32_t)(S * D * E);
    const uint32_t stage_bytes = 2 * page_bytes;
    // smem: [mbarriers][p/carry scratch][stage rings | warp-merge area]
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem) + warp * prm.nstage;
    float *pscr = reinterpret_cast<float *>(smem + attn_hdr_bytes(NW, prm.nstage, GP) -
                                            (size_t)NW * (32 + GP) * 4) +
                  warp * (32 + GP);
    char *ring = smem + attn_hdr_bytes(NW, prm.nstage, GP);
    char *my_stages = ring + (size_t)warp * prm.nstage * stage_bytes;

    const int my_count = (last - first - warp + NW - 1) / NW > 0 ? (last - first - warp + NW - 1) / NW : 0;
    const int32_t *selu = prm.sel + u * (int64_t)prm.sel_stride;

    auto issue = [&](int i) {
        const int j = first + warp + i * NW;
        const int pid = selu[j];
        const int rows = (pid == tail_pid) ? tail_rows : S;
        const uint32_t bytes = (uint32_t)(rows * D * E);
        const int st = i % prm.nstage;
        char *ks = my_stages + (size_t)st * stage_bytes;
        mbar_arrive_expect_tx(&bars[st], 2 * bytes);
        bulk_g2s(ks, static_cast<const char *>(prm.k_pool) + (int64_t)pid * page_bytes, bytes, &bars[st]);
        bulk_g2s(ks + page_bytes, static_cast<const char *>(prm.v_pool) + (int64_t)pid * page_bytes,
                 bytes, &bars[st]);
    };
    if (lane == 0) {
        for (int i = 0; i < prm.nstage; i++) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (lane == 0)
        for (int i = 0; i < min(prm.nstage, my_count); i++) issue(i);

    // q (pre-scaled into the log2 domain), lane-owned dims
    const int d0 = lane * DPL;
    const bool on = d0 < D;
    const float qscale = prm.scale * kLog2e;
    float qr[GP][DPL];
#pragma unroll
    for (int g = 0; g < GP; g++)
#pragma unroll
        for (int j = 0; j < DPL; j++) {
            float v = 0.f;
            if (g < G && on) {
                const int64_t idx = (u * G + g) * (int64_t)D + d0 + j;
                v = prm.q_dtype == PT_F32 ? static_cast<const float *>(prm.q)[idx]
                                          : bf16_bits_to_f32(static_cast<const uint16_t *>(prm.q)[idx]);
            }
            qr[g][j] = v * qscale;
        }
    float acc[GP][DPL];
#pragma unroll
    for (int g = 0; g < GP; g++)
#pragma unroll
        for (int j = 0; j < DPL; j++) acc[g][j] = 0.f;
    const int my_g = lane % GP, my_t = lane / GP;
    float m_run = -INFINITY, l_run = 0.f;

    for (int i = 0; i < my_count; i++) {
        const int st = i % prm.nstage;
        const int j = first + warp + i * NW;
        const int pid = selu[j];
        const int rows = (pid == tail_pid) ? tail_rows : S;
        const float b2 = prm.bias ? prm.bias[u * prm.sel_stride + j] * kLog2e : 0.f;
        mbar_wait(&bars[st], (uint32_t)((i / prm.nstage) & 1));
        const char *ks = my_stages + (size_t)st * stage_bytes;
        const char *vs = ks + page_bytes;
        for (int t0 = 0; t0 < rows; t0 += TB) {
            float part[32];
#pragma unroll
            for (int t = 0; t < TB; t++) {
                float kx[DPL];
                load_lane_row<DT, DPL>(ks + (size_t)(t0 + t) * D * E, d0, on && (t0 + t < rows), kx);
#pragma unroll
                for (int g = 0; g < GP; g++) {
                    float a = 0.f;
#pragma unroll
                    for (int jj = 0; jj < DPL; jj++) a = fmaf(qr[g][jj], kx[jj], a);
                    part[t * GP + g] = a;
                }
            }
            float sc = butterfly_reduce32(part);
            const bool valid = (t0 + my_t < rows) && (my_g < G);
            sc = valid ? sc + b2 : -INFINITY;
            float mb = sc;
#pragma unroll
            for (int o = GP; o < 32; o <<= 1) mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, o));
            const float m_new = fmaxf(m_run, mb);
            const float m_use = m_new == -INFINITY ? 0.f : m_new;
            const float p = exp2f(sc - m_use);
            const float carry = exp2f(m_run - m_use);
            float lb = p;
#pragma unroll
            for (int o = GP; o < 32; o <<= 1) lb += __shfl_xor_sync(0xffffffffu, lb, o);
            l_run = l_run * carry + lb;
            m_run = m_new;
            // broadcast p and carries through the warp scratch
            pscr[lane] = p;
            if (lane < GP) pscr[32 + lane] = carry;
            __syncwarp();
#pragma unroll
            for (int g = 0; g < GP; g++) {
                const float c = pscr[32 + g];
#pragma unroll
                for (int jj = 0; jj < DPL; jj++) acc[g][jj] *= c;
            }
#pragma unroll
            for (int t = 0; t < TB; t++) {
                float vx[DPL];
                load_lane_row<DT, DPL>(vs + (size_t)(t0 + t) * D * E, d0, on && (t0 + t < rows), vx);
#pragma unroll
                for (int g = 0; g < GP; g++) {
                    const float pw = pscr[t * GP + g];
#pragma unroll
                    for (int jj = 0; jj < DPL; jj++) acc[g][jj] = fmaf(pw, vx[jj], acc[g][jj]);
                }
            }
            __syncwarp();
        }
        __syncwarp();  // every lane is done with this stage before it is refilled
        if (lane == 0 && i + prm.nstage < my_count) issue(i + prm.nstage);
    }

    // ---- merge warps (shared memory; stage buffers are free now) ----
    __syncthreads();
    float *macc = reinterpret_cast<float *>(ring);           // [NW][GP][D]
    float *mml = macc + (size_t)NW * GP * D;                  // [NW][GP][2]
#pragma unroll
    for (int g = 0; g < GP; g++)
#pragma unroll
        for (int jj = 0; jj < DPL; jj++)
            if (on) macc[((size_t)warp * GP + g) * D + d0 + jj] = acc[g][jj];
    if (lane < GP) {
        mml[(warp * GP + lane) * 2 + 0] = m_run;
        mml[(warp * GP + lane) * 2 + 1] = l_run;
    }
    __syncthreads();
    const bool single = (nsplit_u == 1);
    float *wacc = prm.ws;                                                    // [U][maxs][G][D]
    float *wml = prm.ws + (size_t)gridDim.y * prm.maxs * G * D;              // [U][maxs][G][2]
    for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
        const int g = i / D, d = i % D;
        float mt = -INFINITY;
        for (int w = 0; w < NW; w++) mt = fmaxf(mt, mml[(w * GP + g) * 2]);
        const float mu = mt == -INFINITY ? 0.f : mt;
        float lt = 0.f, a = 0.f;
        for (int w = 0; w < NW; w++) {
            const float f = exp2f(mml[(w * GP + g) * 2] - mu);
            lt += mml[(w * GP + g) * 2 + 1] * f;
            a += macc[((size_t)w * GP + g) * D + d] * f;
        }
        if (single) {
            prm.out[(u * G + g) * (int64_t)D + d] = a / lt;
            if (d == 0) prm.lse[u * G + g] = (mt + log2f(lt)) * kLn2;
        } else {
            wacc[((u * prm.maxs + s) * G + g) * (int64_t)D + d] = a;
            if (d == 0) {
                wml[((u * prm.maxs + s) * G + g) * 2 + 0] = mt;
                wml[((u * prm.maxs + s) * G + g) * 2 + 1] = lt;
            }
        }
    }
    if (single) return;

    // ---- split merge in the last CTA of the unit ----
    __shared__ int is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int t = atomicAdd(&prm.tickets[u], 1);
        is_last = (t == nsplit_u - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
        const int g = i / D, d = i % D;
        float mt = -INFINITY;
        for (int w = 0; w < nsplit_u; w++)
            mt = fmaxf(mt, __ldcg(&wml[((u * prm.maxs + w) * G + g) * 2]));
        const float mu = mt == -INFINITY ? 0.f : mt;
        float lt = 0.f, a = 0.f;
        for (int w = 0; w < nsplit_u; w++) {
            const float f = exp2f(__ldcg(&wml[((u * prm.maxs + w) * G + g) * 2]) - mu);
            lt += __ldcg(&wml[((u * prm.maxs + w) * G + g) * 2 + 1]) * f;
            a += __ldcg(&wacc[((u * prm.maxs + w) * G + g) * (int64_t)D + d]) * f;
        }
        prm.out[(u * G + g) * (int64_t)D + d] = a / lt;
        if (d == 0) prm.lse[u * G + g] = (mt + log2f(lt)) * kLn2;
    }
    if (threadIdx.x == 0) prm.tickets[u] = 0;
}

}  // namespace pt

using namespace pt;

static int gp_of(int G) { return G <= 1 ? 1 : G <= 2 ? 2 : G <= 4 ? 4 : G <= 8 ? 8 : -1; }
static int dpl_of(int D) { return D <= 32 ? 1 : D <= 64 ? 2 : D <= 128 ? 4 : D <= 256 ? 8 : -1; }

extern "C" size_t pt_attend_workspace_bytes(int U, int G, int D, int sel_stride) {
    (void)sel_stride;
    return (size_t)U * kAttnMaxSplits * G * ((size_t)D + 2) * sizeof(float);
}

template <int DT, int GP, int DPL>
static int launch_attend(const AttnParams &prm, int U, int nsplit, int NW, size_t smem,
                         cudaStream_t st) {
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        PT_CUDA_TRY(cudaFuncSetAttribute(k_attend<DT, GP, DPL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    dim3 grid(nsplit, U);
    k_attend<DT, GP, DPL><<<grid, NW * 32, smem, st>>>(prm);
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}

template <int DT>
static int dispatch_attend(const AttnParams &prm, int U, int nsplit, int NW, size_t smem,
                           cudaStream_t st) {
    const int gp = gp_of(prm.G), dpl = dpl_of(prm.D);
#define PT_ATT(GP_, DPL_) \
    if (gp == GP_ && dpl == DPL_) return launch_attend<DT, GP_, DPL_>(prm, U, nsplit, NW, smem, st);
    PT_ATT(1, 1) PT_ATT(1, 2) PT_ATT(1, 4) PT_ATT(1, 8)
    PT_ATT(2, 1) PT_ATT(2, 2) PT_ATT(2, 4) PT_ATT(2, 8)
    PT_ATT(4, 1) PT_ATT(4, 2) PT_ATT(4, 4) PT_ATT(4, 8)
    PT_ATT(8, 1) PT_ATT(8, 2) PT_ATT(8, 4) PT_ATT(8, 8)
#undef PT_ATT
    return PT_ERR_UNSUPPORTED;
}

extern "C" int pt_attend(const void *q, int q_dtype, const void *k_pool, const void *v_pool,
                         int kv_dtype, const int32_t *sel, int sel_stride, const int32_t *n_sel,
                         const int32_t *page_table, const int32_t *seq_len, int U, int G, int D,
                         int S, int Pmax, const float *bias, float scale, float *out, float *lse,
                         void *workspace, size_t workspace_bytes, int32_t *tickets, int nsplit,
                         void *stream) {
    if (!q || !k_pool || !v_pool || !sel || !page_table || !seq_len || !out || !lse ||
        U < 0 || G < 1 || S < 1 || sel_stride < 1)
        return PT_ERR_INVALID;
    const int E = kv_dtype == PT_F32 ? 4 : 2;
    if (gp_of(G) < 0 || dpl_of(D) < 0 || (D * E) % 16 || D % dpl_of(D)) return PT_ERR_UNSUPPORTED;
    if (U == 0) return PT_OK;
    // warps per CTA and ring depth: keep >= 2 CTAs per SM where the page size allows
    const size_t stage = (size_t)2 * S * D * E;
    int NW = 4, nstage = 3;
    auto smem_of = [&](int nw, int nst) {
        const size_t ring = (size_t)nw * nst * stage;
        const size_t merge = (size_t)nw * gp_of(G) * (D + 2) * 4;
        return attn_hdr_bytes(nw, nst, gp_of(G)) + (ring > merge ? ring : merge);
    };
    while (smem_of(NW, nstage) > 110 * 1024 && nstage > 2) nstage--;
    while (smem_of(NW, nstage) > 110 * 1024 && NW > 1) NW--;
    if (smem_of(NW, nstage) > 220 * 1024) return PT_ERR_UNSUPPORTED;
    const size_t smem = smem_of(NW, nstage);
    const int ctas_per_sm = smem <= 110 * 1024 ? 2 : 1;
    if (nsplit <= 0) {
        const int target = 148 * ctas_per_sm * 2;
        nsplit = (target + U - 1) / U;
    }
    int max_useful = (sel_stride + NW - 1) / NW;
    if (nsplit > max_useful) nsplit = max_useful;
    if (nsplit > kAttnMaxSplits) nsplit = kAttnMaxSplits;
    if (nsplit < 1) nsplit = 1;
    const int pps = (sel_stride + nsplit - 1) / nsplit;
    nsplit = (sel_stride + pps - 1) / pps;
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
    if (kv_dtype == PT_F32) return dispatch_attend<PT_F32>(prm, U, nsplit, NW, smem, st);
    if (kv_dtype == PT_BF16) return dispatch_attend<PT_BF16>(prm, U, nsplit, NW, smem, st);
    return PT_ERR_INVALID;
}
