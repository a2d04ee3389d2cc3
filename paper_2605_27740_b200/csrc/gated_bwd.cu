// gated_bwd.cu -- backward of the soft-mask gated attention (training path).
//
// Restates softmask.py:178-217 gated_attention_backward for every unit (kv head) and its G
// query heads at once, over the paged pool:
//   z_t   = scale * (k_t . q_g) + log(gate_p)           (t in page p; recomputed, flash-style)
//   w_t   = exp(z_t - lse_g)
//   dz_t  = w_t * (v_t . dout_g - dout_g . out_g)
//   dV_t += w_t * dout_g             dK_t += scale * dz_t * q_g        (summed over g)
//   dq_g += scale * sum_t dz_t k_t   dgate_p += sum_{g,t} dz_t / gate_p
// Hard-mode (gate 0) pages carry no weight and are skipped, as the reference.
//
// Layout: grid (page groups, units); one warp per page at a time.  The page's K and V rows
// are staged in warp-private shared memory (XOR-swizzled 16-byte chunks); lanes
// first own tokens (dot products, softmax weights) then dimensions (coalesced dK / dV row
// writes and the dq partial).  dq partials are reduced in the CTA and added to global memory
// with one atomic per (head, dim) per CTA.  f32 throughout (the reference runs float64:
// parity is to a stated tolerance).  The pass reads K and V once and writes dK and dV once:
// HBM-bound like the forward.
#include "common.cuh"

namespace pt {

constexpr int kGBWarps = 4;

struct GatedBwdParams {
    const void *q;          // [U*G][D] q_dtype
    const void *k_pool;     // [pages][S][D] kv_dtype
    const void *v_pool;
    const int32_t *page_table;  // [U][Pmax]
    const int32_t *seq_len;     // [U]
    const float *gates;         // [U][Pmax] gate per logical page (0 = skipped)
    const float *out;           // [U*G][D] forward output
    const float *lse;           // [U*G]
    const float *dout;          // [U*G][D]
    float *dq;                  // [U*G][D] (accumulated: zero it first)
    float *dk_pool;             // [pages][S][D] f32
    float *dv_pool;
    float *dgates;              // [U][Pmax]
    int q_dtype, kv_dtype, G, D, S, Pmax;
    float scale;
};

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Staged rows are unpadded; the 16-byte chunk c of row r sits at chunk c ^ (r & m), m + 1 =
// the largest power of two <= 8 dividing the chunks per row (an XOR swizzle: rows of a page
// map the same logical chunk to different banks, as the former 16-byte row padding did,
// without its shared memory -- three CTAs per SM instead of two)
__device__ __forceinline__ int gb_swz_mask(int vpr) {
    const int low = vpr & -vpr;
    return (low < 8 ? low : 8) - 1;
}
// raw staged element d of row r -> f32
template <int DT>
__device__ __forceinline__ float rawval(const char *row, int r, int d, int m) {
    constexpr int ES = DT == PT_F32 ? 4 : 2, EPV = 16 / ES;
    const char *a = row + (((d / EPV) ^ (r & m)) << 4) + (d % EPV) * ES;
    if constexpr (DT == PT_F32) return *reinterpret_cast<const float *>(a);
    else return bf16_bits_to_f32(*reinterpret_cast<const uint16_t *>(a));
}

// Double-buffered: while a warp computes page i, its next page's K and V rows are already
// in flight (cp.async, 16 B, raw storage format, padded rows); skipped (hard-masked) pages
// and the unused rows of a partial page get zero dK / dV, so the pools need no zero fill.
template <int DT, int MAXG, int DJ>
__global__ void __launch_bounds__(kGBWarps * 32) k_gated_bwd(const GatedBwdParams p) {
    constexpr int ES = DT == PT_F32 ? 4 : 2;
    constexpr int EPV = 16 / ES;  // elements per 16-byte vector
    extern __shared__ __align__(16) float gsm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int D = p.D, S = p.S, G = p.G;
    const int64_t u = blockIdx.y;
    float *qs = gsm;                        // [MAXG][D]
    float *dos = qs + MAXG * D;             // [MAXG][D]
    float *sg = dos + MAXG * D;             // [8]
    float *lg = sg + 8;                     // [8]
    float *dqp = lg + 8;                    // [MAXG][D] CTA partial of dq
    const int rowb = D * ES;                // unpadded row (bytes), chunks swizzled
    const int pageb = S * rowb;
    char *wb = reinterpret_cast<char *>(dqp + MAXG * D) + (size_t)warp * (4 * pageb + 2 * MAXG * S * 4);
    float *wv = reinterpret_cast<float *>(wb + 4 * pageb);  // [S][MAXG]
    float *dzv = wv + MAXG * S;                              // [S][MAXG]
    // heads G..MAXG-1 are padding: zero q / dout and lse = +inf, so their softmax weights
    // and gradients are exactly zero and every per-head loop runs MAXG times, branch-free
    for (int i = threadIdx.x; i < MAXG * D; i += blockDim.x) {
        const int g = i / D, d = i % D;
        float qv = 0.f, dv = 0.f;
        if (g < G) {
            const int64_t row = (u * G + g) * (int64_t)D + d;
            qv = p.q_dtype == PT_F32 ? static_cast<const float *>(p.q)[row]
                                     : bf16_bits_to_f32(static_cast<const uint16_t *>(p.q)[row]);
            dv = p.dout[row];
        }
        qs[g * D + d] = qv;
        dos[g * D + d] = dv;
        dqp[g * D + d] = 0.f;
    }
    __syncthreads();
    for (int g = warp; g < MAXG; g += kGBWarps) {  // s_g = dout_g . out_g (warp per head)
        float a = 0.f;
        if (g < G)
            for (int d = lane; d < D; d += 32) a += dos[g * D + d] * p.out[(u * G + g) * (int64_t)D + d];
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) { sg[g] = a; lg[g] = g < G ? p.lse[u * G + g] : INFINITY; }
    }
    __syncthreads();
    // lanes own DJ consecutive dimensions (d = lane * DJ + j): vector shared loads of the
    // staged K row and vector dK / dV stores in the dims phase
    float qr[MAXG][DJ], dr[MAXG][DJ], dq_acc[MAXG][DJ];
#pragma unroll
    for (int g = 0; g < MAXG; g++)
#pragma unroll
        for (int j = 0; j < DJ; j++) {
            const int d = lane * DJ + j;
            const bool ok = d < D;
            qr[g][j] = ok ? qs[g * D + d] : 0.f;
            dr[g][j] = ok ? dos[g * D + d] : 0.f;
            dq_acc[g][j] = 0.f;
        }
    const int n = p.seq_len[u];
    const int P = (n + S - 1) / S;
    // lanes per token in the dot-product phase: split a row into whole 16-byte vectors
    int lpt = S >= 32 ? 1 : 32 / S;
    while (lpt > 1 && (D / lpt) % EPV) lpt >>= 1;
    const int part = lane % lpt, dlen = D / lpt;
    const int vpr = D * ES / 16;           // 16-byte vectors per row
    const int swm = gb_swz_mask(vpr);
    const int stride = gridDim.x * kGBWarps;
    auto issue = [&](int lp, int b) {      // page lp -> buffer b (nothing for a skipped page)
        if (lp < P && p.gates[u * p.Pmax + lp] != 0.f) {
            const int64_t pid = p.page_table[u * p.Pmax + lp];
            const int rows = min(S, n - lp * S);
            const char *kg = static_cast<const char *>(p.k_pool) + pid * S * D * ES;
            const char *vg = static_cast<const char *>(p.v_pool) + pid * S * D * ES;
            char *kb = wb + b * 2 * pageb, *vb = kb + pageb;
            if (vpr <= 32 && 32 % vpr == 0) {  // fixed chunk per lane, 32 / vpr rows per round
                const int c = lane % vpr, rpi = 32 / vpr;
                for (int r = lane / vpr; r < rows; r += rpi) {
                    const int cs = (c ^ (r & swm)) << 4;
                    const int64_t off = (int64_t)(r * vpr + c) * 16;
                    cp_async16(kb + r * rowb + cs, kg + off);
                    cp_async16(vb + r * rowb + cs, vg + off);
                }
            } else {
                for (int i = lane; i < rows * vpr; i += 32) {
                    const int r = i / vpr, c = i - r * vpr;
                    const int cs = (c ^ (r & swm)) << 4;
                    cp_async16(kb + r * rowb + cs, kg + (int64_t)i * 16);
                    cp_async16(vb + r * rowb + cs, vg + (int64_t)i * 16);
                }
            }
        }
        cp_async_commit();  // (possibly empty) one group per page keeps the accounting uniform
    };
    int lp = blockIdx.x * kGBWarps + warp;
    issue(lp, 0);
    for (int it = 0; lp < P; it++, lp += stride) {
        issue(lp + stride, (it + 1) & 1);
        cp_async_wait1();  // this page's group has landed (the next one may be in flight)
        __syncwarp();
        const float gate = p.gates[u * p.Pmax + lp];
        const int64_t pid = p.page_table[u * p.Pmax + lp];
        const int rows = min(S, n - lp * S);
        const int64_t base = pid * S * D;
        if (gate == 0.f) {  // hard-masked: no weight, no gradient
            for (int i = lane; i < S * D; i += 32) {
                p.dk_pool[base + i] = 0.f;
                p.dv_pool[base + i] = 0.f;
            }
            if (lane == 0) p.dgates[u * p.Pmax + lp] = 0.f;
            __syncwarp();
            continue;
        }
        const float lgate = logf(gate);
        const char *kb = wb + (it & 1) * 2 * pageb, *vb = kb + pageb;
        // lanes own (token, D/lpt slice): 16-byte raw vectors, all heads per vector
        float dgate = 0.f;
        for (int t0 = 0; t0 < S; t0 += 32 / lpt) {
            const int t = t0 + lane / lpt;
            const bool live = t < rows;
            float kq[MAXG], vd[MAXG];
#pragma unroll
            for (int g = 0; g < MAXG; g++) kq[g] = vd[g] = 0.f;
            if (live) {
                const char *kr = kb + t * rowb;
                const char *vr = vb + t * rowb;
                const int c0 = part * dlen / EPV;
                for (int c = 0; c < dlen / EPV; c++) {
                    const int cs = ((c0 + c) ^ (t & swm)) << 4;
                    const uint4 kx = *reinterpret_cast<const uint4 *>(kr + cs);
                    const uint4 vx = *reinterpret_cast<const uint4 *>(vr + cs);
                    float kf[EPV], vf[EPV];
                    if constexpr (DT == PT_F32) {
                        kf[0] = __uint_as_float(kx.x); kf[1] = __uint_as_float(kx.y);
                        kf[2] = __uint_as_float(kx.z); kf[3] = __uint_as_float(kx.w);
                        vf[0] = __uint_as_float(vx.x); vf[1] = __uint_as_float(vx.y);
                        vf[2] = __uint_as_float(vx.z); vf[3] = __uint_as_float(vx.w);
                    } else {
                        const uint32_t kw[4] = {kx.x, kx.y, kx.z, kx.w}, vw[4] = {vx.x, vx.y, vx.z, vx.w};
#pragma unroll
                        for (int q2 = 0; q2 < 4; q2++) {
                            kf[2 * q2] = bf16_lo(kw[q2]); kf[2 * q2 + 1] = bf16_hi(kw[q2]);
                            vf[2 * q2] = bf16_lo(vw[q2]); vf[2 * q2 + 1] = bf16_hi(vw[q2]);
                        }
                    }
                    const int d0 = part * dlen + c * EPV;
#pragma unroll
                    for (int g = 0; g < MAXG; g++) {
#pragma unroll
                        for (int e4 = 0; e4 < EPV; e4 += 4) {
                            const float4 q4 = *reinterpret_cast<const float4 *>(qs + g * D + d0 + e4);
                            const float4 o4 = *reinterpret_cast<const float4 *>(dos + g * D + d0 + e4);
                            kq[g] = fmaf(kf[e4], q4.x, fmaf(kf[e4 + 1], q4.y, fmaf(kf[e4 + 2], q4.z, fmaf(kf[e4 + 3], q4.w, kq[g]))));
                            vd[g] = fmaf(vf[e4], o4.x, fmaf(vf[e4 + 1], o4.y, fmaf(vf[e4 + 2], o4.z, fmaf(vf[e4 + 3], o4.w, vd[g]))));
                        }
                    }
                }
            }
#pragma unroll
            for (int g = 0; g < MAXG; g++) {
                for (int o = 1; o < lpt; o <<= 1) {
                    kq[g] += __shfl_xor_sync(0xffffffffu, kq[g], o);
                    vd[g] += __shfl_xor_sync(0xffffffffu, vd[g], o);
                }
                float w = 0.f, dz = 0.f;
                if (live) {
                    w = expf(kq[g] * p.scale + lgate - lg[g]);
                    dz = w * (vd[g] - sg[g]);
                }
                if (part == 0 && t < S) {
                    wv[t * MAXG + g] = w;
                    dzv[t * MAXG + g] = dz;
                    dgate += dz;
                }
            }
        }
        for (int o = 16; o > 0; o >>= 1) dgate += __shfl_xor_sync(0xffffffffu, dgate, o);
        if (lane == 0) p.dgates[u * p.Pmax + lp] = dgate / gate;
        __syncwarp();
        // lanes own dims: dK / dV rows (summed over heads); rows past the page's end are
        // written as zeros below (their staged K rows are stale, so they stay out of dq)
        for (int t = 0; t < rows; t++) {
            float wt[MAXG], zt[MAXG];
#pragma unroll
            for (int g4 = 0; g4 < MAXG; g4 += 4) {
                const float4 a = *reinterpret_cast<const float4 *>(wv + t * MAXG + g4);
                const float4 b = *reinterpret_cast<const float4 *>(dzv + t * MAXG + g4);
                wt[g4] = a.x; wt[g4 + 1] = a.y; wt[g4 + 2] = a.z; wt[g4 + 3] = a.w;
                zt[g4] = b.x; zt[g4 + 1] = b.y; zt[g4 + 2] = b.z; zt[g4 + 3] = b.w;
            }
            float kv[DJ];
            if (DJ % 4 == 0 && D == 32 * DJ) {  // 4 consecutive dims share one 16-byte chunk
#pragma unroll
                for (int j4 = 0; j4 < DJ; j4 += 4) {
                    const int d = lane * DJ + j4;
                    const char *a = kb + t * rowb + (((d / EPV) ^ (t & swm)) << 4) + (d % EPV) * ES;
                    if constexpr (DT == PT_F32) {
                        const float4 x = *reinterpret_cast<const float4 *>(a);
                        kv[j4] = x.x; kv[j4 + 1] = x.y; kv[j4 + 2] = x.z; kv[j4 + 3] = x.w;
                    } else {
                        const uint2 x = *reinterpret_cast<const uint2 *>(a);
                        kv[j4] = bf16_lo(x.x); kv[j4 + 1] = bf16_hi(x.x);
                        kv[j4 + 2] = bf16_lo(x.y); kv[j4 + 3] = bf16_hi(x.y);
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < DJ; j++) {
                    const int d = lane * DJ + j;
                    kv[j] = d < D ? rawval<DT>(kb + t * rowb, t, d, swm) : 0.f;
                }
            }
            float dk[DJ], dv[DJ];
#pragma unroll
            for (int j = 0; j < DJ; j++) {
                dk[j] = dv[j] = 0.f;
#pragma unroll
                for (int g = 0; g < MAXG; g++) {
                    dv[j] = fmaf(wt[g], dr[g][j], dv[j]);
                    dk[j] = fmaf(zt[g], qr[g][j], dk[j]);
                    dq_acc[g][j] = fmaf(zt[g], kv[j], dq_acc[g][j]);
                }
                dk[j] *= p.scale;
            }
            float *dkr = p.dk_pool + base + (int64_t)t * D;
            float *dvr = p.dv_pool + base + (int64_t)t * D;
            if (DJ % 4 == 0 && D == 32 * DJ) {
#pragma unroll
                for (int j4 = 0; j4 < DJ; j4 += 4) {
                    const int d = lane * DJ + j4;
                    __stcs(reinterpret_cast<float4 *>(dkr + d), make_float4(dk[j4], dk[j4 + 1], dk[j4 + 2], dk[j4 + 3]));
                    __stcs(reinterpret_cast<float4 *>(dvr + d), make_float4(dv[j4], dv[j4 + 1], dv[j4 + 2], dv[j4 + 3]));
                }
            } else {
#pragma unroll
                for (int j = 0; j < DJ; j++) {
                    const int d = lane * DJ + j;
                    if (d < D) { dkr[d] = dk[j]; dvr[d] = dv[j]; }
                }
            }
        }
        for (int i = rows * D + lane; i < S * D; i += 32) {
            p.dk_pool[base + i] = 0.f;
            p.dv_pool[base + i] = 0.f;
        }
        __syncwarp();  // the buffer is reused two pages later
    }
    // dq: warp partials -> CTA (shared atomics) -> global (one atomic per element per CTA)
#pragma unroll
    for (int g = 0; g < MAXG; g++) {
        if (g >= G) break;
#pragma unroll
        for (int j = 0; j < DJ; j++) {
            const int d = lane * DJ + j;
            if (d < D) atomicAdd(&dqp[g * D + d], dq_acc[g][j] * p.scale);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
        const float v = dqp[i];
        if (v != 0.f) atomicAdd(&p.dq[(u * G + i / D) * (int64_t)D + i % D], v);
    }
}

}  // namespace pt

using namespace pt;

template <int DT, int MAXG, int DJ>
static int launch_gbwd(const GatedBwdParams &p, int U, cudaStream_t st) {
    constexpr int ES = DT == PT_F32 ? 4 : 2;
    const size_t pageb = (size_t)p.S * p.D * ES;
    const size_t smem = (size_t)(3 * MAXG * p.D + 16) * 4 +
                        (size_t)kGBWarps * (4 * pageb + 2 * MAXG * p.S * 4);
    if (smem > 220 * 1024) return PT_ERR_UNSUPPORTED;
    static size_t configured = 0;
    if (smem > configured) {
        PT_CUDA_TRY(cudaFuncSetAttribute(k_gated_bwd<DT, MAXG, DJ>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    // one wave: every resident CTA slot (warps stride over the unit's pages), at least one
    // page per warp
    int dev = 0, nsm = 0, per_sm = 0;
    PT_CUDA_TRY(cudaGetDevice(&dev));
    PT_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    PT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gated_bwd<DT, MAXG, DJ>,
                                                              kGBWarps * 32, smem));
    if (per_sm < 1) per_sm = 1;
    int gx = nsm * per_sm / U;
    const int pages = p.Pmax;
    const int maxgx = (pages + kGBWarps - 1) / kGBWarps;
    if (gx > maxgx) gx = maxgx;
    if (gx < 1) gx = 1;
    k_gated_bwd<DT, MAXG, DJ><<<dim3(gx, U), kGBWarps * 32, smem, st>>>(p);
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}

extern "C" int pt_gated_attend_bwd(const void *q, int q_dtype, const void *k_pool,
                                   const void *v_pool, int kv_dtype, const int32_t *page_table,
                                   const int32_t *seq_len, const float *gates, const float *out,
                                   const float *lse, const float *dout, int U, int G, int D,
                                   int S, int Pmax, float scale, float *dq, float *dk_pool,
                                   float *dv_pool, float *dgates, void *stream) {
    if (!q || !k_pool || !v_pool || !page_table || !seq_len || !gates || !out || !lse || !dout ||
        !dq || !dk_pool || !dv_pool || !dgates || U < 0 || G < 1 || D < 1 || S < 1 || Pmax < 1)
        return PT_ERR_INVALID;
    if (G > 8 || D > 256 || S > 64 || D % 8 || (S < 32 && 32 % S)) return PT_ERR_UNSUPPORTED;
    if (U == 0) return PT_OK;
    GatedBwdParams p{q, k_pool, v_pool, page_table, seq_len, gates, out, lse, dout, dq, dk_pool,
                     dv_pool, dgates, q_dtype, kv_dtype, G, D, S, Pmax, scale};
    cudaStream_t st = (cudaStream_t)stream;
    const int dj = (D + 31) / 32;
#define PT_GB(DT_, DJ_) \
    if (kv_dtype == DT_ && dj == DJ_) \
        return G <= 4 ? launch_gbwd<DT_, 4, DJ_>(p, U, st) : launch_gbwd<DT_, 8, DJ_>(p, U, st);
    PT_GB(PT_F32, 1) PT_GB(PT_F32, 2) PT_GB(PT_F32, 4) PT_GB(PT_F32, 8)
    PT_GB(PT_BF16, 1) PT_GB(PT_BF16, 2) PT_GB(PT_BF16, 4) PT_GB(PT_BF16, 8)
#undef PT_GB
    return PT_ERR_UNSUPPORTED;
}

// ---------------------------------------------------------------------------
// Soft-mode forward prologue (softmask.py:108-176): every gate of a live page must lie in
// (0, 1] -- bad = (g <= 0) | (g > 1), NaN passes as in the reference's numpy check -- and the
// attention bias is f32(log(g)) for every (unit, page) slot (the float64 log rounded once,
// as torch.log(g64).to(float32)).  One pass, one flag word for the caller to read.
// ---------------------------------------------------------------------------
__global__ void k_gate_bias(const double *__restrict__ gates, const int32_t *__restrict__ seq_len,
                            int U, int S, int Pmax, float *__restrict__ bias, int32_t *__restrict__ flag) {
    const int64_t total = (int64_t)U * Pmax;
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int u = (int)(i / Pmax), pg = (int)(i - (int64_t)u * Pmax);
        const double g = gates[i];
        const int P = (seq_len[u] + S - 1) / S;
        bad |= (pg < P) && ((g <= 0.0) || (g > 1.0));
        bias[i] = __double2float_rn(log(g));
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

extern "C" int pt_gate_bias(const double *gates, const int32_t *seq_len, int U, int S, int Pmax,
                            float *bias, int32_t *flag, void *stream) {
    if (!gates || !seq_len || !bias || !flag || U < 0 || S < 1 || Pmax < 0) return PT_ERR_INVALID;
    if ((int64_t)U * Pmax == 0) return PT_OK;
    cudaStream_t st = (cudaStream_t)stream;
    PT_CUDA_TRY(cudaMemsetAsync(flag, 0, sizeof(int32_t), st));
    int64_t blocks = ((int64_t)U * Pmax + 255) / 256;
    if (blocks > pt_num_sms() * 8) blocks = pt_num_sms() * 8;
    k_gate_bias<<<(int)blocks, 256, 0, st>>>(gates, seq_len, U, S, Pmax, bias, flag);
    PT_CUDA_TRY(cudaGetLastError());
    return PT_OK;
}
