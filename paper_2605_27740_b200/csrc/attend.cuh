// attend.cuh -- K4: split-KV paged decode attention over the selected pages.
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
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>
#include <cuda_bf16.h>

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

// Combine the per-warp partials (macc [NW][GP][D], mml [NW][GP][2] in shared memory) of
// this CTA; write the result (single split) or the split partial + ticket merge.
static __device__ __noinline__ void cta_finish(const AttnParams &prm, const float *macc, const float *mml,
                                        int NW, int GP, int64_t u, int s, int nsplit_u) {
    const int D = prm.D, G = prm.G;
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
    // the split weights once per CTA (all (m, l) pairs in one parallel round), then every
    // (head, dim) sums its splits with the loads issued 8 at a time -- no chain of
    // dependent L2 round trips per split
    __shared__ float sw[kAttnMaxSplits * 8];   // exp2(m_w - m_max) per (split, head)
    __shared__ float sinv[8], slse[8];
    for (int i = threadIdx.x; i < nsplit_u * G; i += blockDim.x)
        sw[i] = __ldcg(&wml[((u * prm.maxs + i / G) * G + i % G) * 2]);
    __syncthreads();
    if (threadIdx.x < G) {
        const int g = threadIdx.x;
        float mt = -INFINITY;
        for (int w = 0; w < nsplit_u; w++) mt = fmaxf(mt, sw[w * G + g]);
        const float mu = mt == -INFINITY ? 0.f : mt;
        float lt = 0.f;
        for (int w = 0; w < nsplit_u; w++) {
            const float f = exp2f(sw[w * G + g] - mu);
            lt += __ldcg(&wml[((u * prm.maxs + w) * G + g) * 2 + 1]) * f;
            sw[w * G + g] = f;
        }
        sinv[g] = 1.f / lt;
        slse[g] = (mt + log2f(lt)) * kLn2;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
        const int g = i / D, d = i % D;
        float a = 0.f;
        for (int w0 = 0; w0 < nsplit_u; w0 += 8) {
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; j++)
                v[j] = w0 + j < nsplit_u
                           ? __ldcg(&wacc[((u * prm.maxs + w0 + j) * G + g) * (int64_t)D + d])
                           : 0.f;
#pragma unroll
            for (int j = 0; j < 8; j++)
                if (w0 + j < nsplit_u) a += v[j] * sw[(w0 + j) * G + g];
        }
        prm.out[(u * G + g) * (int64_t)D + d] = a * sinv[g];
        if (d == 0) prm.lse[u * G + g] = slse[g];
    }
    if (threadIdx.x == 0) prm.tickets[u] = 0;
}

template <int DT, int GP, int DPL>
__global__ void __launch_bounds__(128) k_attend(const AttnParams prm) {
    constexpr int E = DT == PT_F32 ? 4 : 2;
    constexpr int TB = 32 / GP;  // tokens per sub-block
    extern __shared__ __align__(1024) char smem[];
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
    cta_finish(prm, macc, mml, NW, GP, u, s, nsplit_u);
}


// ===========================================================================
// Tensor-core variant for bf16 KV (mma.sync m16n8k16, f32 accumulate).
//
// A page of S = 16*MT tokens arrives by TMA tensor copies (cp.async.bulk.tensor.2d,
// SASS UTMALDG) in 64-column boxes with the 128-byte swizzle, so ldmatrix reads are
// bank-conflict free.  Per 16-token tile:
//   QK :  S[16 t x 8 g]  = K[16 t x D] . q^T[D x 8 g]      (D/16 MMAs; G <= 8 heads as N)
//   softmax on the C fragment (lane holds 2 tokens x 2 heads); P packed to bf16 and
//   transposed into the B-operand layout with movmatrix (no shared-memory round trip)
//   PV :  O^T[D x 8 g] += V^T[D x 16 t] . P[16 t x 8 g]   (D/16 MMAs, V^T via ldmatrix.trans)
// The accumulator's column (head) ownership equals the softmax state's, so the
// running-max rescale is lane-local.  G <= 8 pads N to 8 (a GQA group of 4 fills half
// the tile); HBM, not the tensor pipe, bounds this kernel.
// ===========================================================================
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ uint32_t movm_t(uint32_t a) {
    uint32_t d;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
    return d;
}
__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&v);
}
__device__ __forceinline__ void tma_load_2d(void *smem_dst, const CUtensorMap *tm, int c0, int c1,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// the same with an L2 cache policy (evict-first for pages read once per step: the stream
// then does not push the step's small re-read state -- keys, tables, kernel code -- out of L2)
__device__ __forceinline__ void tma_load_2d_hint(void *smem_dst, const CUtensorMap *tm, int c0, int c1,
                                                 uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, "
        "{%2, %3}], [%4], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// byte offset of element (t, d) inside a staged page: 64-column boxes of S rows x 128 B,
// 16-byte chunk index XOR (row & 7) (CU_TENSOR_MAP_SWIZZLE_128B)
__device__ __forceinline__ uint32_t swz(int t, int chunk16, int S) {
    const int box = chunk16 >> 3, c = chunk16 & 7;
    return (uint32_t)(box * S * 128 + t * 128 + ((c ^ (t & 7)) << 4));
}

constexpr int kMmaGP = 8;  // heads padded to the MMA N

// [mbarriers][per-warp page-id lists][pad to 1024][stage rings]
__host__ __device__ __forceinline__ int attn_mma_maxc(int pps, int NW) { return (pps + NW - 1) / NW; }
__host__ __device__ __forceinline__ size_t attn_mma_hdr_bytes(int NW, int nstage, int pps) {
    const size_t b = (size_t)NW * nstage * 8 + (size_t)NW * attn_mma_maxc(pps, NW) * 4;
    return (b + 1023) & ~(size_t)1023;
}

template <int D, int MT>
__global__ void __launch_bounds__(128) k_attend_mma(const __grid_constant__ CUtensorMap tmk,
                                                    const __grid_constant__ CUtensorMap tmv,
                                                    const AttnParams prm) {
    constexpr int S = 16 * MT;
    constexpr int KS = D / 16;                   // k-steps of QK == m-tiles of PV
    constexpr uint32_t PAGE_BYTES = S * D * 2;   // one tensor (K or V) of one page
    constexpr uint32_t STAGE_BYTES = 2 * PAGE_BYTES;
    extern __shared__ __align__(1024) char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const int64_t u = blockIdx.y;
    const int s = blockIdx.x;
    const int G = prm.G;
    const int n = prm.seq_len[u];
    const int P = (n + S - 1) / S;
    const int ns = prm.n_sel ? prm.n_sel[u] : P;
    const int first = s * prm.pps;
    if (first >= ns) return;
    const int last = min(first + prm.pps, ns);
    const int nsplit_u = (ns + prm.pps - 1) / prm.pps;
    const int tail_pid = prm.page_table[u * prm.Pmax + P - 1];
    const int tail_rows = n - (P - 1) * S;
    const int nstage = prm.nstage;

    uint64_t *bars = reinterpret_cast<uint64_t *>(smem) + warp * nstage;
    const int maxc = attn_mma_maxc(prm.pps, NW);
    int32_t *my_pids = reinterpret_cast<int32_t *>(smem + (size_t)NW * nstage * 8) + warp * maxc;
    char *ring = smem + attn_mma_hdr_bytes(NW, nstage, prm.pps);
    char *my_stages = ring + (size_t)warp * nstage * STAGE_BYTES;
    const int rem = last - first - warp;
    const int my_count = rem > 0 ? (rem + NW - 1) / NW : 0;
    const int32_t *selu = prm.sel + u * (int64_t)prm.sel_stride;
    // this warp's page ids, fetched once (no dependent global load on the TMA issue path)
    for (int i = lane; i < my_count; i += 32) my_pids[i] = selu[first + warp + i * NW];
    __syncwarp();

    auto issue = [&](int i) {
        const int pid = my_pids[i];
        const int st = i % nstage;
        char *ks = my_stages + (size_t)st * STAGE_BYTES;
        mbar_arrive_expect_tx(&bars[st], STAGE_BYTES);
#pragma unroll
        for (int b = 0; b < D / 64; b++) {
            tma_load_2d(ks + b * S * 128, &tmk, b * 64, pid * S, &bars[st]);
            tma_load_2d(ks + PAGE_BYTES + b * S * 128, &tmv, b * 64, pid * S, &bars[st]);
        }
    };
    if (lane == 0) {
        for (int i = 0; i < nstage; i++) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    if (lane == 0)
        for (int i = 0; i < min(nstage, my_count); i++) issue(i);

    // q as the B operand of QK: lane holds q[g = lane/4][d = 16ks + 2(lane%4) + {0,1} (+8)]
    const int gq = lane >> 2;
    uint32_t qb[KS][2];
#pragma unroll
    for (int ks = 0; ks < KS; ks++) {
        const int d0 = ks * 16 + 2 * (lane & 3);
        uint32_t b0 = 0, b1 = 0;
        if (gq < G) {
            const int64_t row = (u * G + gq) * (int64_t)D;
            if (prm.q_dtype == PT_BF16) {  // d0 is even: one 32-bit load per bf16 pair
                const uint32_t *qp =
                    reinterpret_cast<const uint32_t *>(static_cast<const uint16_t *>(prm.q) + row);
                b0 = __ldg(qp + (d0 >> 1));
                b1 = __ldg(qp + ((d0 + 8) >> 1));
            } else {
                const float *qp = static_cast<const float *>(prm.q) + row;
                b0 = pack_bf16(qp[d0], qp[d0 + 1]);
                b1 = pack_bf16(qp[d0 + 8], qp[d0 + 9]);
            }
        }
        qb[ks][0] = b0;
        qb[ks][1] = b1;
    }
    const float qscale = prm.scale * kLog2e;
    float acc[KS][4];
#pragma unroll
    for (int i = 0; i < KS; i++) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
    const int r8 = lane & 7, mat = lane >> 3;

    for (int i = 0; i < my_count; i++) {
        const int st = i % nstage;
        const int j = first + warp + i * NW;
        const int pid = my_pids[i];
        const int rows = (pid == tail_pid) ? tail_rows : S;
        const float b2 = prm.bias ? prm.bias[u * prm.sel_stride + j] * kLog2e : 0.f;
        mbar_wait(&bars[st], (uint32_t)((i / nstage) & 1));
        const uint32_t kbase = smem_u32(my_stages + (size_t)st * STAGE_BYTES);
        const uint32_t vbase = kbase + PAGE_BYTES;
#pragma unroll
        for (int mt = 0; mt < MT; mt++) {
            if (mt * 16 >= rows) break;
            float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int ks = 0; ks < KS; ks++) {
                uint32_t a[4];
                // a0: t 0-7 / d lo, a1: t 8-15 / d lo, a2: t 0-7 / d hi, a3: t 8-15 / d hi
                const int t = mt * 16 + r8 + ((mat & 1) << 3);
                ldsm_x4(kbase + swz(t, ks * 2 + (mat >> 1), S), a);
                mma_bf16(sc, a, qb[ks][0], qb[ks][1]);
            }
            const int t0 = mt * 16 + (lane >> 2);
            const bool v0 = t0 < rows, v1 = t0 + 8 < rows;
            sc[0] = v0 ? fmaf(sc[0], qscale, b2) : -INFINITY;
            sc[1] = v0 ? fmaf(sc[1], qscale, b2) : -INFINITY;
            sc[2] = v1 ? fmaf(sc[2], qscale, b2) : -INFINITY;
            sc[3] = v1 ? fmaf(sc[3], qscale, b2) : -INFINITY;
            float p[4], carry[2];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                float mx = fmaxf(sc[h], sc[h + 2]);
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
                const float m_new = fmaxf(m_run[h], mx);
                carry[h] = exp2f(m_run[h] - m_new);
                p[h] = exp2f(sc[h] - m_new);
                p[h + 2] = exp2f(sc[h + 2] - m_new);
                float ls = p[h] + p[h + 2];
                ls += __shfl_xor_sync(0xffffffffu, ls, 4);
                ls += __shfl_xor_sync(0xffffffffu, ls, 8);
                ls += __shfl_xor_sync(0xffffffffu, ls, 16);
                l_run[h] = l_run[h] * carry[h] + ls;
                m_run[h] = m_new;
            }
            const uint32_t pb0 = movm_t(pack_bf16(p[0], p[1]));
            const uint32_t pb1 = movm_t(pack_bf16(p[2], p[3]));
#pragma unroll
            for (int dm = 0; dm < KS; dm++) {
                acc[dm][0] *= carry[0];
                acc[dm][1] *= carry[1];
                acc[dm][2] *= carry[0];
                acc[dm][3] *= carry[1];
                uint32_t a[4];
                // V^T fragments: a0 t 0-7/d lo, a1 t 0-7/d hi, a2 t 8-15/d lo, a3 t 8-15/d hi
                const int t = mt * 16 + r8 + ((mat >> 1) << 3);
                ldsm_x4_t(vbase + swz(t, dm * 2 + (mat & 1), S), a);
                mma_bf16(acc[dm], a, pb0, pb1);
            }
        }
        __syncwarp();
        if (lane == 0 && i + nstage < my_count) issue(i + nstage);
    }

    // ---- per-warp partials to shared memory, then the common CTA/split merge ----
    __syncthreads();
    float *macc = reinterpret_cast<float *>(ring);             // [NW][8][D]
    float *mml = macc + (size_t)NW * kMmaGP * D;                // [NW][8][2]
    const int g0 = 2 * (lane & 3);
#pragma unroll
    for (int dm = 0; dm < KS; dm++) {
        const int d = dm * 16 + (lane >> 2);
        macc[((size_t)warp * kMmaGP + g0) * D + d] = acc[dm][0];
        macc[((size_t)warp * kMmaGP + g0 + 1) * D + d] = acc[dm][1];
        macc[((size_t)warp * kMmaGP + g0) * D + d + 8] = acc[dm][2];
        macc[((size_t)warp * kMmaGP + g0 + 1) * D + d + 8] = acc[dm][3];
    }
    if (lane < 4) {
        mml[(warp * kMmaGP + g0) * 2 + 0] = m_run[0];
        mml[(warp * kMmaGP + g0) * 2 + 1] = l_run[0];
        mml[(warp * kMmaGP + g0 + 1) * 2 + 0] = m_run[1];
        mml[(warp * kMmaGP + g0 + 1) * 2 + 1] = l_run[1];
    }
    __syncthreads();
    cta_finish(prm, macc, mml, NW, kMmaGP, u, s, nsplit_u);
}


// ===========================================================================
// Streaming variant of the tensor-core kernel (the sparse decode path).
//
// The short per-unit page lists of a sparse step (k = 128 pages) make per-CTA set-up,
// merge and wave-quantisation costs dominate a grid of (split, unit) CTAs.  Here the
// selected pages of ALL units are concatenated (unit-major, offsets = prefix sum of n_sel)
// and cut into W equal contiguous ranges, one per warp of a persistent grid (one wave).
// Each warp streams its range through ONE continuous TMA ring -- the producer lane runs
// `nstage` pages ahead across unit boundaries, page ids come from a per-warp list staged
// in shared memory -- and emits one result per unit segment it touches: the final output
// when it owns the whole unit, else a partial (m, l, acc) into slot (warp - first warp of
// the unit); the last partial of a unit to land (atomic ticket, self-resetting) merges them.
// ===========================================================================
struct StreamParams {
    const void *q;
    const int32_t *sel;
    const int32_t *n_sel;
    const int32_t *page_table;
    const int32_t *seq_len;
    const float *bias;
    float *out, *lse, *ws;
    int32_t *tickets;
    int q_dtype, sel_stride, U, G, Pmax, L, maxparts, nstage;
    float scale;
};

template <int D>
__device__ __forceinline__ void load_qfrag(const StreamParams &p, int u, int lane,
                                           uint32_t (&qb)[D / 16][2]) {
    const int gq = lane >> 2;
#pragma unroll
    for (int ks = 0; ks < D / 16; ks++) {
        const int d0 = ks * 16 + 2 * (lane & 3);
        uint32_t b0 = 0, b1 = 0;
        if (gq < p.G) {
            const int64_t row = ((int64_t)u * p.G + gq) * D;
            if (p.q_dtype == PT_BF16) {
                const uint32_t *qp =
                    reinterpret_cast<const uint32_t *>(static_cast<const uint16_t *>(p.q) + row);
                b0 = __ldg(qp + (d0 >> 1));
                b1 = __ldg(qp + ((d0 + 8) >> 1));
            } else {
                const float *qp = static_cast<const float *>(p.q) + row;
                b0 = pack_bf16(qp[d0], qp[d0 + 1]);
                b1 = pack_bf16(qp[d0 + 8], qp[d0 + 9]);
            }
        }
        qb[ks][0] = b0;
        qb[ks][1] = b1;
    }
}

// One staged page through QK -> online softmax -> PV (the k_attend_mma inner loop).
template <int D, int MT>
__device__ __forceinline__ void mma_page(uint32_t kbase, uint32_t vbase, int rows, float b2,
                                         float qscale, const uint32_t (&qb)[D / 16][2],
                                         float (&acc)[D / 16][4], float (&m_run)[2],
                                         float (&l_run)[2], int lane) {
    constexpr int S = 16 * MT;
    constexpr int KS = D / 16;
    const int r8 = lane & 7, mat = lane >> 3;
#pragma unroll
    for (int mt = 0; mt < MT; mt++) {
        if (mt * 16 >= rows) break;
        float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ks = 0; ks < KS; ks++) {
            uint32_t a[4];
            const int t = mt * 16 + r8 + ((mat & 1) << 3);
            ldsm_x4(kbase + swz(t, ks * 2 + (mat >> 1), S), a);
            mma_bf16(sc, a, qb[ks][0], qb[ks][1]);
        }
        const int t0 = mt * 16 + (lane >> 2);
        const bool v0 = t0 < rows, v1 = t0 + 8 < rows;
        sc[0] = v0 ? fmaf(sc[0], qscale, b2) : -INFINITY;
        sc[1] = v0 ? fmaf(sc[1], qscale, b2) : -INFINITY;
        sc[2] = v1 ? fmaf(sc[2], qscale, b2) : -INFINITY;
        sc[3] = v1 ? fmaf(sc[3], qscale, b2) : -INFINITY;
        float p[4], carry[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            float mx = fmaxf(sc[h], sc[h + 2]);
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
            const float m_new = fmaxf(m_run[h], mx);
            carry[h] = exp2f(m_run[h] - m_new);
            p[h] = exp2f(sc[h] - m_new);
            p[h + 2] = exp2f(sc[h + 2] - m_new);
            float ls = p[h] + p[h + 2];
            ls += __shfl_xor_sync(0xffffffffu, ls, 4);
            ls += __shfl_xor_sync(0xffffffffu, ls, 8);
            ls += __shfl_xor_sync(0xffffffffu, ls, 16);
            l_run[h] = l_run[h] * carry[h] + ls;
            m_run[h] = m_new;
        }
        const uint32_t pb0 = movm_t(pack_bf16(p[0], p[1]));
        const uint32_t pb1 = movm_t(pack_bf16(p[2], p[3]));
#pragma unroll
        for (int dm = 0; dm < KS; dm++) {
            acc[dm][0] *= carry[0];
            acc[dm][1] *= carry[1];
            acc[dm][2] *= carry[0];
            acc[dm][3] *= carry[1];
            uint32_t a[4];
            const int t = mt * 16 + r8 + ((mat >> 1) << 3);
            ldsm_x4_t(vbase + swz(t, dm * 2 + (mat & 1), S), a);
            mma_bf16(acc[dm], a, pb0, pb1);
        }
    }
}


// smem: [unit offsets (U+1) | per-warp page lists (L ints) | mbarriers | pad] [rings]
__host__ __device__ __forceinline__ size_t attn_stream_hdr(int U, int NW, int L, int nstage) {
    const size_t b = (size_t)(U + 1) * 4 + (size_t)NW * L * 4 + (size_t)NW * nstage * 8 + 8;
    return (b + 1023) & ~(size_t)1023;
}

// merge the nparts partials of unit u (one warp).  All (m, l) pairs are fetched at once
// (lane w holds part w), the per-part scale factors come from warp reductions, and the
// accumulator loads are issued 8 parts at a time (lanes own d = lane + 32 i: coalesced).
template <int D>
__device__ __noinline__ void merge_unit(const StreamParams &p, int u, int nparts, int lane) {
    const float *wacc = p.ws;
    const float *wml = p.ws + (size_t)p.U * p.maxparts * p.G * D;
    constexpr int DI = D / 32;
    float mw[2][8], lw[2][8];
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int w = lane + 32 * h;
#pragma unroll
        for (int g = 0; g < 8; g++) {
            const bool ok = w < nparts && g < p.G;
            const int64_t sl = ((int64_t)u * p.maxparts + w) * p.G + g;
            mw[h][g] = ok ? __ldcg(&wml[sl * 2]) : -INFINITY;
            lw[h][g] = ok ? __ldcg(&wml[sl * 2 + 1]) : 0.f;
        }
    }
    for (int g = 0; g < p.G; g++) {
        float mt = fmaxf(mw[0][g], mw[1][g]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mt = fmaxf(mt, __shfl_xor_sync(0xffffffffu, mt, o));
        const float f0 = exp2f(mw[0][g] - mt), f1 = exp2f(mw[1][g] - mt);
        float lt = lw[0][g] * f0 + lw[1][g] * f1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lt += __shfl_xor_sync(0xffffffffu, lt, o);
        float a[DI];
#pragma unroll
        for (int i = 0; i < DI; i++) a[i] = 0.f;
        for (int w0 = 0; w0 < nparts; w0 += 8) {
            float v[8][DI];
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int w = w0 + j;
                const float *src = wacc + (((int64_t)u * p.maxparts + w) * p.G + g) * D + lane;
#pragma unroll
                for (int i = 0; i < DI; i++) v[j][i] = w < nparts ? __ldcg(src + 32 * i) : 0.f;
            }
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int w = w0 + j;
                const float fw = __shfl_sync(0xffffffffu, (w & 32) ? f1 : f0, w & 31);
#pragma unroll
                for (int i = 0; i < DI; i++) a[i] = fmaf(v[j][i], w < nparts ? fw : 0.f, a[i]);
            }
        }
        const float inv = 1.f / lt;
#pragma unroll
        for (int i = 0; i < DI; i++) p.out[((int64_t)u * p.G + g) * D + lane + 32 * i] = a[i] * inv;
        if (lane == 0) p.lse[u * p.G + g] = (mt + log2f(lt)) * kLn2;
    }
}

template <int D, int MT>
__global__ void __launch_bounds__(128) k_attend_stream(const __grid_constant__ CUtensorMap tmk,
                                                       const __grid_constant__ CUtensorMap tmv,
                                                       const StreamParams prm) {
    constexpr int S = 16 * MT;
    constexpr int KS = D / 16;
    constexpr uint32_t PAGE_BYTES = S * D * 2;
    constexpr uint32_t STAGE_BYTES = 2 * PAGE_BYTES;
    extern __shared__ __align__(1024) char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const int nstage = prm.nstage, U = prm.U, L = prm.L;
    const int gw = blockIdx.x * NW + warp;
    int *off = reinterpret_cast<int *>(smem);                        // [U + 1]
    int *plist = off + (U + 1) + warp * L;                           // this warp's page ids
    uint64_t *bars = reinterpret_cast<uint64_t *>(
                         smem + (((size_t)(U + 1) * 4 + (size_t)NW * L * 4 + 7) & ~(size_t)7)) +
                     warp * nstage;
    char *my_stages = smem + attn_stream_hdr(U, NW, L, nstage) + (size_t)warp * nstage * STAGE_BYTES;

    // exclusive prefix sum of n_sel (every CTA): one coalesced load round, then a
    // shared-memory scan by warp 0
    for (int i = threadIdx.x; i < U; i += blockDim.x) off[i] = prm.n_sel[i];
    if (lane == 0) {
        for (int i = 0; i < nstage; i++) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == 0) {
        int carry = 0;
        for (int base = 0; base < U; base += 32) {
            const int uu = base + lane;
            const int v = uu < U ? off[uu] : 0;
            int inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int x = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += x;
            }
            if (uu < U) off[uu] = carry + inc - v;
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) off[U] = carry;
    }
    __syncthreads();
    const int T = off[U];
    const int a = min(gw * L, T), b = min(a + L, T);
    if (a >= b) return;
    // first unit of the range: largest u with off[u] <= a
    int u = 0;
    {
        int lo = 0, hi = U - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (off[mid] <= a) lo = mid; else hi = mid - 1;
        }
        u = lo;
        while (u < U - 1 && off[u + 1] <= a) u++;
    }
    // stage this warp's page ids (positions a..b-1)
    {
        int uu = u;
        for (int i = a + lane; i < b; i += 32) {
            while (uu < U - 1 && off[uu + 1] <= i) uu++;
            plist[i - a] = prm.sel[(int64_t)uu * prm.sel_stride + (i - off[uu])];
        }
    }
    __syncwarp();

    const int n_pos = b - a;
    int prod_i = 0;
    int cons_i = 0;
    // producer: lane 0 keeps up to nstage pages in flight
    auto fill = [&]() {
        if (lane == 0) {
            while (prod_i < n_pos && prod_i < cons_i + nstage) {
                const int pid = plist[prod_i];
                const int st = prod_i % nstage;
                char *ks = my_stages + (size_t)st * STAGE_BYTES;
                mbar_arrive_expect_tx(&bars[st], STAGE_BYTES);
#pragma unroll
                for (int bb = 0; bb < D / 64; bb++) {
                    tma_load_2d(ks + bb * S * 128, &tmk, bb * 64, pid * S, &bars[st]);
                    tma_load_2d(ks + PAGE_BYTES + bb * S * 128, &tmv, bb * 64, pid * S, &bars[st]);
                }
                prod_i++;
            }
        }
    };
    fill();
    const float qscale = prm.scale * kLog2e;
    float *wacc = prm.ws;
    float *wml = prm.ws + (size_t)U * prm.maxparts * prm.G * D;
    __shared__ int last_flag[4];
    const int g0 = 2 * (lane & 3);
    uint32_t qb[KS][2];
    load_qfrag<D>(prm, u, lane, qb);
    // tail page of a unit: (physical id, rows); lane 0 loads, shuffled to the warp
    auto tail_of = [&](int uu, int &tpid, int &trows) {
        int n = 0, pid = -1;
        if (lane == 0) {
            n = prm.seq_len[uu];
            const int P = (n + S - 1) / S;
            pid = prm.page_table[(int64_t)uu * prm.Pmax + P - 1];
        }
        n = __shfl_sync(0xffffffffu, n, 0);
        tpid = __shfl_sync(0xffffffffu, pid, 0);
        trows = n - ((n + S - 1) / S - 1) * S;
    };
    int tail_pid, tail_rows;
    tail_of(u, tail_pid, tail_rows);
    int pos = a;
    while (pos < b) {
        // segment of unit u: [pos, seg_end)
        const int seg_end = min(b, off[u + 1]);
        // q and tail page of the next (non-empty) unit are fetched while this one computes
        uint32_t qn[KS][2];
        const bool more = seg_end < b;
        int nu = u + 1;
        while (nu < U - 1 && off[nu + 1] <= seg_end) nu++;
        int ntail_pid = -1, ntail_rows = 0;
        if (more) {
            load_qfrag<D>(prm, nu, lane, qn);
            tail_of(nu, ntail_pid, ntail_rows);
        }
        float acc[KS][4];
#pragma unroll
        for (int i = 0; i < KS; i++) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
        float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};
        for (; pos < seg_end; pos++) {
            const int st = cons_i % nstage;
            const int pid = plist[cons_i];
            const int rows = (pid == tail_pid) ? tail_rows : S;
            const float b2 =
                prm.bias ? prm.bias[(int64_t)u * prm.sel_stride + (pos - off[u])] * kLog2e : 0.f;
            mbar_wait(&bars[st], (uint32_t)((cons_i / nstage) & 1));
            const uint32_t kbase = smem_u32(my_stages + (size_t)st * STAGE_BYTES);
            mma_page<D, MT>(kbase, kbase + PAGE_BYTES, rows, b2, qscale, qb, acc, m_run, l_run, lane);
            __syncwarp();
            cons_i++;
            fill();
        }
        // ---- segment epilogue ----
        const int ustart = off[u], uend = off[u + 1];
        if (ustart >= a && uend <= b) {  // this warp owns the whole unit: final output
            const float inv0 = 1.f / l_run[0], inv1 = 1.f / l_run[1];
#pragma unroll
            for (int dm = 0; dm < KS; dm++) {
                const int d = dm * 16 + (lane >> 2);
                if (g0 < prm.G) {
                    prm.out[((int64_t)u * prm.G + g0) * D + d] = acc[dm][0] * inv0;
                    prm.out[((int64_t)u * prm.G + g0) * D + d + 8] = acc[dm][2] * inv0;
                }
                if (g0 + 1 < prm.G) {
                    prm.out[((int64_t)u * prm.G + g0 + 1) * D + d] = acc[dm][1] * inv1;
                    prm.out[((int64_t)u * prm.G + g0 + 1) * D + d + 8] = acc[dm][3] * inv1;
                }
            }
            if (lane < 4) {
                if (g0 < prm.G) prm.lse[u * prm.G + g0] = (m_run[0] + log2f(l_run[0])) * kLn2;
                if (g0 + 1 < prm.G) prm.lse[u * prm.G + g0 + 1] = (m_run[1] + log2f(l_run[1])) * kLn2;
            }
        } else {
            const int wfirst = ustart / L, wlast = (uend - 1) / L;
            const int nparts = wlast - wfirst + 1;
            const int64_t slot = (int64_t)u * prm.maxparts + (gw - wfirst);
#pragma unroll
            for (int dm = 0; dm < KS; dm++) {
                const int d = dm * 16 + (lane >> 2);
                if (g0 < prm.G) {
                    wacc[(slot * prm.G + g0) * D + d] = acc[dm][0];
                    wacc[(slot * prm.G + g0) * D + d + 8] = acc[dm][2];
                }
                if (g0 + 1 < prm.G) {
                    wacc[(slot * prm.G + g0 + 1) * D + d] = acc[dm][1];
                    wacc[(slot * prm.G + g0 + 1) * D + d + 8] = acc[dm][3];
                }
            }
            if (lane < 4) {
                if (g0 < prm.G) {
                    wml[(slot * prm.G + g0) * 2] = m_run[0];
                    wml[(slot * prm.G + g0) * 2 + 1] = l_run[0];
                }
                if (g0 + 1 < prm.G) {
                    wml[(slot * prm.G + g0 + 1) * 2] = m_run[1];
                    wml[(slot * prm.G + g0 + 1) * 2 + 1] = l_run[1];
                }
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                last_flag[warp] = (atomicAdd(&prm.tickets[u], 1) == nparts - 1);
            }
            __syncwarp();
            if (last_flag[warp]) {
                __threadfence();
                merge_unit<D>(prm, u, nparts, lane);
                if (lane == 0) prm.tickets[u] = 0;
            }
        }
        if (!more) break;
        u = nu;
        tail_pid = ntail_pid;
        tail_rows = ntail_rows;
#pragma unroll
        for (int ks = 0; ks < KS; ks++) { qb[ks][0] = qn[ks][0]; qb[ks][1] = qn[ks][1]; }
    }

}

}  // namespace pt
