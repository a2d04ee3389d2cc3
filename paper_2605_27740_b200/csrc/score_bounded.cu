// score_bounded.cu -- K2b: bounded page scoring over the bf16 mirror of the page means.
//
// The reference score of page p (scoring.py:108-124, _kernels_cy.pyx:19-43) is
//   s_p = max_g fl(dot_g + fl(fl(lam*||q_g||) * std_p)),   dot_g = sequential f32 sum of q_g . m_p
// over the f32 page means m_p, and the selection works on key_p = ordered(bf16_rne(s_p)).
// Streaming the f32 means costs P*D*4 bytes per unit -- twice SURVEY 8(d)'s model, which
// reads the means at the KV element size.  This kernel streams the bf16 mirror m~_p instead
// (half the bytes) and computes, on the tensor cores (mma.sync m16n8k16, bf16 x bf16 -> f32:
// products exact), dot~_g = q_g . m~_p.  With err_p = ||m~_p - m_p|| + slack (written by the
// stats kernels, common.cuh store_mirror) and qn_g >= ||q_g|| (pt_lam_norms), the reference
// dot lies in [dot~ - E, dot~ + E], E = qn_g * err_p, so with directed rounding
//   lo_p = max_g fl(RD(dot~_g - E) + off_g) <= s_p <= max_g fl(RU(dot~_g + E) + off_g) = hi_p
// (fl(x + off) is monotone in x).  bf16 rounding and the ordered encoding are monotone too,
// so klo_p = key(lo_p) <= key_p <= key(hi_p) = khi_p: both are written, and the selection
// (attend_fused.cu, bounded mode) recomputes the exact key -- from the f32 means, in the
// reference's order -- only for the pages whose interval is not a single key and reaches the
// cut.  The selected page set, kth and kplus1 are therefore those of the f32 reference.
//
// Structure: persistent grid (CTAs x 4 warps per SM); warp gw streams the contiguous range
// [gw T / W, (gw+1) T / W) of the concatenated 32-page tiles of all units through a private
// ring of NST stages, one stage = one tile (32 pages x D bf16 = one contiguous block of the
// page-interleaved mirror, fetched by one cp.async.bulk) plus its 32 stds and 32 errs; the
// unit's query rows + lam*||q|| + ||q|| ride on the first stage of a run.  Per tile: two
// 16-page MMA row blocks x D/16 k-steps, A fragments by ldmatrix straight from the stage
// (one 16-byte row = 8 dims of one page), B = the G <= 8 query heads (N = 8).
#include "attend.cuh"

namespace pt {

struct BoundedScoreParams {
    const uint16_t *q;       // bf16 [U*G][D]
    const float *lamnorm;    // [U][8] fl(lam * ||q_g||)
    const float *qnorm;      // [U][8] upper bounds of ||q_g||
    const uint16_t *mirror;  // bf16 mirror of the means, tiles [U][Pmax/32][D/8][32][8]
    const float *stds;       // [U][Pmax]
    const float *merr;       // [U][Pmax]
    const int32_t *seq_len;
    uint16_t *keys_lo, *keys_hi;  // [U][Pmax]
    uint16_t *tile_max;           // [U][Pmax/32]: max klo of each tile
    int U, S, Pmax;
    int prof;  // PT_SB_PROF=1: per-CTA %globaltimer stamps (entry, after the PDL wait, exit)
    // early mode (pt_score_bounded_step): no PDL wait for the append -- the lengths come from
    // the append's snapshot (+ the one row it appends), the tiles streamed before the append
    // has finished are every tile but the units' tail tiles, which each warp defers to the end
    // of its range; step_sync = {append: lengths snapshotted, append: stores visible, scorer
    // steps completed, scorer CTA ticket} (see pt_append_step)
    const int32_t *snap;
    int32_t *sync;
};

__device__ __forceinline__ int sb_ld_acquire(const int32_t *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int sb_ld_relaxed(const int32_t *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void sb_spin_until(const int32_t *p, int target) {
    while (sb_ld_acquire(p) < target) __nanosleep(64);
}

constexpr int kSBProfCtas = 2048;
__device__ unsigned long long g_sb_prof[kSBProfCtas * 4];
__device__ __forceinline__ unsigned long long sb_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

constexpr int kSBWarps = 4;
constexpr int kSBMaxUnits = 2048;  // tile prefix over units in shared memory

template <int G, int D, int NST>
struct SBCfg {
    static constexpr int TILE = 32 * D * 2;
    static constexpr int QB = G * D * 2;
    static constexpr int UHDR = (QB + 64 + 127) & ~127;  // q rows | lamnorm[8] | qnorm[8]
    static constexpr int NHU = NST + 1;
    static constexpr int THDR = 256;  // 32 stds | 32 errs
    static constexpr int NHDR = NST;
    static constexpr int PER_WARP = NST * TILE + NHU * UHDR + NHDR * THDR;
};

__host__ __device__ __forceinline__ size_t sb_hdr_bytes(int U) {
    const size_t ps = ((size_t)(2 * U + 1) * 4 + 15) & ~(size_t)15;  // tile prefix | pages
    return (ps + (size_t)kSBWarps * 8 * 8 + 127) & ~(size_t)127;
}

template <int G, int D, int NST>
__global__ void __launch_bounds__(kSBWarps * 32, 1) k_score_bounded(const BoundedScoreParams prm) {
    using C = SBCfg<G, D, NST>;
    constexpr int KS = D / 16;
    extern __shared__ __align__(1024) char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int S = prm.S, Pmax = prm.Pmax, U = prm.U;
    const int TPU = Pmax >> 5;
    const int W = gridDim.x * kSBWarps;
    const int gw = blockIdx.x * kSBWarps + warp;
    int *Tp = reinterpret_cast<int *>(smem);
    int *Pu = Tp + U + 1;  // pages per unit
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (((size_t)(2 * U + 1) * 4 + 15) & ~(size_t)15)) + warp * 8;
    char *ring = smem + sb_hdr_bytes(U) + (size_t)warp * C::PER_WARP;
    char *uhdrs = ring + NST * C::TILE;
    char *thdrs = uhdrs + C::NHU * C::UHDR;
    const bool prof = prm.prof && threadIdx.x == 0 && blockIdx.x < kSBProfCtas;
    if (prof) g_sb_prof[blockIdx.x * 4 + 0] = sb_gtimer();
    if (lane == 0) {
        for (int i = 0; i < NST; i++) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    const bool early = prm.sync != nullptr;
    __shared__ int s_my;
    int my = 0;
    if (!early) {
        pdl_wait();
        pdl_trigger();
    } else {
        // the append (the previous kernel) publishes the snapshot of the lengths right after
        // its own PDL wait: the predecessor's readers of the keys / norms are done by then
        if (threadIdx.x == 0) {
            const int m = sb_ld_acquire(prm.sync + 2) + 1;
            sb_spin_until(prm.sync, m);
            s_my = m;
        }
        __syncthreads();
        my = s_my;
        asm volatile("fence.proxy.async.global;" ::: "memory");  // bulk copies after the acquire
    }
    // unit length: early mode -- the append's snapshot + its row (the kernel reads nothing
    // the running append writes before step_sync[1])
    auto unit_len = [&](int uu) -> int {
        return early ? __ldcg(prm.snap + uu) + 1 : __ldcg(prm.seq_len + uu);
    };
    if (prof) g_sb_prof[blockIdx.x * 4 + 1] = sb_gtimer();
    {  // tile prefix over units (block scan)
        __shared__ int wsum[kSBWarps];
        int carry = 0;
        for (int b0 = 0; b0 < U; b0 += kSBWarps * 32) {
            const int uu = b0 + threadIdx.x;
            const int np = uu < U ? (unit_len(uu) + S - 1) / S : 0;
            if (uu < U) Pu[uu] = np;
            const int nt = (np + 31) >> 5;
            int inc = nt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) wsum[warp] = inc;
            __syncthreads();
            int pw = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < kSBWarps; w++) {
                if (w < warp) pw += wsum[w];
                tot += wsum[w];
            }
            if (uu < U) Tp[uu] = carry + pw + inc - nt;
            carry += tot;
            __syncthreads();
        }
        if (threadIdx.x == 0) Tp[U] = carry;
    }
    __syncthreads();
    struct Cur { int u, t, g, pass; };
    // static contiguous per-warp tile ranges: measured against dynamic chunk grabbing from a
    // global counter (2-8 tiles per grab: 178-205 vs 168.5 us/step at cfg3) and round-robin
    // chunks of 1-16 tiles (179-260 us/step) -- both finish units in tile order, both slower
    const int64_t T = Tp[U];
    const int64_t g0 = (int64_t)gw * T / W, g_end = (int64_t)(gw + 1) * T / W;
    // early mode: pass 0 = the range's tiles but the units' tail tiles (the append may still
    // be rewriting them), pass 1 = those tail tiles, after step_sync[1]
    Cur pc{U, 0, 0, 0};
    int u_first = U;
    if (g0 < g_end) {
        int lo = 0, hi = U;  // last unit with Tp[u] <= g0
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (Tp[mid] <= g0) lo = mid; else hi = mid;
        }
        pc = Cur{lo, (int)(g0 - Tp[lo]), (int)g0, 0};
        u_first = lo;
    }
    auto nt_of = [&](int uu) { return Tp[uu + 1] - Tp[uu]; };
    auto settle = [&](Cur &c) {  // forward to the next tile of this warp's visiting order
        for (;;) {
            if (c.u >= U) return;
            if (c.pass == 0) {
                if (c.g >= g_end) {
                    if (!early) { c.u = U; return; }
                    c.pass = 1;
                    c.u = u_first;
                    continue;
                }
                while (c.t >= nt_of(c.u)) { c.u++; c.t = 0; }
                if (!early || c.t != nt_of(c.u) - 1) return;
                c.g++;
                c.t++;
            } else {
                while (c.u < U && nt_of(c.u) == 0) c.u++;
                if (c.u >= U) return;
                const int64_t gt = (int64_t)Tp[c.u + 1] - 1;
                if (gt >= g_end) { c.u = U; return; }
                if (gt < g0) { c.u++; continue; }
                c.t = nt_of(c.u) - 1;
                c.g = (int)gt;
                return;
            }
        }
    };
    auto advance = [&](Cur &c) {
        if (c.pass == 0) { c.g++; c.t++; } else { c.u++; }
        settle(c);
    };
    settle(pc);
    Cur cc = pc;
    int issued = 0, p_run = -1, p_unit = -1;
    bool tails_ok = !early, triggered = !early;
    const uint64_t evict_first = l2_evict_first_policy();
    auto fill = [&](int consumed) {
        while (pc.u < U && issued < consumed + NST) {
            if (pc.pass == 1 && !tails_ok) {  // the append's stores are visible from here on
                if (lane == 0) sb_spin_until(prm.sync + 1, my);
                __syncwarp();
                asm volatile("fence.proxy.async.global;" ::: "memory");
                tails_ok = true;
                if (!triggered) { pdl_trigger(); triggered = true; }
            }
            const int slot = issued % NST;
            const bool new_run = pc.u != p_unit;
            if (new_run) { p_run++; p_unit = pc.u; }
            if (lane == 0) {
                const int64_t pg = (int64_t)pc.u * Pmax + (int64_t)pc.t * 32;
                mbar_arrive_expect_tx(&bars[slot], C::TILE + C::THDR + (new_run ? C::QB + 64 : 0));
                bulk_g2s_hint(ring + slot * C::TILE, prm.mirror + pg * D, C::TILE, &bars[slot], evict_first);
                char *th = thdrs + (issued % C::NHDR) * C::THDR;
                bulk_g2s_hint(th, prm.stds + pg, 128, &bars[slot], evict_first);
                bulk_g2s_hint(th + 128, prm.merr + pg, 128, &bars[slot], evict_first);
                if (new_run) {
                    char *h = uhdrs + (p_run % C::NHU) * C::UHDR;
                    bulk_g2s(h, prm.q + (int64_t)pc.u * G * D, C::QB, &bars[slot]);
                    bulk_g2s(h + C::QB, prm.lamnorm + (int64_t)pc.u * 8, 32, &bars[slot]);
                    bulk_g2s(h + C::QB + 32, prm.qnorm + (int64_t)pc.u * 8, 32, &bars[slot]);
                }
            }
            issued++;
            advance(pc);
        }
    };
    fill(0);
    const int h0 = 2 * (lane & 3), h1 = h0 + 1;
    const int gq = lane >> 2;
    uint32_t qb[KS][2];
    float ln0 = 0.f, ln1 = 0.f, qn0 = 0.f, qn1 = 0.f;
    int consumed = 0, c_run = -1, c_unit = -1, c_pages = 0;
    // ldmatrix row address of this lane within a tile: matrix mi = lane / 8 holds pages
    // (mi & 1) * 8 + lane % 8 of the 16-page block, dims 8 * (2 ks + (mi >> 1)) ..
    const int lrow = ((lane >> 3) & 1) * 8 + (lane & 7);
    const int lchk = lane >> 4;
    int pv = 0;  // early mode: step_sync[1] polled one tile ahead of its use (latency hidden)
    while (cc.u < U) {
        const int slot = consumed % NST;
        if (!triggered) {
            // the select+attend grid may launch (and read lengths / page table / pool rows
            // before its own wait) only once the append is complete
            if (pv >= my) { pdl_trigger(); triggered = true; }
            else pv = sb_ld_relaxed(prm.sync + 1);
        }
        mbar_wait(&bars[slot], (uint32_t)((consumed / NST) & 1));
        if (cc.u != c_unit) {  // a new run: the unit's query fragments and norms
            c_run++;
            c_unit = cc.u;
            c_pages = Pu[cc.u];
            const char *uh = uhdrs + (c_run % C::NHU) * C::UHDR;
            const uint16_t *qh = reinterpret_cast<const uint16_t *>(uh);
#pragma unroll
            for (int ks = 0; ks < KS; ks++) {
                const int d0 = ks * 16 + h0;
                qb[ks][0] = gq < G ? *reinterpret_cast<const uint32_t *>(qh + gq * D + d0) : 0u;
                qb[ks][1] = gq < G ? *reinterpret_cast<const uint32_t *>(qh + gq * D + d0 + 8) : 0u;
            }
            const float *lnp = reinterpret_cast<const float *>(uh + C::QB);
            ln0 = lnp[h0]; ln1 = lnp[h1]; qn0 = lnp[8 + h0]; qn1 = lnp[8 + h1];
        }
        float acc[2][4];
#pragma unroll
        for (int mb = 0; mb < 2; mb++) acc[mb][0] = acc[mb][1] = acc[mb][2] = acc[mb][3] = 0.f;
        const uint32_t sbase = smem_u32(ring + slot * C::TILE) + (uint32_t)(lchk * 512 + lrow * 16);
#pragma unroll
        for (int ks = 0; ks < KS; ks++) {
#pragma unroll
            for (int mb = 0; mb < 2; mb++) {
                uint32_t a[4];
                ldsm_x4(sbase + (uint32_t)(ks * 1024 + mb * 256), a);
                mma_bf16(acc[mb], a, qb[ks][0], qb[ks][1]);
            }
        }
        // epilogue: per (page, head) the interval of the reference score, max over heads
        const float *th = reinterpret_cast<const float *>(thdrs + (consumed % C::NHDR) * C::THDR);
        float lo[4], hi[4];  // pages gq, gq + 8, gq + 16, gq + 24 of the tile
#pragma unroll
        for (int mb = 0; mb < 2; mb++) {
#pragma unroll
            for (int half = 0; half < 2; half++) {
                const int pp = mb * 16 + half * 8 + gq;
                const float sd = th[pp], er = th[32 + pp];
                float l = -INFINITY, h = -INFINITY;
                if (h0 < G) {
                    const float c = acc[mb][2 * half], off = __fmul_rn(ln0, sd);
                    const float E = __fadd_ru(__fmul_ru(qn0, er), 1.17549435e-38f);
                    l = __fadd_rn(__fsub_rd(c, E), off);
                    h = __fadd_rn(__fadd_ru(c, E), off);
                }
                if (h1 < G) {
                    const float c = acc[mb][2 * half + 1], off = __fmul_rn(ln1, sd);
                    const float E = __fadd_ru(__fmul_ru(qn1, er), 1.17549435e-38f);
                    l = fmaxf(l, __fadd_rn(__fsub_rd(c, E), off));
                    h = fmaxf(h, __fadd_rn(__fadd_ru(c, E), off));
                }
                l = fmaxf(l, __shfl_xor_sync(0xffffffffu, l, 1));
                h = fmaxf(h, __shfl_xor_sync(0xffffffffu, h, 1));
                l = fmaxf(l, __shfl_xor_sync(0xffffffffu, l, 2));
                h = fmaxf(h, __shfl_xor_sync(0xffffffffu, h, 2));
                lo[mb * 2 + half] = l;
                hi[mb * 2 + half] = h;
            }
        }
        __syncwarp();  // stage + headers read: the slot may be refilled
        consumed++;
        fill(consumed);
        // lane (gq, j) writes page gq + 8 j: one 64-byte store per array per tile
        const int j = lane & 3;
        const float l = j == 0 ? lo[0] : j == 1 ? lo[1] : j == 2 ? lo[2] : lo[3];
        const float h = j == 0 ? hi[0] : j == 1 ? hi[1] : j == 2 ? hi[2] : hi[3];
        const int p = cc.t * 32 + gq + 8 * j;
        const int Pc = c_pages;
        const uint32_t klo = encode_ordered(f32_to_bf16_rne(l));
        const uint32_t khi = encode_ordered(f32_to_bf16_rne(h));
        if (p < Pc) {
            prm.keys_lo[(int64_t)cc.u * Pmax + p] = (uint16_t)klo;
            prm.keys_hi[(int64_t)cc.u * Pmax + p] = (uint16_t)khi;
        }
        const uint32_t m = __reduce_max_sync(0xffffffffu, p < Pc ? klo : 0u);
        if (lane == 0) prm.tile_max[(int64_t)cc.u * TPU + cc.t] = (uint16_t)m;
        advance(cc);
    }
    if (prm.prof) {
        __syncwarp();
        if (prof) g_sb_prof[blockIdx.x * 4 + 2] = sb_gtimer();  // warp 0's last tile done
    }
    if (early) {
        if (!triggered) {
            if (lane == 0) sb_spin_until(prm.sync + 1, my);
            __syncwarp();
            pdl_trigger();
        }
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(prm.sync + 3, 1) == (int)gridDim.x - 1) {
            // every CTA has read the step count: this scorer step is done
            atomicExch(prm.sync + 3, 0);
            __threadfence();
            atomicAdd(prm.sync + 2, 1);
        }
    }
}

template <int G, int D, int NST>
static int sb_launch(const BoundedScoreParams &sp, int ctas, cudaStream_t st) {
    using C = SBCfg<G, D, NST>;
    const size_t smem = sb_hdr_bytes(sp.U) + (size_t)kSBWarps * C::PER_WARP;
    while (ctas > 1 && (smem + 1024) * ctas > 227 * 1024) ctas--;
    if (smem > 227 * 1024) return PT_ERR_UNSUPPORTED;
    static size_t configured = 0;
    if (smem > configured) {
        PT_CUDA_TRY(cudaFuncSetAttribute(k_score_bounded<G, D, NST>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        configured = smem;
    }
    PT_CUDA_TRY(pt_launch(k_score_bounded<G, D, NST>, dim3(pt_num_sms() * ctas), dim3(kSBWarps * 32),
                          smem, st, sp));
    return PT_OK;
}

static int sb_env(const char *name, int dflt) {
    const char *e = getenv(name);
    return (e && *e) ? atoi(e) : dflt;
}

template <int G, int D>
static int sb_nst(const BoundedScoreParams &sp, cudaStream_t st) {
    // ring depth x CTAs per SM (PT_SB_NST / PT_SB_CTAS: tuning)
    // measured (tools/probe_score.py): D = 128: 2 stages x 2 CTAs (cfg3 82.5 us = 6.66 TB/s; deeper
    // rings drop to one CTA per SM: 141-150 us); D = 64: 2 stages x 5 CTAs (the cfg4 step 101.4
    // vs 107.5 us with 3 x 3, 103.2 with 2 x 4, 116.0 with 2 x 3: profiles/r02/score_d64_r02i.txt)
    const int nst = sb_env("PT_SB_NST", 2), ctas = sb_env("PT_SB_CTAS", D == 64 ? 5 : 2);
    switch (nst) {
        case 3: return sb_launch<G, D, 3>(sp, ctas, st);
        case 4: return sb_launch<G, D, 4>(sp, ctas, st);
        default: return sb_launch<G, D, 2>(sp, ctas, st);
    }
}

template <int D>
static int sb_g(const BoundedScoreParams &sp, int G, cudaStream_t st) {
    switch (G) {
        case 1: return sb_nst<1, D>(sp, st);
        case 2: return sb_nst<2, D>(sp, st);
        case 3: return sb_nst<3, D>(sp, st);
        case 4: return sb_nst<4, D>(sp, st);
        case 5: return sb_nst<5, D>(sp, st);
        case 6: return sb_nst<6, D>(sp, st);
        case 7: return sb_nst<7, D>(sp, st);
        case 8: return sb_nst<8, D>(sp, st);
        default: return PT_ERR_UNSUPPORTED;
    }
}

}  // namespace pt

using namespace pt;

// tuning aid: copy the stamps of the last PT_SB_PROF=1 launch (n <= 4 * 2048)
extern "C" int pt_debug_sb_prof(unsigned long long *host, int n) {
    if (!host || n < 0 || n > kSBProfCtas * 4) return PT_ERR_INVALID;
    PT_CUDA_TRY(cudaMemcpyFromSymbol(host, g_sb_prof, (size_t)n * 8));
    return PT_OK;
}

static int score_bounded_impl(const void *q, int q_dtype, const float *lamnorm, const float *qnorm,
                              const void *mirror, const float *stds, const int32_t *seq_len, int U_all,
                              int u0, int nu, int G, int D, int S, int Pmax, uint16_t *keys_lo,
                              uint16_t *keys_hi, uint16_t *tile_max, void *stream,
                              const int32_t *snap, int32_t *step_sync) {
    if (!q || !lamnorm || !qnorm || !mirror || !stds || !seq_len || !keys_lo || !keys_hi ||
        !tile_max || U_all < 0 || u0 < 0 || nu < 0 || u0 + nu > U_all || S < 1 || Pmax % 32 || G < 1)
        return PT_ERR_INVALID;
    const int U = nu;  // units [u0, u0 + nu) of a U_all-unit cache
    if (q_dtype != PT_BF16 || G > 8 || !(D == 64 || D == 128) || U > kSBMaxUnits ||
        (long long)U * (Pmax / 32) >= (1LL << 31))
        return PT_ERR_UNSUPPORTED;
    if (U == 0) return PT_OK;
    const MirrorView mv = mirror_view(mirror, U_all, Pmax, D);
    const int64_t o = u0;
    BoundedScoreParams sp{static_cast<const uint16_t *>(q) + o * G * D, lamnorm + o * 8, qnorm + o * 8,
                          mv.tiles + o * Pmax * D, stds + o * Pmax, mv.err + o * Pmax, seq_len + o,
                          keys_lo + o * Pmax, keys_hi + o * Pmax, tile_max + o * (Pmax / 32), U, S, Pmax,
                          sb_env("PT_SB_PROF", 0), snap ? snap + o : nullptr, step_sync};
    cudaStream_t st = (cudaStream_t)stream;
    return D == 128 ? sb_g<128>(sp, G, st) : sb_g<64>(sp, G, st);
}

extern "C" int pt_score_bounded(const void *q, int q_dtype, const float *lamnorm, const float *qnorm,
                                const void *mirror, const float *stds, const int32_t *seq_len, int U_all,
                                int u0, int nu, int G, int D, int S, int Pmax, uint16_t *keys_lo,
                                uint16_t *keys_hi, uint16_t *tile_max, void *stream) {
    return score_bounded_impl(q, q_dtype, lamnorm, qnorm, mirror, stds, seq_len, U_all, u0, nu, G, D,
                              S, Pmax, keys_lo, keys_hi, tile_max, stream, nullptr, nullptr);
}

// The decode step's scorer launched right after pt_append_step (same slot_scratch and
// step_sync, every unit): it streams every tile but the units' tail tiles while the append
// runs, then the tail tiles once the append's stores are visible.  PT_ERR_UNSUPPORTED exactly
// where pt_score_bounded is unsupported (then the caller must not have launched the append
// with step_sync).
extern "C" int pt_score_bounded_step(const void *q, int q_dtype, const float *lamnorm,
                                     const float *qnorm, const void *mirror, const float *stds,
                                     const int32_t *seq_len, int U, int G, int D, int S, int Pmax,
                                     uint16_t *keys_lo, uint16_t *keys_hi, uint16_t *tile_max,
                                     const int32_t *slot_scratch, int32_t *step_sync, void *stream) {
    if (!slot_scratch || !step_sync) return PT_ERR_INVALID;
    return score_bounded_impl(q, q_dtype, lamnorm, qnorm, mirror, stds, seq_len, U, 0, U, G, D, S,
                              Pmax, keys_lo, keys_hi, tile_max, stream, slot_scratch + U + 4, step_sync);
}
