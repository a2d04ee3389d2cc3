// score_stream.cuh -- K2 streaming scoring kernel (default path), fully specialised on
// (query dtype, stats dtype, G, D) so every index is a compile-time constant.
//
// Restates, per page p of unit u (see score.cu for the reference citations):
//   acc_g = fl(... fl(fl(0 + fl(q[g,0]*m[p,0])) + fl(q[g,1]*m[p,1])) ...)  (sequential d)
//   score = max_g fl(acc_g + fl(fl(lam*norm_g) * std_p));  key = ordered(bf16_rne(score))
// bit-identical to _kernels_cy.pyx:19-43 (non-FMA x86 build).
//
// Structure: a persistent grid (3 CTAs x 4 warps per SM); warp gw owns the 32-page tiles
// T = gw, gw + W, ... of the unit-major tile space, so units complete progressively.  Each
// warp streams its tiles through a private ring of NST = 3 stages; one stage = CPS 16-byte
// chunks of all 32 pages of a tile = one contiguous block of CPS*512 bytes in the
// page-interleaved means layout, fetched by a single cp.async.bulk (UBLKCP) on the stage's
// mbarrier.  The first stage of a tile also fetches the tile header (the unit's G query
// rows, lam*||q_g|| padded to 8, the 32 page stds) into one of NHDR header slots.  The query
// rows are widened once per tile into a head-pair-interleaved f32 buffer so each 16-byte
// broadcast read yields (q_g[d], q_g+1[d], q_g[d+1], q_g+1[d+1]); products of two heads are
// formed by one FMUL2 and accumulated by scalar FADDs (two roundings, as the reference --
// an f32x2 add after an f32x2 mul would be contracted to FFMA2 by ptxas).  With bf16 x bf16
// operands the products are exact in f32, so FFMA2 is bit-identical and used.
#pragma once
#include <stdlib.h>

#include "common.cuh"

namespace pt {

struct StreamScoreParams {
    const void *q;
    const float *lamnorm;  // [U][8]: fl(lam * norm_g), padded
    const void *means;
    const float *stds;
    const int32_t *seq_len;
    uint16_t *keys;
    float *scores;
    int U, S, Pmax;
    uint16_t *tile_max;  // [U][Pmax/32] max key of each 32-page tile, or null
    int contig;          // contiguous per-warp tile ranges (set by the launcher, see below)
};

// Tile order: contiguous per-warp ranges (one query-header fetch + widening per run of a
// unit's tiles) win for bf16 page means (cfg3: 104 vs 117 us -- half the bytes per element,
// so the per-tile overhead matters); the grid-stride order (all warps sweep one moving window
// of the means) wins for f32 (155 vs 160 us).  PT_SS_CONTIG=0/1 overrides (tuning).
static inline int ss_contig(int sdt) {
    const char *e = getenv("PT_SS_CONTIG");
    const int forced = e && *e ? atoi(e) : -1;
    return forced >= 0 ? forced : (sdt == PT_BF16 ? 1 : 0);
}

constexpr int kSSWarps = 4;
constexpr int kSSCtas = 3;  // per SM, at most
// CTAs per SM of the persistent grid (PT_SS_CTAS overrides, 1..3: tuning).  Measured: two
// (8 warps) beat three at long contexts (cfg3: 161 vs 169 us f32, 105 vs 107 us bf16 means),
// three win for short ones (8K context: 17 tiles per unit, per-tile header / cursor latency).
static inline int ss_ctas_per_sm(int Pmax) {
    const char *e = getenv("PT_SS_CTAS");
    const int forced = e && *e ? atoi(e) : 0;
    const int x = forced ? forced : ((Pmax >> 5) < 32 ? 3 : 2);
    return x < 1 ? 1 : (x > kSSCtas ? kSSCtas : x);
}
// ring shape per warp (stages x chunk): two CTAs per SM stream 2 x 8 KB stages (cfg3: 160
// us = 6.77 TB/s, vs 168 us for 4 x 4 KB and 172 us for 3 x 4 KB -- fewer, larger bulk
// copies for the same bytes in flight); three CTAs per SM (short contexts) keep 3 x 4 KB,
// the most that fits three
constexpr int kSSNstMax = 3;

__device__ __forceinline__ float2 ss_mul2(float m, float2 q) {
    unsigned long long r;
    const float2 mm = make_float2(m, m);
    asm("mul.rn.f32x2 %0, %1, %2;"
        : "=l"(r)
        : "l"(*reinterpret_cast<const unsigned long long *>(&mm)),
          "l"(*reinterpret_cast<const unsigned long long *>(&q)));
    return *reinterpret_cast<float2 *>(&r);
}
__device__ __forceinline__ float2 ss_fma2(float m, float2 q, float2 acc) {
    unsigned long long r;
    const float2 mm = make_float2(m, m);
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(r)
        : "l"(*reinterpret_cast<const unsigned long long *>(&mm)),
          "l"(*reinterpret_cast<const unsigned long long *>(&q)),
          "l"(*reinterpret_cast<const unsigned long long *>(&acc)));
    return *reinterpret_cast<float2 *>(&r);
}

template <int QDT, int SDT, int G, int D, int NST_, int CPSW>
struct SSCfg {
    static constexpr int NST = NST_;
    static constexpr int ES = SDT == PT_F32 ? 4 : 2;
    static constexpr int QES = QDT == PT_F32 ? 4 : 2;
    static constexpr int V = 16 / ES;            // means per 16-byte chunk
    static constexpr int NCH = D / V;            // chunks per page row
    static constexpr int CPS = NCH < CPSW ? NCH : CPSW;  // 16-byte chunks per stage
    static constexpr int SPT = NCH / CPS;        // stages per tile
    static constexpr int GP2 = (G + 1) / 2;      // head pairs
    static constexpr int STAGE = CPS * 512;
    // unit header (the unit's G query rows + lam*||q_g|| padded to 8): fetched once per run of
    // consecutive tiles of one unit.  The producer is at most NST stages ahead of the consumer,
    // i.e. at most (SPT - 1 + NST) / SPT tiles (and runs) ahead: one slot more than that
    static constexpr int UH_LN = (G * D * QES + 15) & ~15;
    static constexpr int UHDR = (UH_LN + 32 + 127) & ~127;
    static constexpr int NHU = (SPT - 1 + NST) / SPT + 1;
    // per-tile header (the 32 page stds), NHDR slots
    static constexpr int NHDR = NST / SPT + 2;
    static constexpr int QF = (GP2 * 2 * D * 4 + 127) & ~127;
    static constexpr int PER_WARP = NST * STAGE + NHU * UHDR + NHDR * 128 + QF;
    static constexpr uint32_t QCOPY = (uint32_t)((G * D * QES + 15) & ~15);
    static_assert(NCH % CPS == 0, "chunks per stage must divide the row");
};

// page counts of up to kSSPsMax units are cached in shared memory; beyond that (thousands
// of short sequences) they are read through L1 from seq_len
constexpr int kSSPsMax = 2048;

__host__ __device__ __forceinline__ size_t ss_hdr_bytes(int U) {
    if (U > kSSPsMax) U = kSSPsMax;
    const size_t ps = ((size_t)(U + 1) * 4 + 15) & ~(size_t)15;
    return (ps + (size_t)kSSWarps * kSSNstMax * 8 + 127) & ~(size_t)127;
}

template <int QDT, int SDT, int G, int D, int NST, int CPSW>
__global__ void __launch_bounds__(kSSWarps * 32, kSSCtas) k_score_stream(const StreamScoreParams prm) {
    using C = SSCfg<QDT, SDT, G, D, NST, CPSW>;
    constexpr bool kExactProduct = (QDT == PT_BF16 && SDT == PT_BF16);
    extern __shared__ __align__(128) char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int S = prm.S, Pmax = prm.Pmax, U = prm.U;
    const int TPU = Pmax >> 5;
    const int W = gridDim.x * kSSWarps;
    const int gw = blockIdx.x * kSSWarps + warp;
    // contiguous order (U <= kSSPsMax): Tp[u] = first tile of unit u in the concatenation of
    // every unit's ceil(P_u / 32) tiles, and warp gw streams the tiles [gw T / W, (gw+1) T / W)
    // (runs of one unit: its query header is fetched and widened once per run).  Grid-stride
    // order: tiles gw, gw + W, ... of the unit-major tile space (a header per tile).
    // one shared array: Tp (contiguous order) or the page counts Ps (grid-stride order, the
    // cursor's skip test reads them per tile)
    int *Tp = reinterpret_cast<int *>(smem);
    int *Ps = Tp;
    const bool contig = prm.contig && U <= kSSPsMax;
    const bool ps_smem = !contig && U <= kSSPsMax;
    uint64_t *bars =
        reinterpret_cast<uint64_t *>(smem + (((size_t)((U < kSSPsMax ? U : kSSPsMax) + 1) * 4 + 15) & ~(size_t)15)) +
        warp * kSSNstMax;
    char *wbase = smem + ss_hdr_bytes(U) + (size_t)warp * C::PER_WARP;
    char *ring = wbase;
    char *uhdrs = wbase + NST * C::STAGE;
    char *thdrs = uhdrs + C::NHU * C::UHDR;
    float *qf = reinterpret_cast<float *>(thdrs + C::NHDR * 128);
    if (lane == 0) {
        for (int i = 0; i < NST; i++) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    pdl_wait();
    // dependents may launch only once every CTA is past its own wait: an overlapped
    // select+attend then never runs beside a predecessor of this kernel (the append)
    pdl_trigger();
    if (contig) {  // tile prefix over units (block scan; U <= kSSPsMax)
        __shared__ int wsum[kSSWarps];
        int carry = 0;
        for (int b0 = 0; b0 < U; b0 += kSSWarps * 32) {
            const int uu = b0 + threadIdx.x;
            const int nt = uu < U ? ((prm.seq_len[uu] + S - 1) / S + 31) >> 5 : 0;
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
            for (int w = 0; w < kSSWarps; w++) {
                if (w < warp) pw += wsum[w];
                tot += wsum[w];
            }
            if (uu < U) Tp[uu] = carry + pw + inc - nt;
            carry += tot;
            __syncthreads();
        }
        if (threadIdx.x == 0) Tp[U] = carry;
    } else if (ps_smem) {
        for (int i = threadIdx.x; i < U; i += blockDim.x) Ps[i] = (prm.seq_len[i] + S - 1) / S;
    }
    __syncthreads();
    auto pages_of = [&](int uu) -> int {
        return ps_smem ? Ps[uu] : (__ldg(prm.seq_len + uu) + S - 1) / S;
    };
    // ---- tile cursor: (u, t) plus the position in this warp's range ----
    struct Cur { int u, t, g; };
    int64_t g_end = 0;
    auto first_cursor = [&]() -> Cur {
        Cur c{U, 0, 0};
        if (contig) {
            const int64_t T = Tp[U];
            const int64_t g0 = (int64_t)gw * T / W;
            g_end = (int64_t)(gw + 1) * T / W;
            if (g0 >= g_end) return c;
            int lo = 0, hi = U;  // last unit with Tp[u] <= g0 (it has tiles)
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (Tp[mid] <= g0) lo = mid; else hi = mid;
            }
            c.u = lo;
            c.t = (int)(g0 - Tp[lo]);
            c.g = (int)g0;
        } else {
            c.u = gw / TPU;
            c.t = gw - c.u * TPU;
            while (c.u < U) {  // settle: skip tiles past a unit's last page
                if (c.t >= TPU) { c.u += c.t / TPU; c.t %= TPU; }
                if (c.u >= U || c.t * 32 < pages_of(c.u)) break;
                c.t += W;
            }
        }
        return c;
    };
    auto advance = [&](Cur &c) {
        if (contig) {
            c.g++;
            if (c.g >= g_end) { c.u = U; return; }
            c.t++;
            while (c.t >= Tp[c.u + 1] - Tp[c.u]) { c.u++; c.t = 0; }  // c.g < T: a unit follows
        } else {
            c.t += W;
            while (c.u < U) {
                if (c.t >= TPU) { c.u += c.t / TPU; c.t %= TPU; }
                if (c.u >= U || c.t * 32 < pages_of(c.u)) break;
                c.t += W;
            }
        }
    };
    Cur pc = first_cursor();  // producer
    Cur cc = pc;              // consumer
    int p_part = 0, p_seq = 0, p_run = -1, p_unit = -1, issued = 0;
    const uint64_t evict_first = l2_evict_first_policy();
    auto fill = [&](int consumed) {
        while (pc.u < U && issued < consumed + NST) {
            const int slot = issued % NST;
            const bool new_run = p_part == 0 && pc.u != p_unit;
            if (new_run) { p_run++; p_unit = pc.u; }
            if (lane == 0) {
                const char *gsrc = static_cast<const char *>(prm.means) +
                                   ((int64_t)pc.u * Pmax + (int64_t)pc.t * 32) * D * C::ES;
                uint32_t tx = C::STAGE;
                if (p_part == 0) tx += 128 + (new_run ? C::QCOPY + 32 : 0);
                mbar_arrive_expect_tx(&bars[slot], tx);
                bulk_g2s_hint(ring + slot * C::STAGE, gsrc + p_part * C::STAGE, C::STAGE, &bars[slot],
                              evict_first);
                if (p_part == 0) {
                    bulk_g2s(thdrs + (p_seq % C::NHDR) * 128, prm.stds + (int64_t)pc.u * Pmax + pc.t * 32,
                             128, &bars[slot]);
                    if (new_run) {
                        char *h = uhdrs + (p_run % C::NHU) * C::UHDR;
                        bulk_g2s(h, static_cast<const char *>(prm.q) + (int64_t)pc.u * G * D * C::QES,
                                 C::QCOPY, &bars[slot]);
                        bulk_g2s(h + C::UH_LN, prm.lamnorm + (int64_t)pc.u * 8, 32, &bars[slot]);
                    }
                }
            }
            issued++;
            if (++p_part == C::SPT) {
                p_part = 0;
                p_seq++;
                advance(pc);
            }
        }
    };
    fill(0);
    int consumed = 0, seq = 0, c_run = -1, c_unit = -1;
    float2 *qf2 = reinterpret_cast<float2 *>(qf);
    while (cc.u < U) {
        const bool new_run = cc.u != c_unit;
        if (new_run) { c_run++; c_unit = cc.u; }
        const char *uh = uhdrs + (c_run % C::NHU) * C::UHDR;
        float2 acc[C::GP2];
#pragma unroll
        for (int g = 0; g < C::GP2; g++) acc[g] = make_float2(0.f, 0.f);
#pragma unroll
        for (int part = 0; part < C::SPT; part++) {
            const int slot = consumed % NST;
            mbar_wait(&bars[slot], (uint32_t)((consumed / NST) & 1));
            if (part == 0 && new_run) {  // widen the run's query rows, head-pair interleaved
#pragma unroll
                for (int pr = 0; pr < C::GP2; pr++) {
#pragma unroll
                    for (int d = lane; d < D; d += 32) {
                        float a, b = 0.f;
                        if constexpr (QDT == PT_F32) {
                            const float *qh = reinterpret_cast<const float *>(uh);
                            a = qh[(2 * pr) * D + d];
                            if (2 * pr + 1 < G) b = qh[(2 * pr + 1) * D + d];
                        } else {
                            const uint16_t *qh = reinterpret_cast<const uint16_t *>(uh);
                            a = bf16_bits_to_f32(qh[(2 * pr) * D + d]);
                            if (2 * pr + 1 < G) b = bf16_bits_to_f32(qh[(2 * pr + 1) * D + d]);
                        }
                        qf2[pr * D + d] = make_float2(a, b);
                    }
                }
                __syncwarp();
            }
            const char *mp = ring + slot * C::STAGE + lane * 16;
#pragma unroll
            for (int c = 0; c < C::CPS; c++) {
                const int cc = part * C::CPS + c;  // chunk index within the page row
                float m[C::V];
                if constexpr (SDT == PT_F32) {
                    const float4 v = *reinterpret_cast<const float4 *>(mp + c * 512);
                    m[0] = v.x; m[1] = v.y; m[2] = v.z; m[3] = v.w;
                } else {
                    const uint4 v = *reinterpret_cast<const uint4 *>(mp + c * 512);
                    m[0] = bf16_lo(v.x); m[1] = bf16_hi(v.x); m[2] = bf16_lo(v.y); m[3] = bf16_hi(v.y);
                    m[4] = bf16_lo(v.z); m[5] = bf16_hi(v.z); m[6] = bf16_lo(v.w); m[7] = bf16_hi(v.w);
                }
#pragma unroll
                for (int pr = 0; pr < C::GP2; pr++) {
#pragma unroll
                    for (int j = 0; j < C::V; j += 2) {
                        const float4 w =
                            *reinterpret_cast<const float4 *>(qf2 + pr * D + cc * C::V + j);
                        if constexpr (kExactProduct) {
                            acc[pr] = ss_fma2(m[j], make_float2(w.x, w.y), acc[pr]);
                            acc[pr] = ss_fma2(m[j + 1], make_float2(w.z, w.w), acc[pr]);
                        } else {
                            const float2 p0 = ss_mul2(m[j], make_float2(w.x, w.y));
                            acc[pr].x = __fadd_rn(acc[pr].x, p0.x);
                            acc[pr].y = __fadd_rn(acc[pr].y, p0.y);
                            const float2 p1 = ss_mul2(m[j + 1], make_float2(w.z, w.w));
                            acc[pr].x = __fadd_rn(acc[pr].x, p1.x);
                            acc[pr].y = __fadd_rn(acc[pr].y, p1.y);
                        }
                    }
                }
            }
            __syncwarp();  // stage fully read
            consumed++;
            if (part < C::SPT - 1) fill(consumed);
        }
        const float *ln = reinterpret_cast<const float *>(uh + C::UH_LN);
        const float sd = reinterpret_cast<const float *>(thdrs + (seq % C::NHDR) * 128)[lane];
        float best = -INFINITY;
#pragma unroll
        for (int g = 0; g < G; g++) {
            const float ag = (g & 1) ? acc[g >> 1].y : acc[g >> 1].x;
            const float a = __fadd_rn(ag, __fmul_rn(ln[g], sd));
            if (a > best) best = a;
        }
        const int p = cc.t * 32 + lane;
        const uint32_t key = encode_ordered(f32_to_bf16_rne(best));
        const int Pc = pages_of(cc.u);
        if (p < Pc) {
            prm.keys[(int64_t)cc.u * Pmax + p] = (uint16_t)key;
            if (prm.scores) prm.scores[(int64_t)cc.u * Pmax + p] = best;
        }
        if (prm.tile_max) {  // the tile's largest key (pads contribute key 0, the minimum)
            const uint32_t m = __reduce_max_sync(0xffffffffu, p < Pc ? key : 0u);
            if (lane == 0) prm.tile_max[(int64_t)cc.u * TPU + cc.t] = (uint16_t)m;
        }
        __syncwarp();  // header + qf reads done before their slots are refilled
        fill(consumed);
        seq++;
        advance(cc);
    }
}

}  // namespace pt
