#include <stdlib.h>
// capi.cu -- library identity + section A of pagetopk_b200.h: the reference's kernel
// backend contract (backend.py:14-58; _kernels_cy.pyx:19-172) served from HOST buffers.
// Each call stages its inputs into device memory, runs the same sm_100a kernels the
// batched device API uses, and copies the result back (synchronous, like the reference).
#include <mutex>
#include <vector>

#include "common.cuh"

namespace {

std::mutex g_mu;
cudaStream_t g_stream = nullptr;

int host_stream(cudaStream_t *out) {
    if (!g_stream) PT_CUDA_TRY(cudaStreamCreateWithFlags(&g_stream, cudaStreamNonBlocking));
    *out = g_stream;
    return PT_OK;
}

struct DevBuf {
    void *p = nullptr;
    cudaStream_t st;
    explicit DevBuf(cudaStream_t s) : st(s) {}
    cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes ? bytes : 16, st); }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

}  // namespace

bool pt_pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("PT_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

int pt_num_sms() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
    if (dev < 64 && cache[dev]) return cache[dev];
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    if (dev < 64) cache[dev] = n;
    return n;
}

extern "C" int pt_version(void) { return 200; }

extern "C" size_t pt_mirror_bytes(int U, int Pmax, int D) {
    if (U < 0 || Pmax < 0 || D < 1) return 0;
    return pt::mirror_bytes(U, Pmax, D);
}

extern "C" const char *pt_status_string(int status) {
    switch (status) {
        case PT_OK: return "ok";
        case PT_ERR_INVALID: return "invalid argument";
        case PT_ERR_UNSUPPORTED: return "shape outside the compiled envelope";
        case PT_ERR_K: return "k must be at least 1";
        case PT_ERR_EMPTY: return "no pages to select from";
        case PT_ERR_CAPACITY: return "page pool exhausted";
        default: break;
    }
    if (status >= PT_ERR_CUDA_BASE) return cudaGetErrorString((cudaError_t)(status - PT_ERR_CUDA_BASE));
    return "unknown status";
}

// _kernels_cy.pyx:19-43
extern "C" int pt_fused_scores_host(const float *queries, const float *norms, const float *means,
                                    const float *stds, int G, int64_t P, int D, float lam,
                                    float *out) {
    if (!queries || !norms || !means || !stds || !out || G < 1 || P < 0 || D < 1)
        return PT_ERR_INVALID;
    if (P == 0) return PT_OK;
    if (P > (int64_t)1 << 30) return PT_ERR_UNSUPPORTED;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t st;
    int rc = host_stream(&st);
    if (rc) return rc;
    const int Dp = (int)round_up(D, 4);  // zero padding leaves every partial sum unchanged
    const int Pmax = (int)round_up(P, 32);
    DevBuf dq(st), dn(st), dm(st), dmt(st), ds(st), dsl(st), dk(st), dsc(st);
    PT_CUDA_TRY(dq.alloc((size_t)G * Dp * 4));
    PT_CUDA_TRY(dn.alloc((size_t)G * 4));
    PT_CUDA_TRY(dm.alloc((size_t)P * Dp * 4));
    PT_CUDA_TRY(dmt.alloc((size_t)Pmax * Dp * 4));
    PT_CUDA_TRY(ds.alloc((size_t)Pmax * 4));
    PT_CUDA_TRY(dsl.alloc(4));
    PT_CUDA_TRY(dk.alloc((size_t)Pmax * 2));
    PT_CUDA_TRY(dsc.alloc((size_t)Pmax * 4));
    PT_CUDA_TRY(cudaMemsetAsync(dq.p, 0, (size_t)G * Dp * 4, st));
    PT_CUDA_TRY(cudaMemsetAsync(dm.p, 0, (size_t)P * Dp * 4, st));
    PT_CUDA_TRY(cudaMemsetAsync(dmt.p, 0, (size_t)Pmax * Dp * 4, st));
    PT_CUDA_TRY(cudaMemcpy2DAsync(dq.p, (size_t)Dp * 4, queries, (size_t)D * 4, (size_t)D * 4, G,
                                  cudaMemcpyHostToDevice, st));
    PT_CUDA_TRY(cudaMemcpy2DAsync(dm.p, (size_t)Dp * 4, means, (size_t)D * 4, (size_t)D * 4, P,
                                  cudaMemcpyHostToDevice, st));
    PT_CUDA_TRY(cudaMemcpyAsync(dn.p, norms, (size_t)G * 4, cudaMemcpyHostToDevice, st));
    PT_CUDA_TRY(cudaMemcpyAsync(ds.p, stds, (size_t)P * 4, cudaMemcpyHostToDevice, st));
    const int32_t n_tok = (int32_t)P;  // one row per "page": seq_len = P with S = 1
    PT_CUDA_TRY(cudaMemcpyAsync(dsl.p, &n_tok, 4, cudaMemcpyHostToDevice, st));
    rc = pt_tile_means((const float *)dm.p, 1, (int)P, Dp, Pmax, dmt.p, PT_F32, st);
    if (rc) return rc;
    rc = pt_score(dq.p, PT_F32, (const float *)dn.p, dmt.p, PT_F32, (const float *)ds.p,
                  (const int32_t *)dsl.p, 1, G, Dp, 1, Pmax, lam, (uint16_t *)dk.p, (float *)dsc.p, nullptr,
                  nullptr, st);
    if (rc) return rc;
    PT_CUDA_TRY(cudaMemcpyAsync(out, dsc.p, (size_t)P * 4, cudaMemcpyDeviceToHost, st));
    PT_CUDA_TRY(cudaStreamSynchronize(st));
    return PT_OK;
}

// _kernels_cy.pyx:46-126
extern "C" int pt_radix_select_desc_host(const uint16_t *keys, int64_t P, int64_t k,
                                         int64_t *ids_out, int *threshold_out, int *kplus1_out) {
    if (!keys || !ids_out || !threshold_out || !kplus1_out || P < 0) return PT_ERR_INVALID;
    if (k < 1) return PT_ERR_K;
    if (P == 0) return PT_ERR_EMPTY;
    if (k >= P || P > (int64_t)1 << 30) return PT_ERR_INVALID;  // reference precondition 1 <= k < P
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t st;
    int rc = host_stream(&st);
    if (rc) return rc;
    const int Pmax = (int)round_up(P, 32);
    std::vector<int32_t> ident((size_t)P);
    for (int64_t i = 0; i < P; i++) ident[(size_t)i] = (int32_t)i;
    DevBuf dk(st), dt(st), dsl(st), dsel(st), dlog(st), dmeta(st);
    PT_CUDA_TRY(dk.alloc((size_t)Pmax * 2));
    PT_CUDA_TRY(dt.alloc((size_t)Pmax * 4));
    PT_CUDA_TRY(dsl.alloc(4));
    PT_CUDA_TRY(dsel.alloc((size_t)k * 4));
    PT_CUDA_TRY(dlog.alloc((size_t)k * 4));
    PT_CUDA_TRY(dmeta.alloc(16));
    PT_CUDA_TRY(cudaMemcpyAsync(dk.p, keys, (size_t)P * 2, cudaMemcpyHostToDevice, st));
    PT_CUDA_TRY(cudaMemcpyAsync(dt.p, ident.data(), (size_t)P * 4, cudaMemcpyHostToDevice, st));
    const int32_t n_tok = (int32_t)P;
    PT_CUDA_TRY(cudaMemcpyAsync(dsl.p, &n_tok, 4, cudaMemcpyHostToDevice, st));
    int32_t *meta = (int32_t *)dmeta.p;  // n_sel, kth, kplus1
    rc = pt_topk((const uint16_t *)dk.p, (const int32_t *)dsl.p, (const int32_t *)dt.p, 1, 1, Pmax,
                 (int)k, (int32_t *)dsel.p, (int32_t *)dlog.p, meta, meta + 1, meta + 2, st);
    if (rc) return rc;
    std::vector<int32_t> ids((size_t)k);
    int32_t hmeta[3];
    PT_CUDA_TRY(cudaMemcpyAsync(ids.data(), dlog.p, (size_t)k * 4, cudaMemcpyDeviceToHost, st));
    PT_CUDA_TRY(cudaMemcpyAsync(hmeta, meta, 12, cudaMemcpyDeviceToHost, st));
    PT_CUDA_TRY(cudaStreamSynchronize(st));
    for (int64_t i = 0; i < k; i++) ids_out[i] = ids[(size_t)i];
    *threshold_out = hmeta[1];
    *kplus1_out = hmeta[2];
    return PT_OK;
}

// _kernels_cy.pyx:129-172.  The reference's online-softmax block is a numerical detail
// (results agree to f32 tolerance for any block, test_attention.py:67-76); the only
// semantic use of `block` is the per-block additive bias, so the contiguous rows are
// served as pages of S' rows with S' | block (bias of page p = block_bias[p*S'/block]).
extern "C" int pt_stream_attention_host(const float *q, const float *keys, const float *values,
                                        int64_t n, int D, float scale, int64_t block,
                                        const float *block_bias, float *out, double *lse) {
    if (!q || !keys || !values || !out || !lse || n < 1 || D < 1 || block < 1)
        return PT_ERR_INVALID;
    if (n > (int64_t)1 << 28) return PT_ERR_UNSUPPORTED;
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t st;
    int rc = host_stream(&st);
    if (rc) return rc;
    int Sp = 1;
    for (int c = 32; c >= 1; c--)
        if (block % c == 0) { Sp = c; break; }
    const int Dp = (int)round_up(D, 4);
    const int64_t npages = (n + Sp - 1) / Sp;
    const int Pmax = (int)round_up(npages, 32);
    std::vector<int32_t> ident((size_t)npages);
    for (int64_t i = 0; i < npages; i++) ident[(size_t)i] = (int32_t)i;
    std::vector<float> pbias;
    if (block_bias) {
        pbias.resize((size_t)npages);
        for (int64_t p = 0; p < npages; p++) pbias[(size_t)p] = block_bias[(p * Sp) / block];
    }
    DevBuf dq(st), dkp(st), dvp(st), dt(st), dsl(st), dns(st), db(st), dout(st), dlse(st),
        dws(st), dtk(st);
    const size_t pool = (size_t)npages * Sp * Dp * 4;
    PT_CUDA_TRY(dq.alloc((size_t)Dp * 4));
    PT_CUDA_TRY(dkp.alloc(pool));
    PT_CUDA_TRY(dvp.alloc(pool));
    PT_CUDA_TRY(dt.alloc((size_t)Pmax * 4));
    PT_CUDA_TRY(dsl.alloc(4));
    PT_CUDA_TRY(dns.alloc(4));
    PT_CUDA_TRY(db.alloc((size_t)npages * 4));
    PT_CUDA_TRY(dout.alloc((size_t)Dp * 4));
    PT_CUDA_TRY(dlse.alloc(4));
    const size_t wsb = pt_attend_workspace_bytes(1, 1, Dp, (int)npages);
    PT_CUDA_TRY(dws.alloc(wsb));
    PT_CUDA_TRY(dtk.alloc(4));
    PT_CUDA_TRY(cudaMemsetAsync(dtk.p, 0, 4, st));
    if (Dp != D) {
        PT_CUDA_TRY(cudaMemsetAsync(dq.p, 0, (size_t)Dp * 4, st));
        PT_CUDA_TRY(cudaMemsetAsync(dkp.p, 0, pool, st));
        PT_CUDA_TRY(cudaMemsetAsync(dvp.p, 0, pool, st));
    }
    PT_CUDA_TRY(cudaMemcpyAsync(dq.p, q, (size_t)D * 4, cudaMemcpyHostToDevice, st));
    PT_CUDA_TRY(cudaMemcpy2DAsync(dkp.p, (size_t)Dp * 4, keys, (size_t)D * 4, (size_t)D * 4, n,
                                  cudaMemcpyHostToDevice, st));
    PT_CUDA_TRY(cudaMemcpy2DAsync(dvp.p, (size_t)Dp * 4, values, (size_t)D * 4, (size_t)D * 4, n,
                                  cudaMemcpyHostToDevice, st));
    PT_CUDA_TRY(cudaMemcpyAsync(dt.p, ident.data(), (size_t)npages * 4, cudaMemcpyHostToDevice, st));
    const int32_t n_tok = (int32_t)n, n_pages = (int32_t)npages;
    PT_CUDA_TRY(cudaMemcpyAsync(dsl.p, &n_tok, 4, cudaMemcpyHostToDevice, st));
    PT_CUDA_TRY(cudaMemcpyAsync(dns.p, &n_pages, 4, cudaMemcpyHostToDevice, st));
    if (block_bias)
        PT_CUDA_TRY(cudaMemcpyAsync(db.p, pbias.data(), (size_t)npages * 4, cudaMemcpyHostToDevice, st));
    rc = pt_attend(dq.p, PT_F32, dkp.p, dvp.p, PT_F32, (int)npages, (const int32_t *)dt.p, (int)npages,
                   (const int32_t *)dns.p, (const int32_t *)dt.p, (const int32_t *)dsl.p, 1, 1, Dp,
                   Sp, Pmax, block_bias ? (const float *)db.p : nullptr, scale, (float *)dout.p,
                   (float *)dlse.p, dws.p, wsb, (int32_t *)dtk.p, 0, st);
    if (rc) return rc;
    float hl;
    PT_CUDA_TRY(cudaMemcpyAsync(out, dout.p, (size_t)D * 4, cudaMemcpyDeviceToHost, st));
    PT_CUDA_TRY(cudaMemcpyAsync(&hl, dlse.p, 4, cudaMemcpyDeviceToHost, st));
    PT_CUDA_TRY(cudaStreamSynchronize(st));
    *lse = (double)hl;
    return PT_OK;
}
