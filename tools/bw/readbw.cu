// Read-bandwidth probe (tuning aid): how fast can an SM-resident kernel stream HBM on this
// B200 when it only reads?  (a) 16-byte vector loads, grid-stride, 8 in flight per thread;
// (b) per-warp rings of 1-D bulk async copies (cp.async.bulk, mbarrier) like the scorer.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o readbw readbw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_ld(const uint4 *__restrict__ a, size_t n, unsigned *out) {
    unsigned acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n; i += 8 * stride) {
        uint4 v[8];
#pragma unroll
        for (int j = 0; j < 8; j++) v[j] = __ldcs(a + i + j * stride);
#pragma unroll
        for (int j = 0; j < 8; j++) acc ^= v[j].x ^ v[j].y ^ v[j].z ^ v[j].w;
    }
    for (; i < n; i += stride) { uint4 v = a[i]; acc ^= v.x ^ v.w; }
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int NST, int CH>
__global__ void __launch_bounds__(128) k_bulk(const char *__restrict__ a, size_t nbytes, unsigned *out) {
    extern __shared__ __align__(128) char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char *ring = sm + (size_t)warp * NST * CH;
    __shared__ __align__(8) uint64_t bars[4][NST];
    const size_t nch = nbytes / CH;
    const size_t gw = (size_t)blockIdx.x * 4 + warp, W = (size_t)gridDim.x * 4;
    const size_t c0 = gw * nch / W, c1 = (gw + 1) * nch / W;
    const int cnt = (int)(c1 - c0);
    if (lane == 0) {
        for (int s = 0; s < NST; s++)
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bars[warp][s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    auto issue = [&](int i) {
        const int s = i % NST;
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bars[warp][s])), "r"(CH));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(ring + (size_t)s * CH)), "l"(a + (c0 + i) * CH), "r"(CH), "r"(su32(&bars[warp][s])) : "memory");
    };
    if (lane == 0) for (int i = 0; i < NST && i < cnt; i++) issue(i);
    unsigned acc = 0;
    for (int i = 0; i < cnt; i++) {
        const int s = i % NST;
        const uint32_t ph = (i / NST) & 1;
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done) : "r"(su32(&bars[warp][s])), "r"(ph));
        acc ^= reinterpret_cast<const unsigned *>(ring + (size_t)s * CH)[lane];
        __syncwarp();
        if (lane == 0 && i + NST < cnt) issue(i + NST);
    }
    if (acc == 0x12345678u) out[0] = acc;
}

int main() {
    const size_t nbytes = (size_t)2 << 30;
    char *a; unsigned *o;
    cudaMalloc(&a, nbytes); cudaMalloc(&o, 4);
    cudaMemset(a, 1, nbytes);
    char *flush; cudaMalloc(&flush, (size_t)256 << 20);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](auto launch, const char *name) {
        float best = 1e9;
        for (int r = 0; r < 8; r++) {
            cudaMemsetAsync(flush, r, (size_t)256 << 20);
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (r > 0 && ms < best) best = ms;
        }
        printf("{\"kernel\": \"%s\", \"GBs\": %.1f, \"us\": %.1f}\n", name, nbytes / (best * 1e-3) / 1e9, best * 1e3);
    };
    for (int per : {4, 8, 16}) {
        char nm[64]; snprintf(nm, 64, "ld128 grid=%dxSM x256", per);
        timeit([&] { k_ld<<<nsm * per, 256>>>((const uint4 *)a, nbytes / 16, o); }, nm);
    }
    {
        constexpr int NST = 4, CH = 8192;
        const size_t smem = 4 * NST * CH;
        cudaFuncSetAttribute(k_bulk<NST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int per : {1, 2}) {
            char nm[64]; snprintf(nm, 64, "bulk 4st x 8KB grid=%dxSM", per);
            timeit([&] { k_bulk<NST, CH><<<nsm * per, 128, smem>>>(a, nbytes, o); }, nm);
        }
    }
    {
        constexpr int NST = 3, CH = 16384;
        const size_t smem = 4 * NST * CH;
        cudaFuncSetAttribute(k_bulk<NST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        timeit([&] { k_bulk<NST, CH><<<nsm, 128, smem>>>(a, nbytes, o); }, "bulk 3st x 16KB grid=1xSM");
    }
    {
        constexpr int NST = 6, CH = 4096;
        const size_t smem = 4 * NST * CH;
        cudaFuncSetAttribute(k_bulk<NST, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int per : {2, 3}) {
            char nm[64]; snprintf(nm, 64, "bulk 6st x 4KB grid=%dxSM", per);
            timeit([&] { k_bulk<NST, CH><<<nsm * per, 128, smem>>>(a, nbytes, o); }, nm);
        }
    }
    // copy for reference (read + write bytes)
    {
        char *b; cudaMalloc(&b, nbytes / 2);
        float best = 1e9;
        for (int r = 0; r < 8; r++) {
            cudaEventRecord(e0); cudaMemcpyAsync(b, a, nbytes / 2, cudaMemcpyDeviceToDevice); cudaEventRecord(e1);
            cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r > 0 && ms < best) best = ms;
        }
        printf("{\"kernel\": \"memcpy d2d (r+w bytes)\", \"GBs\": %.1f}\n", nbytes / (best * 1e-3) / 1e9);
    }
    cudaError_t err = cudaGetLastError();
    printf("{\"status\": \"%s\"}\n", cudaGetErrorString(err));
    return 0;
}
