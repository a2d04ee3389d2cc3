// runtime.cu -- the host-side serving loop of the decode step in native code.
//
// pt_pipe_submit queues one decode step of a depth-slot pipeline (pipeline.py
// PipelinedDecoder): H2D of the step's packed inputs on the h2d stream, the slot's captured
// step graph on the compute stream, D2H of its outputs on the d2h stream, with the event
// edges that let step n + 1's H2D and step n - 1's D2H run under step n's kernels:
//
//   h2d:     wait done[s] (slot's previous step consumed its inputs) -> H2D -> rec in_ready[s]
//   compute: wait in_ready[s], wait out_ready[s] (previous outputs read) -> graph -> rec done[s]
//   d2h:     wait done[s] -> D2H -> rec out_ready[s]
//
// H2D and D2H sit on two streams: on one, step n + 1's H2D would queue behind step n's D2H,
// which waits for step n's kernels -- the copy would serialise with the step.
//
// ten CUDA runtime calls, no Python in between (the per-step host cost bounds the
// end-to-end rate once the device step is ~180 us).
#include <cuda_runtime.h>

#include "common.cuh"

namespace {

constexpr int kPipeMaxDepth = 8;

struct Pipe {
    cudaStream_t compute = nullptr, h2d = nullptr, d2h = nullptr;
    cudaEvent_t in_ready[kPipeMaxDepth] = {}, done[kPipeMaxDepth] = {}, out_ready[kPipeMaxDepth] = {};
    bool used[kPipeMaxDepth] = {};
    int depth = 0;
};

}  // namespace

extern "C" int pt_pipe_create(void *compute_stream, void *h2d_stream, void *d2h_stream, int depth,
                              void **pipe_out) {
    if (!pipe_out || depth < 1 || depth > kPipeMaxDepth || !h2d_stream || !d2h_stream ||
        h2d_stream == d2h_stream)
        return PT_ERR_INVALID;
    Pipe *p = new Pipe();
    p->compute = (cudaStream_t)compute_stream;
    p->h2d = (cudaStream_t)h2d_stream;
    p->d2h = (cudaStream_t)d2h_stream;
    p->depth = depth;
    for (int i = 0; i < depth; i++) {
        const unsigned fl = cudaEventDisableTiming;
        if (cudaEventCreateWithFlags(&p->in_ready[i], fl) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->done[i], fl) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->out_ready[i], fl) != cudaSuccess) {
            delete p;
            return PT_ERR_CUDA_BASE + (int)cudaGetLastError();
        }
    }
    *pipe_out = p;
    return PT_OK;
}

extern "C" int pt_pipe_submit(void *pipe, int slot, void *graph_exec, void *dev_in, const void *host_in,
                              size_t in_bytes, void *host_out, const void *dev_out, size_t out_bytes) {
    Pipe *p = static_cast<Pipe *>(pipe);
    if (!p || slot < 0 || slot >= p->depth || !graph_exec || !dev_in || !host_in || !host_out ||
        !dev_out)
        return PT_ERR_INVALID;
    const int s = slot;
    if (p->used[s]) PT_CUDA_TRY(cudaStreamWaitEvent(p->h2d, p->done[s], 0));
    PT_CUDA_TRY(cudaMemcpyAsync(dev_in, host_in, in_bytes, cudaMemcpyHostToDevice, p->h2d));
    PT_CUDA_TRY(cudaEventRecord(p->in_ready[s], p->h2d));
    PT_CUDA_TRY(cudaStreamWaitEvent(p->compute, p->in_ready[s], 0));
    if (p->used[s]) PT_CUDA_TRY(cudaStreamWaitEvent(p->compute, p->out_ready[s], 0));
    PT_CUDA_TRY(cudaGraphLaunch((cudaGraphExec_t)graph_exec, p->compute));
    PT_CUDA_TRY(cudaEventRecord(p->done[s], p->compute));
    PT_CUDA_TRY(cudaStreamWaitEvent(p->d2h, p->done[s], 0));
    PT_CUDA_TRY(cudaMemcpyAsync(host_out, dev_out, out_bytes, cudaMemcpyDeviceToHost, p->d2h));
    PT_CUDA_TRY(cudaEventRecord(p->out_ready[s], p->d2h));
    p->used[s] = true;
    return PT_OK;
}

// block the host until the slot's outputs are in host memory
extern "C" int pt_pipe_wait(void *pipe, int slot) {
    Pipe *p = static_cast<Pipe *>(pipe);
    if (!p || slot < 0 || slot >= p->depth) return PT_ERR_INVALID;
    if (p->used[slot]) PT_CUDA_TRY(cudaEventSynchronize(p->out_ready[slot]));
    return PT_OK;
}

extern "C" int pt_pipe_destroy(void *pipe) {
    Pipe *p = static_cast<Pipe *>(pipe);
    if (!p) return PT_OK;
    for (int i = 0; i < p->depth; i++) {
        if (p->in_ready[i]) cudaEventDestroy(p->in_ready[i]);
        if (p->done[i]) cudaEventDestroy(p->done[i]);
        if (p->out_ready[i]) cudaEventDestroy(p->out_ready[i]);
    }
    delete p;
    return PT_OK;
}
