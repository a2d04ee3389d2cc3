"""Soft-mask training path throughput (tuning aid): gated attention forward (K4 dense with
log-gate bias) and backward (pt_gated_attend_bwd) over a batched cache, with the HBM bytes
each pass must move (fwd: K+V read; bwd: K+V read, dK+dV f32 written, dq/dgates).

    python tools/probe_gated.py [--batch 4] [--ctx 32768]
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    from paper_2605_27740_b200 import softmask as sm

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--ctx", type=int, default=32768)
    a = ap.parse_args()
    ns = argparse.Namespace(batch=a.batch, ctx=a.ctx, q_heads=32, kv_heads=8, head_dim=128,
                            page=16, budget=2048, stats_dtype="f32", warmup=3, steps=10)
    d = torch.device("cuda", 0)
    cache = bench.build_cache(ns, d, seed=1234)
    U, G, D, S = cache.num_units, 4, 128, 16
    P = -(-a.ctx // S)
    g = torch.Generator(device=d)
    g.manual_seed(3)
    q = torch.randn(U * G, D, generator=g, device=d).to(torch.bfloat16)
    gates = torch.rand(U, cache.Pmax, generator=g, device=d, dtype=torch.float64) * 0.9 + 0.1
    gates[:, P:] = 0
    stream = torch.cuda.current_stream()

    def timeit(fn, reps=10):
        # median of individually timed calls: a back-to-back loop that keeps the previous
        # result alive makes the caching allocator cudaMalloc fresh 0.5 GB gradient pools
        # now and then (one 16 ms outlier dominated the former 10-call mean)
        r = fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            del r
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1000)
        return sorted(ts)[len(ts) // 2], r

    t_fwd, (out, lse) = timeit(lambda: sm.gated_forward(cache, q, gates))
    # the forward's kernel alone (pt_attend dense mode + per-page bias), buffers preallocated
    from paper_2605_27740_b200 import _lib
    from paper_2605_27740_b200 import _device as dv
    bias = torch.log(gates).to(torch.float32).contiguous()
    o2, l2 = torch.empty_like(out), torch.empty_like(lse)
    ws = torch.empty(_lib.load().pt_attend_workspace_bytes(U, G, D, cache.Pmax), dtype=torch.uint8, device=d)
    tk = torch.zeros(U, dtype=torch.int32, device=d)

    def fwd_kernel():
        _lib.call("pt_attend", q.data_ptr(), dv.dtype_code(q.dtype), cache.k_pool.data_ptr(),
                  cache.v_pool.data_ptr(), cache.kv_code, cache.layout.max_pages,
                  cache.page_table.data_ptr(), cache.Pmax, None, cache.page_table.data_ptr(),
                  cache.seq_lens.data_ptr(), U, G, D, S, cache.Pmax, bias.data_ptr(),
                  1.0 / math.sqrt(D), o2.data_ptr(), l2.data_ptr(), ws.data_ptr(), ws.numel(),
                  tk.data_ptr(), 0, dv.stream_handle())
        return o2
    t_fwd_k, _ = timeit(fwd_kernel)
    # back-to-back launches (no host gap between them): the kernel's own rate
    fwd_kernel()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(20):
        fwd_kernel()
    e1.record(stream)
    torch.cuda.synchronize()
    t_fwd_k_b2b = e0.elapsed_time(e1) * 1000 / 20
    # the same dense pass through the streaming kernel (every page listed, n_sel = pages)
    nsel = ((cache.seq_lens + S - 1) // S).to(torch.int32)
    o3, l3 = torch.empty_like(out), torch.empty_like(lse)

    def fwd_stream():
        _lib.call("pt_attend", q.data_ptr(), dv.dtype_code(q.dtype), cache.k_pool.data_ptr(),
                  cache.v_pool.data_ptr(), cache.kv_code, cache.layout.max_pages,
                  cache.page_table.data_ptr(), cache.Pmax, nsel.data_ptr(), cache.page_table.data_ptr(),
                  cache.seq_lens.data_ptr(), U, G, D, S, cache.Pmax, bias.data_ptr(),
                  1.0 / math.sqrt(D), o3.data_ptr(), l3.data_ptr(), ws.data_ptr(), ws.numel(),
                  tk.data_ptr(), 0, dv.stream_handle())
    fwd_stream()
    e0.record(stream)
    for _ in range(20):
        fwd_stream()
    e1.record(stream)
    torch.cuda.synchronize()
    t_fwd_s_b2b = e0.elapsed_time(e1) * 1000 / 20
    stream_diff = float((o3 - o2).abs().max()), float((l3 - l2).abs().max())
    dout = torch.randn(U * G, D, generator=g, device=d)
    t_bwd, _ = timeit(lambda: sm.gated_backward(cache, q, gates, out, lse, dout))
    bwd_bytes_all = None
    ntok = U * a.ctx
    fwd_bytes = ntok * D * 2 * 2
    bwd_bytes = ntok * D * 2 * 2 + ntok * D * 4 * 2
    print(json.dumps({"units": U, "group": G, "ctx": a.ctx, "tokens": ntok,
                      "fwd_us": t_fwd, "fwd_GBs": fwd_bytes / (t_fwd * 1e-6) / 1e9,
                      "fwd_kernel_us": t_fwd_k, "fwd_kernel_GBs": fwd_bytes / (t_fwd_k * 1e-6) / 1e9,
                      "fwd_kernel_b2b_us": t_fwd_k_b2b,
                      "fwd_kernel_b2b_GBs": fwd_bytes / (t_fwd_k_b2b * 1e-6) / 1e9,
                      "fwd_stream_b2b_us": t_fwd_s_b2b, "fwd_stream_vs_split_maxdiff": stream_diff,
                      "bwd_us": t_bwd, "bwd_GBs": bwd_bytes / (t_bwd * 1e-6) / 1e9,
                      "note": "median of 10 individually timed calls (CUDA events; fwd_kernel_b2b: 20 back-to-back launches); fwd = pt_attend dense + "
                              "log-gate bias (incl. the host-side gate checks); bwd = gated_backward "
                              "(pt_gated_attend_bwd + output allocation: K, V read; f32 dK, dV written)"},
                     indent=1))


if __name__ == "__main__":
    main()
