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
        fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            r = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1000 / reps, r

    t_fwd, (out, lse) = timeit(lambda: sm.gated_forward(cache, q, gates))
    dout = torch.randn(U * G, D, generator=g, device=d)
    t_bwd, _ = timeit(lambda: sm.gated_backward(cache, q, gates, out, lse, dout))
    bwd_bytes_all = None
    ntok = U * a.ctx
    fwd_bytes = ntok * D * 2 * 2
    bwd_bytes = ntok * D * 2 * 2 + ntok * D * 4 * 2
    print(json.dumps({"units": U, "group": G, "ctx": a.ctx, "tokens": ntok,
                      "fwd_us": t_fwd, "fwd_GBs": fwd_bytes / (t_fwd * 1e-6) / 1e9,
                      "bwd_us": t_bwd, "bwd_GBs": bwd_bytes / (t_bwd * 1e-6) / 1e9,
                      "note": "fwd = pt_attend dense + log-gate bias (incl. the host-side gate "
                              "checks); bwd = pt_gated_attend_bwd (K, V read; f32 dK, dV written)"},
                     indent=1))


if __name__ == "__main__":
    main()
