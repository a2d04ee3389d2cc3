"""Paper Table 5 on B200: fused one-launch scoring (K2) vs the naive three-launch scorer
(GEMM -> rank-one offset add -> column max, scoring.py:127-143) at a batched decode shape.

    python tools/table5.py [--batch 32] [--ctx 131072] > profiles/r01/table5_r01.json

Both paths read the same page statistics; the naive one materialises two G x P f32
intermediates per unit in HBM (traffic_of_naive, scoring.py:146-180).  Reported: device time
per step (CUDA events, 20 launches), the closed-form traffic of each path, the write ratio
(2G + 1), and the agreement of the two score vectors.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_2605_27740_b200 as pt
    from paper_2605_27740_b200 import _device as dev
    from paper_2605_27740_b200.scoring import traffic_of_fused, traffic_of_naive, traffic_write_ratio

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=131072)
    a = ap.parse_args()
    ns = argparse.Namespace(batch=a.batch, ctx=a.ctx, q_heads=32, kv_heads=8, head_dim=128,
                            page=16, budget=2048, stats_dtype="f32", warmup=3, steps=10)
    d = torch.device("cuda", 0)
    cache = bench.build_cache(ns, d, seed=1234)
    G, D, S = 4, 128, 16
    U = cache.num_units
    P = -(-a.ctx // S)
    g = torch.Generator(device=d)
    g.manual_seed(7)
    q = torch.randn(U * G, D, generator=g, device=d)  # f32 queries (the reference's dtype)
    eng = pt.DecodeEngine(cache, G, 128, keep_scores=True)
    lam = 0.5
    # naive inputs: row-major means [U, P, D] f32, stds [U, P], norms [U, G]
    means = dev.untile_means(cache.means, U, cache.Pmax, D, cache.stats_dtype)[:, :P].contiguous()
    stds = cache.stds[:, :P].contiguous()
    qg = q.view(U, G, D)
    norms = torch.linalg.vector_norm(qg.double(), dim=2).float()

    def naive():
        raw = torch.bmm(qg, means.transpose(1, 2))                       # launch 1: U x G x P
        off = raw + (lam * norms)[:, :, None] * stds[:, None, :]          # launch 2
        return off.max(dim=1).values                                      # launch 3

    def fused():
        eng.score(q)

    stream = torch.cuda.current_stream()

    def timeit(fn, reps=20):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1000 / reps

    t_fused = timeit(fused)
    t_naive = timeit(naive)
    fused()
    s_naive = naive()
    torch.cuda.synchronize()
    s_fused = eng.scores[:, :P]
    rel = ((s_fused - s_naive).abs() / s_naive.abs().clamp_min(1e-30)).max().item()
    tf = traffic_of_fused(G, P, D)
    tn = traffic_of_naive(G, P, D)
    print(json.dumps({
        "shape": {"units": U, "group": G, "pages": P, "head_dim": D, "batch": a.batch, "ctx": a.ctx},
        "fused_us": t_fused, "naive_us": t_naive, "speedup": t_naive / t_fused,
        "fused_launches": tf.launches, "naive_launches": tn.launches,
        "fused_scalar_traffic_per_unit": tf.total, "naive_scalar_traffic_per_unit": tn.total,
        "write_ratio_naive_over_fused": traffic_write_ratio(tn, tf),
        "fused_GBs": U * tf.total * 4 / (t_fused * 1e-6) / 1e9,
        "naive_GBs_closed_form": U * tn.total * 4 / (t_naive * 1e-6) / 1e9,
        "max_rel_diff_fused_vs_naive": rel,
        "note": "fused = pt_score (lambda*norm precompute + streaming K2, f32 queries/stats); "
                "naive = torch bmm + broadcast add + max over G (cuBLAS / library kernels)",
    }, indent=1))


if __name__ == "__main__":
    main()
