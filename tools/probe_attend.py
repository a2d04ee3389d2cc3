"""Attention-kernel probe (tuning aid, not a bench line): K4 time vs page budget, scattered vs
contiguous pages, to split fixed per-launch overhead from per-byte streaming cost.

    python tools/probe_attend.py [--batch 32] [--ctx 131072]
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

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--budgets", default="512,1024,2048,4096,8192")
    ap.add_argument("--env", default="", help="extra env sweeps: NAME=v1,v2;NAME2=...")
    ap.add_argument("--split", default="", help="(split, unit)-grid kernel at these nsplit values")
    a = ap.parse_args()
    ns = argparse.Namespace(batch=a.batch, ctx=a.ctx, q_heads=32, kv_heads=8, head_dim=128,
                            page=16, budget=2048, stats_dtype="f32", warmup=3, steps=10)
    dev = torch.device("cuda", 0)
    cache = bench.build_cache(ns, dev, seed=1234)
    G, D, S = 4, 128, 16
    U = cache.num_units
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    q = torch.randn(U * G, D, generator=g, device=dev).to(torch.bfloat16)
    stream = torch.cuda.current_stream()

    def timeit(fn, reps=30):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1000 / reps

    res = {}
    for bud in [int(x) for x in a.budgets.split(",")]:
        kp = bud // S
        eng = pt.DecodeEngine(cache, G, kp)
        eng.score_select(q)
        torch.cuda.synchronize()
        mb = U * (2 * kp * S * D * 2) / 1e6
        t_sc = timeit(lambda: eng.attend(q))
        saved = eng.sel.clone()
        eng.sel.copy_(cache.page_table[:, :kp])
        t_ct = timeit(lambda: eng.attend(q))
        eng.sel.copy_(saved)
        res[f"k{kp}"] = {"MB": mb, "scattered_us": t_sc, "contig_us": t_ct,
                         "scattered_GBs": mb / t_sc * 1e3, "contig_GBs": mb / t_ct * 1e3}
        if a.env:
            for spec in a.env.split(";"):
                name, vals = spec.split("=")
                for v in vals.split(","):
                    os.environ[name] = v
                    try:
                        res[f"k{kp}"][f"{name}={v}"] = timeit(lambda: eng.attend(q))
                    except Exception as e:  # noqa: BLE001
                        res[f"k{kp}"][f"{name}={v}"] = str(e)[:80]
                    os.environ.pop(name)
        for ns in [int(x) for x in a.split.split(",") if x]:
            os.environ["PT_ATTEND_SPLIT"] = "1"
            res[f"k{kp}"][f"split{ns}"] = timeit(lambda: eng.attend(q, nsplit=ns))
            os.environ.pop("PT_ATTEND_SPLIT")
        del eng
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
