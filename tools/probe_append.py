"""Phase timeline of the decode append kernel (tuning aid): per-unit %globaltimer stamps ->
median / max of each phase boundary relative to the earliest warp entry.  Runs the append as
in the bench step (after a scoring kernel, so PDL overlap is live) for several steps."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_2605_27740_b200 as pt
    from paper_2605_27740_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--clock", action="store_true", help="%%clock64 stamps: per-unit durations (cycles)")
    a = ap.parse_args()
    ns = argparse.Namespace(batch=a.batch, ctx=a.ctx, q_heads=32, kv_heads=8, head_dim=128,
                            page=16, budget=2048, stats_dtype="f32", warmup=3, steps=10)
    dev = torch.device("cuda", 0)
    cache = bench.build_cache(ns, dev, seed=1234)
    U, D = cache.num_units, 128
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    kn = torch.randn(U, D, generator=g, device=dev).to(torch.bfloat16)
    vn = torch.randn(U, D, generator=g, device=dev).to(torch.bfloat16)
    names = os.environ.get("APP_NAMES", "entry,pdl_wait,row,pid,staged,stats,snap_seen,exit").split(",")
    for _ in range(3):
        cache.append_batch(kn, vn)
    torch.cuda.synchronize()
    os.environ["PT_APP_PROF"] = "2" if a.clock else "1"
    per = []
    for _ in range(a.steps):
        cache.append_batch(kn, vn)
        torch.cuda.synchronize()
        buf = np.zeros(U * 8, dtype=np.uint64)
        _lib.check(_lib.load().pt_debug_append_prof(buf.ctypes.data, U * 8))
        t = buf.reshape(U, 8).astype(np.float64)
        if a.clock:  # per unit, relative to its own entry; cycles -> us at 1.965 GHz
            per.append((t - t[:, :1]) / 1965.0)
        else:
            per.append((t - t[:, 0].min()) / 1000.0)
    os.environ.pop("PT_APP_PROF")
    rel = np.stack(per)  # [steps, U, 8]
    out = {nm: {"median": float(np.median(rel[:, :, i])), "max": float(np.median(rel[:, :, i].max(axis=1)))}
           for i, nm in enumerate(names)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
