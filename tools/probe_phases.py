"""Phase timeline of the fused select+attend kernel (tuning aid): per-CTA %globaltimer
stamps -> percentiles of each phase boundary relative to the earliest CTA entry."""
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
    ap.add_argument("--budget", type=int, default=2048)
    a = ap.parse_args()
    ns = argparse.Namespace(batch=a.batch, ctx=a.ctx, q_heads=32, kv_heads=8, head_dim=128,
                            page=16, budget=a.budget, stats_dtype="f32", warmup=3, steps=10)
    dev = torch.device("cuda", 0)
    cache = bench.build_cache(ns, dev, seed=1234)
    G, D, S = 4, 128, 16
    U = cache.num_units
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    q = torch.randn(U * G, D, generator=g, device=dev).to(torch.bfloat16)
    eng = pt.DecodeEngine(cache, G, a.budget // S)
    eng.score(q)
    for _ in range(3):
        eng.select_attend(q)
    torch.cuda.synchronize()
    os.environ["PT_SA_PROF"] = "1"
    eng.select_attend(q)
    torch.cuda.synchronize()
    os.environ.pop("PT_SA_PROF")
    n = U * 10
    buf = np.zeros(n, dtype=np.uint64)
    _lib.check(_lib.load().pt_debug_sa_prof(buf.ctypes.data, n))
    t = buf.reshape(U, 10).astype(np.float64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0
    names = ["entry", "keys_staged", "selected", "first_page", "stream_done", "exit",
             "sel_loads_max", "sel_L", "sel_cands", "sel_thr"]
    out = {}
    for i, nm in enumerate(names):
        col = rel[:, i]
        out[nm] = {p: round(float(np.percentile(col, p)), 2) for p in (0, 10, 50, 90, 100)}
    out["durations_us_median"] = {
        "stage_keys": float(np.median(rel[:, 1] - rel[:, 0])),
        "select": float(np.median(rel[:, 2] - rel[:, 1])),
        "first_page": float(np.median(rel[:, 3] - rel[:, 2])),
        "stream": float(np.median(rel[:, 4] - rel[:, 3])),
        "merge": float(np.median(rel[:, 5] - rel[:, 4])),
        "sel_loads_max": float(np.median(rel[:, 6] - rel[:, 1])),
        "sel_L": float(np.median(rel[:, 7] - rel[:, 6])),
        "sel_cands": float(np.median(rel[:, 8] - rel[:, 7])),
        "sel_thr": float(np.median(rel[:, 9] - rel[:, 8])),
        "sel_pick_translate": float(np.median(rel[:, 2] - rel[:, 9])),
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
