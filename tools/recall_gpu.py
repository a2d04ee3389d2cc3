"""Selection quality at GPU scale: unique vs mean-only vs Quest page
recall / mass recall / output error on dilution workloads (planted pages) at long context.

    python tools/recall_gpu.py [--units 64] [--ctx 131072] > profiles/r01/recall_r01.json
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2605_27740_b200 import recall

    ap = argparse.ArgumentParser()
    ap.add_argument("--units", type=int, default=64)
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--page", type=int, default=16)
    ap.add_argument("--planted", type=int, default=16)
    ap.add_argument("--gain", type=float, default=6.0)
    ap.add_argument("--budgets", default="512,1024,2048,4096")
    a = ap.parse_args()
    out = {"units": a.units, "ctx": a.ctx, "page": a.page, "planted_pages": a.planted,
           "planted_gain": a.gain, "head_dim": 128, "kv_dtype": "bf16", "results": {}}
    wl = recall.gen_units_workload(a.units, a.ctx, 128, page_size=a.page,
                                   planted_pages=a.planted, planted_gain=a.gain, seed=1,
                                   dtype=torch.bfloat16)
    masses = recall.oracle_page_masses(wl.cache, wl.queries)
    for b in [int(x) for x in a.budgets.split(",")]:
        k = b // a.page
        rep = recall.eval_recall_units(wl.cache, wl.queries, k, masses=masses)
        res = {}
        for m, rows in rep.items():
            res[m] = {"page_recall": float(np.mean([r.page_recall for r in rows])),
                      "mass_recall": float(np.mean([r.mass_recall for r in rows])),
                      "output_err": float(np.mean([r.output_err for r in rows]))}
        out["results"][f"budget_{b}_tokens"] = res
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
