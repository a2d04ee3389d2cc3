"""Timeline of one captured decode step (tuning aid): %globaltimer stamps of the append
(per unit), the bounded scorer (per CTA: entry, after its PDL wait, exit) and select+attend
(per CTA), replayed from the bench's CUDA graph -> percentiles relative to the first append
entry, i.e. where the step's time goes between and inside the kernels.

    python tools/probe_step.py [--batch 32 --ctx 131072]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pct(x):
    return {p: round(float(np.percentile(x, p)), 2) for p in (0, 50, 100)}


def main():
    import torch

    import bench
    import paper_2605_27740_b200 as pt
    from paper_2605_27740_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=131072)
    a = ap.parse_args()
    args = bench.parse(["--batch", str(a.batch), "--ctx", str(a.ctx), "--steps", "8", "--warmup", "3"])
    dev = torch.device("cuda", 0)
    cache = bench.build_cache(args, dev, bench.SEED)
    G, kp = args.q_heads // args.kv_heads, args.budget // args.page
    eng = pt.DecodeEngine(cache, G, kp)
    qs, kn, vn = bench.step_inputs(args, dev)
    for i in range(3):
        eng.step(qs[i], kn, vn)
    torch.cuda.synchronize()
    os.environ.update(PT_APP_PROF="1", PT_SA_PROF="1", PT_SB_PROF="1")
    graphs = bench.capture_steps(eng, cache, qs[:1], kn, vn)
    for k in ("PT_APP_PROF", "PT_SA_PROF", "PT_SB_PROF"):
        os.environ.pop(k)
    runs = []
    U = cache.num_units
    L = _lib.load()
    for r in range(5):
        graphs[0].replay()
        torch.cuda.synchronize()
        app = np.zeros(U * 8, np.uint64)
        L.pt_debug_append_prof(app.ctypes.data, U * 8)
        sb = np.zeros(2048 * 4, np.uint64)
        L.pt_debug_sb_prof(sb.ctypes.data, 2048 * 4)
        nsa = U * 20
        sa = np.zeros(nsa, np.uint64)
        L.pt_debug_sa_prof(sa.ctypes.data, nsa)
        app = app.reshape(U, 8).astype(np.float64)
        nsb = torch.cuda.get_device_properties(0).multi_processor_count * 2
        sb = sb.reshape(2048, 4)[:nsb].astype(np.float64)
        sa = sa.reshape(U, 20).astype(np.float64)
        t0 = app[:, 0].min()
        f = lambda x: (x - t0) / 1000.0  # noqa: E731
        runs.append({
            "append_entry": pct(f(app[:, 0])), "append_exit": pct(f(app[:, 7])),
            "score_entry": pct(f(sb[:, 0])), "score_after_wait": pct(f(sb[:, 1])),
            "score_exit": pct(f(sb[:, 2])),
            "sa_entry": pct(f(sa[:, 0])), "sa_after_wait": pct(f(sa[:, 1])),
            "sa_split": pct(f(sa[:, 2])), "sa_first_page": pct(f(sa[:, 3])),
            "sa_stream_done": pct(f(sa[:, 4])), "sa_exit": pct(f(sa[:, 5])),
        })
    print(json.dumps({"shape": vars(a), "runs": runs[-2:]}, indent=1))


if __name__ == "__main__":
    main()
