"""A/B of two engine variants on ONE cache in one process (tuning aid): each variant's step is
captured as CUDA graphs (bench.capture_steps) and the two are timed in alternating blocks of
replays, so box-to-box and run-to-run drift cancel.  The variant is an environment variable
read when the engine is built (default PT_NORMS_SEPARATE: 0 vs 1).

    python tools/ab_step.py [--var PT_NORMS_SEPARATE] [--a 0] [--b 1] [--batch 32 --ctx 131072]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_2605_27740_b200 as pt

    ap = argparse.ArgumentParser()
    ap.add_argument("--var", default="PT_NORMS_SEPARATE")
    ap.add_argument("--a", default="0")
    ap.add_argument("--b", default="1")
    ap.add_argument("--blocks", type=int, default=8)
    ap.add_argument("--reps", type=int, default=100)
    a, rest = ap.parse_known_args()
    # capacity for every replayed append (blocks x 2 variants x (reps + 10) + warm-up)
    args = bench.parse(rest + ["--steps", str(a.blocks * 2 * (a.reps + 10) // 3 + 50)])
    dev = torch.device("cuda", 0)
    cache = bench.build_cache(args, dev, bench.SEED)
    qs, kn, vn = bench.step_inputs(args, dev)
    G = args.q_heads // args.kv_heads
    kp = args.budget // args.page
    graphs = {}
    for name in (a.a, a.b):
        os.environ[a.var] = name
        eng = pt.DecodeEngine(cache, G, kp)
        for _ in range(3):
            eng.step(qs[0], kn, vn)
        torch.cuda.synchronize()
        graphs[name] = (eng, bench.capture_steps(eng, cache, qs, kn, vn))
    os.environ.pop(a.var)
    res = {a.a: [], a.b: []}
    s = torch.cuda.current_stream()
    for blk in range(a.blocks):
        for name in ((a.a, a.b) if blk % 2 == 0 else (a.b, a.a)):
            gs = graphs[name][1]
            for i in range(10):
                gs[i % len(gs)].replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            for i in range(a.reps):
                gs[i % len(gs)].replay()
            e1.record(s)
            torch.cuda.synchronize()
            res[name].append(e0.elapsed_time(e1) * 1000.0 / a.reps)
            cache._seq_host += a.reps + 10
    out = {"var": a.var, "us_per_step": {k: {"median": statistics.median(v), "all": [round(x, 2) for x in v]}
                                         for k, v in res.items()}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
