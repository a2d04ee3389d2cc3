"""Bounded scorer tuning aid: time pt_score_bounded (single-launch CUDA graphs, 20 replays)
under ring-depth x CTAs-per-SM settings at a bench shape.

    python tools/probe_score.py [--batch 32 --ctx 131072 --kv-heads 8 --q-heads 32 --head-dim 128 --page 16]
"""
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
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--q-heads", type=int, default=32)
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--page", type=int, default=16)
    ap.add_argument("--budget", type=int, default=2048)
    a = ap.parse_args()
    args = bench.parse(["--batch", str(a.batch), "--ctx", str(a.ctx), "--kv-heads", str(a.kv_heads),
                        "--q-heads", str(a.q_heads), "--head-dim", str(a.head_dim), "--page",
                        str(a.page), "--budget", str(a.budget), "--steps", "1", "--warmup", "1"])
    dev = torch.device("cuda", 0)
    os.environ["PT_BOUNDED"] = "1"
    cache = bench.build_cache(args, dev, bench.SEED)
    G = a.q_heads // a.kv_heads
    eng = pt.DecodeEngine(cache, G, -(-a.budget // a.page))
    qs, _, _ = bench.step_inputs(args, dev)
    q = qs[0]
    eng.lam_norms(q)
    st = torch.cuda.current_stream()
    res = {}
    U, P, D = cache.num_units, -(-a.ctx // a.page), a.head_dim
    by = bench.step_bytes(U, G, D, P, 1, a.page, 2, 2, a.ctx)["score"]
    for nst in ("2", "3", "4"):
        for ctas in ("1", "2", "3"):
            os.environ["PT_SB_NST"], os.environ["PT_SB_CTAS"] = nst, ctas
            eng.score_bounded(q)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                eng.score_bounded(q)
            g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(20):
                g.replay()
            e1.record(st)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1000 / 20
            res[f"nst{nst}_ctas{ctas}"] = {"us": round(us, 2), "TBs": round(by / us / 1e6, 3)}
            del g
    os.environ["PT_BOUNDED"] = "0"
    eng2 = pt.DecodeEngine(cache, G, -(-a.budget // a.page))
    eng2.bounded = False
    eng2.lam_norms(q)
    eng2.score_prenorm(q)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        eng2.score_prenorm(q)
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(20):
        g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    res["exact_f32"] = {"us": round(e0.elapsed_time(e1) * 1000 / 20, 2)}
    print(json.dumps({"shape": vars(a), "score_bytes_8d": by, "results": res}))


if __name__ == "__main__":
    main()
