"""Feasibility probe (tuning aid): does running one half-batch's select+attend concurrently with
the other half-batch's scorer (two streams) beat the serial order?  Two half caches (16
sequences each, the cfg3 shape), no appends; times (a) serial: scoreA, saA, scoreB, saB and
(b) overlapped: scoreA; [stream 2: saA] || [stream 1: scoreB]; saB, with CUDA events, as
single-stage CUDA graphs replayed 20 times."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_2605_27740_b200 as pt

    args = bench.parse(["--batch", "16", "--steps", "1", "--warmup", "1"])
    dev = torch.device("cuda", 0)
    caches = [bench.build_cache(args, dev, bench.SEED + i) for i in range(2)]
    G, kp = 4, 128
    engs = [pt.DecodeEngine(c, G, kp) for c in caches]
    qs, _, _ = bench.step_inputs(args, dev)
    q = qs[0]
    for e in engs:
        e.lam_norms(q)
        e.score_step(q)
        e.select_attend(q)
    torch.cuda.synchronize()
    s1 = torch.cuda.current_stream()
    s2 = torch.cuda.Stream()

    def serial():
        for e in engs:
            e.score_step(q)
            e.select_attend(q)

    def overlapped():
        a, b = engs
        a.score_step(q)
        ev = torch.cuda.Event()
        ev.record(s1)
        s2.wait_event(ev)
        with torch.cuda.stream(s2):
            a.select_attend(q, stream=s2)
        b.score_step(q)
        b.select_attend(q)
        ev2 = torch.cuda.Event()
        ev2.record(s2)
        s1.wait_event(ev2)

    res = {}
    for name, fn in (("serial", serial), ("overlapped", overlapped)):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s0 = torch.cuda.Stream()
        s0.wait_stream(s1)
        with torch.cuda.stream(s0):
            with torch.cuda.graph(g, stream=s0):
                fn()
        s1.wait_stream(s0)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s1)
        for _ in range(20):
            g.replay()
        e1.record(s1)
        torch.cuda.synchronize()
        res[name + "_us"] = e0.elapsed_time(e1) * 1000 / 20
        del g
    print(json.dumps(res))


if __name__ == "__main__":
    main()
