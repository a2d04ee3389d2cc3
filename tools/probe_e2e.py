"""Where the end-to-end step's time goes (tuning aid): per-step wall time of
  A  H2D (one pinned block) -> DecodeEngine.replay() -> D2H -> sync   (bench.py's e2e)
  B  replay() -> sync                      (no copies)
  C  one CUDA graph holding the H2D copy, the step and the D2H copy -> sync
at the bench shape, 100 steps each, medians of 3 runs."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_2605_27740_b200 as pt

    ns = argparse.Namespace(batch=32, ctx=131072, q_heads=32, kv_heads=8, head_dim=128,
                            page=16, budget=2048, stats_dtype="f32", warmup=3, steps=10)
    d = torch.device("cuda", 0)
    cache = bench.build_cache(ns, d, seed=1234)
    U, G, D = cache.num_units, 4, 128
    eng = pt.DecodeEngine(cache, G, 128)
    nq, nk = U * G * D, U * D
    host_in = torch.randn(nq + 2 * nk).to(torch.bfloat16).pin_memory()
    dev_in = host_in.to(d)
    q, kn, vn = dev_in[:nq].view(U * G, D), dev_in[nq:nq + nk].view(U, D), dev_in[nq + nk:].view(U, D)
    out_h = torch.empty(U * G, D, dtype=torch.float32).pin_memory()
    eng.capture(q, kn, vn)
    st = torch.cuda.current_stream()

    def run(step, n=100):
        for _ in range(5):
            step()
        res = []
        for _ in range(3):
            t0 = time.perf_counter()
            for _ in range(n):
                step()
            res.append((time.perf_counter() - t0) / n * 1e6)
        return sorted(res)[1]

    def a():
        dev_in.copy_(host_in, non_blocking=True)
        eng.replay()
        out_h.copy_(eng.out, non_blocking=True)
        st.synchronize()

    def b():
        eng.replay()
        st.synchronize()

    # C: the copies inside the captured graph
    s2 = torch.cuda.Stream()
    s2.wait_stream(st)
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s2):
        with torch.cuda.graph(g2, stream=s2):
            dev_in.copy_(host_in, non_blocking=True)
            eng.step(q, kn, vn)
            out_h.copy_(eng.out, non_blocking=True)
    st.wait_stream(s2)

    def c():
        g2.replay()
        st.synchronize()

    r = {"A_h2d_replay_d2h_us": run(a), "B_replay_only_us": run(b), "C_one_graph_us": run(c)}
    print(json.dumps(r, indent=1))


if __name__ == "__main__":
    main()
