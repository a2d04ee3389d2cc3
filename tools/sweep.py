"""Config sweep: decode-step latency, per-kernel breakdown,
HBM roofline fraction and dense speed-up per shape, plus the prefill page-stat build.

    python tools/sweep.py [--quick] > profiles/r01/sweep.jsonl

One JSON line per configuration.  Synthetic N(0,1) K/V/q generated on the device; the step is
the CUDA-graph replay of DecodeEngine.step (append | norms, score, select+attend).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def configs(quick: bool):
    out = [
        # name, batch, q_heads, kv_heads, head_dim, page, ctx, budget tokens
        ("cfg1 f32 8q/8kv b1 4K k32pages", 1, 8, 8, 128, 16, 4096, 512),
        ("cfg1 f32 8q/1kv b1 4K k32pages", 1, 8, 1, 128, 16, 4096, 512),
        ("cfg2 llama-8b b1 32K k2048", 1, 32, 8, 128, 16, 32768, 2048),
        ("cfg3 llama-8b b32 128K k2048", 32, 32, 8, 128, 16, 131072, 2048),
        ("cfg4 speech b64 60K d64 p32 k512", 64, 16, 16, 64, 32, 60000, 512),
    ]
    ctxs = [8192, 32768, 131072, 524288] if not quick else [32768, 131072]
    ratios = [64, 16, 8] if not quick else [64, 8]
    pages = [16, 32, 64] if not quick else [16, 64]
    for ctx in ctxs:
        batch = max(1, 32 * 131072 // ctx)  # ~4M tokens per kv-head set: 17 GB of KV at bf16
        for S in pages:
            for r in ratios:
                out.append((f"cfg5 ctx{ctx // 1024}K p{S} k=ctx/{r}", batch, 32, 8, 128, S, ctx,
                            ctx // r))
    return out


def main():
    import torch

    import bench
    import paper_2605_27740_b200 as pt

    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--only", default="")
    ap.add_argument("--no-mirror", action="store_true", help="exact f32-means scoring")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    peak = bench.measured_peaks()[0]["hbm_gbs"]

    def ev():
        return torch.cuda.Event(enable_timing=True)

    for name, B, Hq, Hkv, D, S, ctx, budget in configs(a.quick):
        if a.only and a.only not in name:
            continue
        G = Hq // Hkv
        kp = -(-budget // S)
        U = B * Hkv
        spare = 64 * 4 + 64
        P_cap = -(-(ctx + spare) // S)
        layout = pt.CacheLayout(num_kv_heads=Hkv, head_dim=D, page_size=S, max_pages=U * P_cap)
        kvdt = torch.float32 if name.startswith("cfg1") else torch.bfloat16  # cfg1: the f32 path
        cache = pt.PagedKvCache(layout, batch=B, dtype=kvdt, stats_dtype=torch.float32,
                                max_pages_per_head=P_cap, device=dev,
                                mirror=(not a.no_mirror) and kvdt == torch.bfloat16)
        g = torch.Generator(device=dev)
        g.manual_seed(1234)
        chunk = max(1, min(ctx, (1 << 27) // (U * D)))  # <= 256 MB of staging per tensor
        done, pre_ms = 0, 0.0
        while done < ctx:
            n = min(chunk, ctx - done)
            kk = torch.randn(U, n, D, generator=g, device=dev).to(kvdt)
            vv = torch.randn(U, n, D, generator=g, device=dev).to(kvdt)
            e0, e1 = ev(), ev()
            e0.record(stream)
            cache.extend_units(kk, vv)
            e1.record(stream)
            torch.cuda.synchronize()
            pre_ms += e0.elapsed_time(e1)
            done += n
            del kk, vv
        P = -(-ctx // S)
        # prefill bytes: staging K,V read + pool K,V written + stats written
        pre_bytes = U * (4 * ctx * D * 2 + P * (D * 4 + 4))
        eng = pt.DecodeEngine(cache, G, kp)
        q = torch.randn(U * G, D, generator=g, device=dev).to(kvdt)
        kn = torch.randn(U, D, generator=g, device=dev).to(kvdt)
        vn = torch.randn(U, D, generator=g, device=dev).to(kvdt)
        for _ in range(3):
            eng.step(q, kn, vn)
        torch.cuda.synchronize()
        eng.capture(q, kn, vn)
        for _ in range(3):
            eng.replay()
        e0, e1 = ev(), ev()
        e0.record(stream)
        for _ in range(a.steps):
            eng.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1000 / a.steps
        cache.check_errors()
        # per-stage device time: each stage captured alone as a CUDA graph, 20 replays
        brk = {}
        for nm, fn in (("append", lambda: cache.append_batch(kn, vn)),
                       ("lam_norms", lambda: eng.lam_norms(q)),
                       ("score", lambda: eng.score_step(q)),
                       ("select_attend", lambda: eng.select_attend(q))):
            fn()
            torch.cuda.synchronize()
            gs = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gs):
                fn()
            gs.replay()
            x0, x1 = ev(), ev()
            x0.record(stream)
            for _ in range(20):
                gs.replay()
            x1.record(stream)
            torch.cuda.synchronize()
            brk[nm] = x0.elapsed_time(x1) * 1000 / 20
            del gs
        cache._seq_host = cache.seq_lens.cpu().numpy().astype("int64")
        fused = eng.fused_attend
        bounded = bool(eng._step_bounded)
        for _ in range(2):
            eng.dense(q)
        d0, d1 = ev(), ev()
        d0.record(stream)
        for _ in range(5):
            eng.dense(q)
        d1.record(stream)
        torch.cuda.synchronize()
        dense_us = d0.elapsed_time(d1) * 1000 / 5
        N = int(cache.seq_lens.max().item())
        e = 4 if kvdt == torch.float32 else 2
        by = bench.step_bytes(U, G, D, -(-N // S), kp, S, e, e, N)  # e = KV element
        step_total = by["append"] + by["score"] + by["topk"] + by["attend"]
        sparse_us = brk["score"] + brk["select_attend"]
        print(json.dumps({
            "config": name, "batch": B, "q_heads": Hq, "kv_heads": Hkv, "head_dim": D, "page": S,
            "ctx": ctx, "k_pages": kp, "units": U,
            "us_per_step": us, "tokens_per_s": B / (us * 1e-6),
            "step_bytes": step_total, "step_frac_of_hbm": step_total / (us * 1e-6) / 1e9 / peak,
            "breakdown_us": brk, "fused_select_attend": fused, "scoring": "bounded" if bounded else "exact",
            "score_frac_of_hbm": by["score"] / (brk["score"] * 1e-6) / 1e9 / peak,
            "dense_us": dense_us, "x_over_dense": dense_us / sparse_us,
            "prefill_ms": pre_ms, "prefill_GBs": pre_bytes / (pre_ms * 1e-3) / 1e9,
            "peak_GBs": peak,
        }), flush=True)
        eng.graph = None
        del eng, cache, q, kn, vn
        import gc

        gc.collect()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
