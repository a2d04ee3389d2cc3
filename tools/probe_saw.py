"""Phase timeline of the warp-per-unit select+attend (tuning aid, cfg4 shape by default):
per-warp %clock64 stamps (PT_SA_PROF=2) -> median cycles / us from each warp's entry to
after the PDL wait, the selection, the first page, the stream's end and the exit."""
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
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--ctx", type=int, default=60000)
    ap.add_argument("--q-heads", type=int, default=16)
    ap.add_argument("--kv-heads", type=int, default=16)
    ap.add_argument("--head-dim", type=int, default=64)
    ap.add_argument("--page", type=int, default=32)
    ap.add_argument("--budget", type=int, default=512)
    ap.add_argument("--bounded", action="store_true")
    a = ap.parse_args()
    if a.bounded:
        os.environ["PT_BOUNDED"] = "1"
    ns = argparse.Namespace(batch=a.batch, ctx=a.ctx, q_heads=a.q_heads, kv_heads=a.kv_heads,
                            head_dim=a.head_dim, page=a.page, budget=a.budget, stats_dtype="f32",
                            warmup=3, steps=10)
    dev = torch.device("cuda", 0)
    cache = bench.build_cache(ns, dev, seed=1234)
    G, D = a.q_heads // a.kv_heads, a.head_dim
    U = cache.num_units
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    q = torch.randn(U * G, D, generator=g, device=dev).to(torch.bfloat16)
    eng = pt.DecodeEngine(cache, G, a.budget // a.page)
    for _ in range(3):
        eng.lam_norms(q)
        eng.score_step(q)
        eng.select_attend(q)
    torch.cuda.synchronize()
    stats = {}
    if eng._step_bounded:
        k = a.budget // a.page
        klo = eng.keys.cpu().numpy().view(np.uint16).astype(np.int64)
        khi = eng.keys_hi.cpu().numpy().view(np.uint16).astype(np.int64)
        P = cache.num_pages(0)
        lo_, hi_ = klo[:, :P], khi[:, :P]
        A = -np.sort(-lo_, axis=1)[:, k]
        B = -np.sort(-hi_, axis=1)[:, k - 1]
        br = (lo_ != hi_) & (hi_ >= A[:, None]) & (lo_ <= B[:, None])
        stats = {"pages": P, "k": k, "unsure_frac": float((lo_ != hi_).mean()),
                 "bracket_per_unit_mean": float(br.sum(1).mean()),
                 "bracket_per_unit_max": int(br.sum(1).max()),
                 "bracket_width_keys_mean": float((B - A).mean())}
    os.environ["PT_SA_PROF"] = "2"
    eng.select_attend(q)
    torch.cuda.synchronize()
    os.environ.pop("PT_SA_PROF")
    n = min(U, 4096)
    buf = np.zeros(n * 20, dtype=np.uint64)
    _lib.check(_lib.load().pt_debug_sa_prof(buf.ctypes.data, n * 20))
    raw = buf.reshape(n, 20).astype(np.int64)
    try:
        import pynvml

        pynvml.nvmlInit()
        mhz = pynvml.nvmlDeviceGetClockInfo(pynvml.nvmlDeviceGetHandleByIndex(0), pynvml.NVML_CLOCK_SM)
    except Exception:
        mhz = 1965
    names = ["entry", "after_wait", "selected", "first_page", "stream_done", "exit",
             "sw_keys_issued", "sw_tile_bound", "sw_bracket", "sw_resolved", "", "sw_minmax",
             "sw_threshold", "sw_counts", "sw_compacted"]
    out = {"shape": vars(a), "bounded": bool(eng._step_bounded), "units": U, "sm_mhz": mhz,
           "resolve": stats,
           "note": "median over warps of (stamp - the warp's entry)"}
    cyc = {}
    for i, nm in enumerate(names):
        if not nm:
            continue
        d = raw[:, i] - raw[:, 0]
        ok = (d >= 0) & (d < 10**8)
        cyc[nm] = int(np.median(d[ok])) if ok.any() else None
    out["cycles"] = cyc
    out["us"] = {k: (round(v / mhz, 3) if v is not None else None) for k, v in cyc.items()}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
