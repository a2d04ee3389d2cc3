"""Phase timeline of the fused select+attend kernel (tuning aid): per-CTA %globaltimer
stamps -> percentiles of each phase boundary relative to the earliest CTA entry."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def eng_nchunk(U, k):
    """chunks per unit of the fused kernel's grid (attend_fused.cu: 2 CTAs per SM, at least
    4 pages per streaming warp per chunk)"""
    import torch

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = max(1, (sms * 2) // U)
    return min(n, (k + 15) // 16)


def main():
    import torch

    import bench
    import paper_2605_27740_b200 as pt
    from paper_2605_27740_b200 import _lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--budget", type=int, default=2048)
    ap.add_argument("--exact", action="store_true", help="exact f32-means keys (no mirror)")
    ap.add_argument("--clock", action="store_true",
                    help="%%clock64 stamps: per-CTA phase durations in SM cycles (fine-grained)")
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
    if a.exact:
        eng.bounded = False
    eng.lam_norms(q)
    eng.score_step(q)
    stats = {"bounded": bool(eng._step_bounded)}
    if eng._step_bounded:
        # how many pages the selection must resolve: interval not one key and reaching L
        # (the (k+1)-th largest tile maximum of the lower keys)
        k = a.budget // S
        klo = eng.keys.cpu().numpy().view(np.uint16).astype(np.int64)
        khi = eng.keys_hi.cpu().numpy().view(np.uint16).astype(np.int64)
        tm = eng.tile_max.cpu().numpy().view(np.uint16).astype(np.int64)
        P = cache.num_pages(0)
        nt = -(-P // 32)
        L = -np.sort(-tm[:, :nt], axis=1)[:, k]
        unsure = klo[:, :P] != khi[:, :P]
        reach = khi[:, :P] >= L[:, None]
        stats["unsure_frac"] = float(unsure.mean())
        stats["cand_per_unit"] = float(reach.sum(1).mean())
        stats["resolve_per_unit_mean"] = float((unsure & reach).sum(1).mean())
        stats["resolve_per_unit_max"] = int((unsure & reach).sum(1).max())
        stats["exact_ge_L_per_unit"] = float((klo[:, :P] >= L[:, None]).sum(1).mean())
        stats["width_keys_mean"] = float((khi[:, :P] - klo[:, :P]).mean())
        # bracket: A = (k+1)-th largest lower key <= exact (k+1)-th key, B = k-th largest upper
        # key >= the threshold; only intervals meeting [A, B] matter
        A = -np.sort(-klo[:, :P], axis=1)[:, k]
        Bq = -np.sort(-khi[:, :P], axis=1)[:, k - 1]
        br = unsure & (khi[:, :P] >= A[:, None]) & (klo[:, :P] <= Bq[:, None])
        stats["bracket_per_unit_mean"] = float(br.sum(1).mean())
        stats["bracket_per_unit_max"] = int(br.sum(1).max())
        stats["bracket_width_keys_mean"] = float((Bq - A).mean())
    for _ in range(3):
        eng.select_attend(q)
    torch.cuda.synchronize()
    os.environ["PT_SA_PROF"] = "2" if a.clock else "1"
    eng.select_attend(q)
    torch.cuda.synchronize()
    os.environ.pop("PT_SA_PROF")
    nch = int(eng_nchunk(U, a.budget // S))
    n = U * nch * 20
    buf = np.zeros(n, dtype=np.uint64)
    _lib.check(_lib.load().pt_debug_sa_prof(buf.ctypes.data, n))
    raw = buf.reshape(U * nch, 20)
    t = raw[:, :15].astype(np.float64)
    # stamps 10..13: resolve start / scan done / rows staged / resolved; 14: khi+q staged;
    # 15: rounds * 1e6 + pages listed in the last round
    info = raw[:, 15]
    t0 = t[:, 0].min()
    T = lambda i: (raw[:, i].astype(np.float64) - t0) / 1000.0  # noqa: E731
    rel = (t - t0) / 1000.0
    names = ["entry", "keys_staged", "selected", "first_page", "stream_done", "exit",
             "sel_loads_max", "sel_L", "sel_cands", "sel_thr", "res_start", "res_scan", "res_staged",
             "res_done", "bnd_staged"]
    out = {"resolve": stats}
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
    if stats.get("bounded"):
        out["durations_us_median"].update({
            "bnd_khi_q_staged": float(np.median(rel[:, 14] - rel[:, 1])),
            "res_scan": float(np.median(rel[:, 11] - rel[:, 10])),
            "res_stage": float(np.median(rel[:, 12] - rel[:, 11])),
            "res_compute": float(np.median(rel[:, 13] - rel[:, 12])),
            "res_total": float(np.median(rel[:, 13] - rel[:, 10])),
            "L_before_resolve": float(np.median(rel[:, 10] - rel[:, 14])),
            "b_cand_pass": float(np.median(T(16) - rel[:, 6])),
            "b_mxh": float(np.median(T(17) - T(16))),
            "b_histB": float(np.median(T(18) - T(17))),
            "b_histA": float(np.median(T(19) - T(18))),
            "b_to_resolve": float(np.median(rel[:, 10] - T(19))),
        })

    if a.clock:
        # per-CTA deltas from the CTA's own entry stamp (clocks are per SM), in cycles and in
        # us at the SM clock read during the run
        try:
            import pynvml

            pynvml.nvmlInit()
            mhz = pynvml.nvmlDeviceGetClockInfo(pynvml.nvmlDeviceGetHandleByIndex(0), pynvml.NVML_CLOCK_SM)
        except Exception:
            mhz = 1965
        out = {"resolve": stats, "sm_mhz": mhz, "note": "median over CTAs of (stamp - entry), cycles"}
        ent = raw[:, 0].astype(np.int64)
        cyc = {}
        for i, nm in enumerate(names + ["", "b_cand_pass", "b_mxh", "b_hist", "b_hist2"]):
            if not nm or i >= 20:
                continue
            d = raw[:, i].astype(np.int64) - ent
            ok = (d >= 0) & (d < 10**8)
            if ok.any():
                cyc[nm] = int(np.median(d[ok]))
        out["cycles"] = cyc
        out["us"] = {k2: round(v / mhz, 3) for k2, v in cyc.items()}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
