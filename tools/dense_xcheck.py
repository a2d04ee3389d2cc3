"""Cross-check of the speed-up denominator: our dense paged decode (K4 in
dense mode) against flashinfer's BatchDecodeWithPagedKVCacheWrapper on the SAME pool at the
headline shape -- each (sequence, kv-head) unit as one flashinfer request with 1 kv head and
G query heads over the unit's pages (our pool layout [pages][S][D] is flashinfer's NHD layout
with one head).  Reports both kernels' times and the max output difference.  Library code,
tool only (not on the decode path).

    python tools/dense_xcheck.py [--batch 32 --ctx 131072]
"""
import argparse
import json
import math
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
    a = ap.parse_args()
    args = bench.parse(["--batch", str(a.batch), "--ctx", str(a.ctx), "--steps", "1", "--warmup", "1"])
    dev = torch.device("cuda", 0)
    cache = bench.build_cache(args, dev, bench.SEED)
    G, D, S = args.q_heads // args.kv_heads, args.head_dim, args.page
    U = cache.num_units
    eng = pt.DecodeEngine(cache, G, args.budget // S)
    qs, _, _ = bench.step_inputs(args, dev)
    q = qs[0]
    st = torch.cuda.current_stream()

    def timeit(fn, reps=20):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1000 / reps

    ours_us = timeit(lambda: eng.dense(q))
    ours = eng.dense_out.clone()
    res = {"shape": vars(a), "ours_dense_us": ours_us}
    try:
        import flashinfer

        P = -(-a.ctx // S)
        table = cache.page_table[:, :P].contiguous()
        indices = table.reshape(-1).to(torch.int32)
        indptr = torch.arange(0, U * P + 1, P, dtype=torch.int32, device=dev)
        last = torch.full((U,), a.ctx - (P - 1) * S, dtype=torch.int32, device=dev)
        ws = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(ws, "NHD")
        w.plan(indptr, indices, last, G, 1, D, S, pos_encoding_mode="NONE",
               q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16, sm_scale=1.0 / math.sqrt(D))
        kc = cache.k_pool.view(-1, S, 1, D)
        vc = cache.v_pool.view(-1, S, 1, D)
        q3 = q.view(U, G, D)
        fi_us = timeit(lambda: w.run(q3, (kc, vc)))
        out = w.run(q3, (kc, vc)).float().reshape(U * G, D)
        res.update(flashinfer=flashinfer.__version__, flashinfer_us=fi_us,
                   max_abs_diff=float((out - ours).abs().max()), ours_over_flashinfer=fi_us / ours_us,
                   bytes=2 * U * a.ctx * D * 2, ours_TBs=2 * U * a.ctx * D * 2 / ours_us / 1e6,
                   flashinfer_TBs=2 * U * a.ctx * D * 2 / fi_us / 1e6)
    except Exception as e:  # noqa: BLE001
        res["flashinfer_error"] = repr(e)[:400]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
