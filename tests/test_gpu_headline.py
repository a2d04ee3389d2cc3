"""Parity at the headline configuration itself (BASELINE configs[2]: B=32, 128K context,
32q/8kv, d=128, page 16, k = 2048 tokens, bf16 KV): the bench's own workload and engine,
one decode step after appends, compared with the oracle's restatement of
attention.py:110-147 on a sampled 2 sequences x 8 kv-heads (a full f32 oracle
batch would be ~32 GB).  Selections bit-exact, kth / kplus1 equal, outputs within 2e-2
(bf16), for both scoring modes: bounded (bf16 mirror + exact resolution, the bench default)
and exact f32 means."""

from __future__ import annotations

import gc

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mirror", [True, False])
def test_cfg3_sample_matches_oracle(cuda, mirror):
    import bench
    import paper_2605_27740_b200 as pt

    args = bench.parse(["--steps", "4", "--warmup", "3"] + ([] if mirror else ["--no-mirror"]))
    G = args.q_heads // args.kv_heads
    kp = -(-args.budget // args.page)
    cache = bench.build_cache(args, cuda, bench.SEED)
    eng = pt.DecodeEngine(cache, G, kp)
    qs, kn, vn = bench.step_inputs(args, cuda)
    for i in range(3):  # appends: a fresh tail page plus rows on it
        eng.step(qs[i], kn, vn)
    torch.cuda.synchronize()
    cache.check_errors()
    res, _ = bench.parity_check(eng, cache, qs[3], args)  # raises on any mismatch
    assert eng._step_bounded == mirror
    assert res["units"] == 16 and res["selection_mismatches"] == 0
    assert res["kth_equal"] and res["kplus1_equal"] and res["out_max_abs_err"] <= 2e-2
    del eng, cache
    gc.collect()
    torch.cuda.empty_cache()
