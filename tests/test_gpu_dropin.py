"""The reference-signature drop-in API on the GPU, against the reference's own outputs.

Every expected value here was produced by the live reference package (tests/golden/
make_golden.py: `pagetopk` with its compiled backend) -- not by this repo's oracle:

* ``decode_step`` (reference attention.py:110-147) on the reference's decode workloads,
  loaded from the reference's own UNQK snapshots (kvcache.py:289-341) through
  ``PagedKvCache.load``: outputs, lse, logical selections, kth / kplus1;
* ``PagedKvCache.load``: page stats bit-exact with the reference cache's, ``full_kv``
  byte-identical, ``save`` round-trips the snapshot byte for byte;
* ``score_pages_grouped`` / ``radix_topk`` / ``sparse_attention`` / per-head
  ``append`` / ``extend`` through the package API (scoring.py:108-124, select.py:87-115,
  attention.py:94-107, kvcache.py:185-233);
* the naive three-launch scorer at the reference's own tolerance (test_scoring.py:88-101).
"""

from __future__ import annotations

import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "golden.npz"))


def _pt():
    import paper_2605_27740_b200 as pt

    return pt


@pytest.mark.parametrize("i", [0, 1])
def test_unqk_snapshot_load_stats_and_round_trip(cuda, gold, i, tmp_path):
    pt = _pt()
    path = os.path.join(GOLD, f"decode{i}.unqk")
    cache = pt.PagedKvCache.load(path)
    n, d, s, hq, hkv, k = gold[f"decode{i}_shape"].tolist()
    assert cache.num_units == hkv and cache.layout.head_dim == d and cache.layout.page_size == s
    for h in range(hkv):
        assert cache.seq_len(h) == n
        keys, values = cache.full_kv(h)
        np.testing.assert_array_equal(keys, gold[f"decode{i}_kv"][h, 0])
        np.testing.assert_array_equal(values, gold[f"decode{i}_kv"][h, 1])
        means, stds, counts = cache.stats_arrays(h)
        np.testing.assert_array_equal(means, gold[f"decode{i}_means"][h])
        np.testing.assert_array_equal(stds, gold[f"decode{i}_stds"][h])
        np.testing.assert_array_equal(counts, gold[f"decode{i}_counts"][h])
    out = tmp_path / "rt.unqk"
    cache.save(str(out))
    with open(path, "rb") as a, open(out, "rb") as b:
        assert a.read() == b.read()


@pytest.mark.parametrize("i", [0, 1])
def test_decode_step_reference_signature_on_reference_snapshot(cuda, gold, i):
    """pt.decode_step(cache, queries, DecodeConfig(k)) == the reference's decode_step."""
    pt = _pt()
    cache = pt.PagedKvCache.load(os.path.join(GOLD, f"decode{i}.unqk"))
    n, d, s, hq, hkv, k = gold[f"decode{i}_shape"].tolist()
    outs, sels = pt.decode_step(cache, gold[f"decode{i}_q"], pt.DecodeConfig(k=k))
    assert len(outs) == hq and len(sels) == hkv
    np.testing.assert_allclose(np.stack([o.out for o in outs]), gold[f"decode{i}_out"],
                               rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose([o.lse for o in outs], gold[f"decode{i}_lse"], rtol=1e-5)
    for h in range(hkv):
        logical = np.sort(cache.table.to_logical(h, sels[h].physical_ids))
        np.testing.assert_array_equal(logical, gold[f"decode{i}_sel"][h])
        assert sels[h].kth_score == gold[f"decode{i}_kth"][h]
        kp1 = gold[f"decode{i}_kp1"][h]
        if np.isnan(kp1):
            assert sels[h].kplus1_score is None
        else:
            assert sels[h].kplus1_score == kp1


@pytest.mark.parametrize("i", [0, 1, 2, 3])
def test_score_pages_grouped_api(cuda, gold, i):
    pt = _pt()
    g = pt.QueryGroup.from_queries(gold[f"score{i}_q"])
    np.testing.assert_array_equal(g.norms, gold[f"score{i}_norms"])
    sv = pt.score_pages_grouped(g, (gold[f"score{i}_means"], gold[f"score{i}_stds"]), 0.5)
    np.testing.assert_array_equal(sv.scores_f32, gold[f"score{i}_f32"])
    np.testing.assert_array_equal(sv.scores_bf16, gold[f"score{i}_bf16"])


@pytest.mark.parametrize("i", [0, 1, 2, 3, 4])
def test_radix_topk_api(cuda, gold, i):
    pt = _pt()
    keys = gold[f"select{i}_keys"]
    k = int(gold[f"select{i}_k"])
    P = keys.shape[0]
    bits = pt.decode_ordered(keys)
    sv = pt.ScoreVector(head=0, scores_f32=pt.bf16_to_f32(bits), scores_bf16=bits)
    table = pt.PageTable(1)
    # physical = logical + 1000: the selection must come back translated
    for p in range(P):
        table.append_page(0, 1000 + p)
    sel = pt.radix_topk(sv, k, table, 0)
    np.testing.assert_array_equal(np.sort(sel.physical_ids), gold[f"select{i}_ids"] + 1000)
    thr, kp1, passes = gold[f"select{i}_meta"].tolist()
    from paper_2605_27740_b200.select import key_to_score

    assert sel.kth_score == key_to_score(thr) and sel.kplus1_score == key_to_score(kp1)
    assert sel.passes == passes


def test_sparse_attention_and_per_head_append_extend(cuda, oracle):
    """Per-head append / extend on the device cache keep stats bit-exact with the reference
    restatement; sparse_attention over a selection equals the reference stream over the
    gathered rows (attention.py:94-107)."""
    pt = _pt()
    rng = np.random.default_rng(77)
    D, S, H = 64, 16, 3
    layout = pt.CacheLayout(num_kv_heads=H, head_dim=D, page_size=S, max_pages=H * 20)
    cache = pt.PagedKvCache(layout, max_pages_per_head=20)
    for h in range(H):
        rows = rng.standard_normal((37 + 5 * h, D)).astype(np.float32)
        cache.extend(h, rows, -rows)
        for _ in range(4 + h):
            r = rng.standard_normal(D).astype(np.float32)
            cache.append(h, r, r * 2)
    for h in range(H):
        keys, _ = cache.full_kv(h)
        means, stds, counts = cache.stats_arrays(h)
        for p in range(cache.num_pages(h)):
            rows = keys[p * S:(p + 1) * S]
            want_mean, want_std = oracle.compute_page_stats(rows)  # kvcache.py:59-71
            np.testing.assert_array_equal(means[p], want_mean)
            assert stds[p] == np.float32(want_std) and counts[p] == rows.shape[0]
    h = 1
    q = rng.standard_normal(D).astype(np.float32)
    mapping = cache.table.mapping(h)
    pick = np.asarray([mapping[0], mapping[-1], mapping[1]], dtype=np.int64)
    sel = pt.TopKSelection(physical_ids=pick, kth_score=0.0, kplus1_score=None, regime="registers",
                           passes=1)
    got = pt.sparse_attention(q, cache, h, sel)
    kk, vv = cache.gather_pages(h, pick)
    out, lse = oracle.stream_attention(q, kk, vv, 1.0 / math.sqrt(D), S)
    np.testing.assert_allclose(got.out, out, rtol=1e-5, atol=1e-5)
    assert got.lse == pytest.approx(lse, rel=1e-5)
    with pytest.raises(ValueError, match="empty selection"):
        pt.sparse_attention(q, cache, h, pt.TopKSelection(np.empty(0, np.int64), 0.0, None, "registers", 1))
    with pytest.raises(LookupError):
        pt.sparse_attention(q, cache, 0, sel)  # pages of head 1


def test_naive_scorer_matches_fused_at_reference_tolerance(cuda):
    """score_pages_naive (3 launches on the GPU) vs the fused K2 scores, the reference's
    test_scoring.py:88-101 check (rtol 1e-5, atol 1e-6) -- the comparison behind
    profiles/r01/table5_r01e.json (paper Table 5) -- plus the exact traffic counts."""
    pt = _pt()
    rng = np.random.default_rng(1234 + 3)
    for trial in range(10):
        n_pages = int(rng.integers(1, 200))
        g = int(rng.integers(1, 5))
        means = rng.standard_normal((n_pages, 64)).astype(np.float32)
        stds = np.abs(rng.standard_normal(n_pages)).astype(np.float32)
        group = pt.QueryGroup.from_queries(rng.standard_normal((g, 64)).astype(np.float32))
        fused = pt.score_pages_grouped(group, (means, stds), 0.5)
        naive, traffic = pt.score_pages_naive(group, (means, stds), 0.5)
        np.testing.assert_allclose(fused.scores_f32, naive.scores_f32, rtol=1e-5, atol=1e-6)
        assert traffic == pt.traffic_of_naive(g, n_pages, 64)
