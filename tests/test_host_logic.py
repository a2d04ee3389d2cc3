"""Host-side API pieces of the drop-in that need no GPU: types, validation, closed-form
traffic, key encoding, the standalone page table, regime labels (CPU only)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2605_27740_b200 as pt
from paper_2605_27740_b200 import select as sel


def test_layout_validation():
    with pytest.raises(ValueError, match="num_kv_heads"):
        pt.CacheLayout(num_kv_heads=0, head_dim=16)
    with pytest.raises(ValueError, match="head_dim"):
        pt.CacheLayout(num_kv_heads=1, head_dim=-1)
    with pytest.raises(ValueError, match="page_size"):
        pt.CacheLayout(num_kv_heads=1, head_dim=16, page_size=0)
    with pytest.raises(ValueError, match="max_pages"):
        pt.CacheLayout(num_kv_heads=1, head_dim=16, max_pages=0)
    lay = pt.CacheLayout(num_kv_heads=2, head_dim=16)
    assert (lay.page_size, lay.max_pages) == (8, 4096)
    with pytest.raises(AttributeError):
        lay.page_size = 4  # frozen


def test_decode_config():
    assert pt.DecodeConfig.from_budget(512, 8).k == 64
    assert pt.DecodeConfig.from_budget(513, 8).k == 65
    assert pt.DecodeConfig.from_budget(1, 8).k == 1
    assert pt.DecodeConfig.from_budget(2048, 16).k == 128  # cfg2/cfg3 budget
    assert pt.DecodeConfig().resolve_scale(16) == pytest.approx(0.25)
    assert pt.DecodeConfig(scale=2.0).resolve_scale(16) == 2.0
    with pytest.raises(ValueError, match="at least 1"):
        pt.DecodeConfig(k=0)
    with pytest.raises(ValueError):
        pt.DecodeConfig.from_budget(0, 8)


def test_traffic_closed_forms():
    for g, p, d in ((4, 1024, 128), (1, 1, 16), (8, 37, 64)):
        f = pt.traffic_of_fused(g, p, d)
        n = pt.traffic_of_naive(g, p, d)
        assert (f.scalar_reads, f.scalar_writes, f.launches) == (g * d + p * (d + 1), p, 1)
        assert n.scalar_reads - f.scalar_reads == 2 * g * p
        assert n.scalar_writes - f.scalar_writes == 2 * g * p
        assert n.launches == 3
    f = pt.traffic_of_fused(4, 1024, 128)
    assert (f.scalar_reads, f.scalar_writes) == (132608, 1024)
    for g in (1, 4, 8):
        assert pt.traffic_write_ratio(pt.traffic_of_naive(g, 2048, 128),
                                      pt.traffic_of_fused(g, 2048, 128)) == 2 * g + 1


def test_query_group():
    rng = np.random.default_rng(7)
    q = rng.standard_normal((4, 32)).astype(np.float32)
    g = pt.QueryGroup.from_queries(q)
    np.testing.assert_allclose(g.norms, np.linalg.norm(q.astype(np.float64), axis=1), rtol=1e-6)
    assert (g.group_size, g.head_dim) == (4, 32)
    assert pt.QueryGroup.from_queries(np.ones(8, np.float32)).queries.shape == (1, 8)
    with pytest.raises(ValueError):
        pt.QueryGroup.from_queries(np.zeros((0, 8), np.float32))


def test_query_norms_match_oracle(oracle):
    rng = np.random.default_rng(1)
    for _ in range(50):
        q = rng.standard_normal((int(rng.integers(1, 9)), int(rng.integers(1, 300)))).astype(np.float32)
        np.testing.assert_array_equal(pt.QueryGroup.from_queries(q).norms, oracle.query_norms(q))


def test_bf16_helpers_match_oracle(oracle):
    rng = np.random.default_rng(3)
    x = (rng.standard_normal(5000) * 10.0 ** rng.integers(-20, 20, 5000)).astype(np.float32)
    x[:3] = [np.nan, np.inf, -np.inf]
    np.testing.assert_array_equal(pt.f32_to_bf16(x), oracle.f32_to_bf16(x))
    bits = pt.f32_to_bf16(x[3:])
    np.testing.assert_array_equal(pt.f32_to_bf16(pt.bf16_to_f32(bits)), bits)
    np.testing.assert_array_equal(pt.is_nan_bf16(np.uint16([0x7F80, 0xFF80, 0x7FC0, 0x7F81, 1])),
                                  [False, False, True, True, False])


def test_encode_landmarks():
    seq = np.array([0xFF7F, 0xBF80, 0x8000, 0x0000, 0x3F80, 0x7F7F], dtype=np.uint16)
    keys = pt.encode_ordered(seq).astype(np.int64)
    assert np.all(np.diff(keys) > 0)
    with pytest.raises(ValueError, match="NaN"):
        pt.encode_ordered(np.array([0x7FC1], dtype=np.uint16))


def test_standalone_page_table():
    t = pt.PageTable(2)
    for pid in (40, 10, 30):
        t.append_page(0, pid)
    t.append_page(1, 7)
    assert t.num_pages(0) == 3 and t.num_pages(1) == 1
    np.testing.assert_array_equal(t.mapping(0), [40, 10, 30])
    assert t.physical(0, 1) == 10
    np.testing.assert_array_equal(t.to_logical(0, [30, 40]), [2, 0])
    with pytest.raises(LookupError):
        t.to_logical(0, [7])
    with pytest.raises(LookupError):
        t.physical(1, 1)
    with pytest.raises(ValueError, match="already mapped"):
        t.append_page(1, 40)
    with pytest.raises(ValueError):
        t.mapping(0)[0] = 1  # read-only view


def test_regime_labels():
    assert sel._regime(64) == "registers"
    assert sel._regime(pt.REGISTER_MAX_PAGES) == "registers"
    assert sel._regime(pt.REGISTER_MAX_PAGES + 1) == "staged"
    assert sel._regime(pt.STAGED_MAX_PAGES) == "staged"
    assert sel._regime(pt.STAGED_MAX_PAGES + 1) == "fallback"


def test_selection_errors_before_any_kernel():
    table = pt.PageTable(1)
    table.append_page(0, 0)
    one = pt.ScoreVector(0, np.float32([1.0]), pt.f32_to_bf16(np.float32([1.0])))
    with pytest.raises(ValueError, match="at least 1"):
        pt.radix_topk(one, 0, table, 0)
    empty = pt.ScoreVector(0, np.empty(0, np.float32), np.empty(0, np.uint16))
    with pytest.raises(ValueError, match="no pages"):
        pt.radix_topk(empty, 1, table, 0)
    with pytest.raises(ValueError, match="no pages"):
        pt.topk_fallback(empty, 1, table, 0)
    # take-all needs no kernel: P <= k returns every mapped page
    s = pt.radix_topk(one, 4, table, 0)
    assert list(s.physical_ids) == [0] and s.kplus1_score is None and s.passes == 1


def test_public_names_cover_the_reference_hot_path():
    for name in ("CacheLayout", "CapacityError", "PagedKvCache", "PageStats", "PageTable",
                 "compute_page_stats", "QueryGroup", "ScoreVector", "TrafficReport", "score_page",
                 "score_pages_grouped", "score_pages_naive", "traffic_of_fused",
                 "traffic_of_naive", "traffic_write_ratio", "TopKSelection", "encode_ordered",
                 "decode_ordered", "radix_topk", "topk_fallback", "AttentionOutput",
                 "DecodeConfig", "decode_step", "dense_attention", "sparse_attention",
                 "f32_to_bf16", "bf16_to_f32", "round_f32_to_bf16_value", "backend_name"):
        assert hasattr(pt, name), name
    assert pt.backend.NAME == "b200"
    for fn in ("fused_scores", "radix_select_desc", "stream_attention"):
        assert callable(getattr(pt.backend, fn))


def test_unqk_header_errors_raise_before_touching_a_device(tmp_path):
    """PagedKvCache.load rejects a bad magic / version (kvcache.py:326-330) with the
    reference's ValueError messages before any device allocation."""
    import struct

    import paper_2605_27740_b200 as pt

    bad = tmp_path / "bad.unqk"
    bad.write_bytes(b"XXXX" + struct.pack("<IIIII", 1, 1, 4, 2, 0))
    with pytest.raises(ValueError, match="bad snapshot magic"):
        pt.PagedKvCache.load(str(bad))
    bad.write_bytes(b"UNQK" + struct.pack("<IIIII", 99, 1, 4, 2, 0))
    with pytest.raises(ValueError, match="unsupported snapshot version"):
        pt.PagedKvCache.load(str(bad))


def test_reference_snapshot_fixture_header():
    """The committed reference-written snapshots parse as the reference's format."""
    import os
    import struct

    import numpy as np

    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    z = np.load(os.path.join(gold, "golden.npz"))
    for i in (0, 1):
        with open(os.path.join(gold, f"decode{i}.unqk"), "rb") as f:
            assert f.read(4) == b"UNQK"
            version, heads, dim, size, n = struct.unpack("<IIIII", f.read(20))
            body = np.frombuffer(f.read(), dtype="<f4")
        sn, sd, ss, shq, shkv, sk = z[f"decode{i}_shape"].tolist()
        assert (version, heads, dim, size, n) == (1, shkv, sd, ss, sn)
        np.testing.assert_array_equal(body.reshape(heads, 2, n, dim), z[f"decode{i}_kv"])
