"""Pin the CPU oracle (oracle/pagetopk_oracle.c) before trusting it as the GPU checker.

* against the golden vectors produced by the live reference (tests/golden/golden.npz,
  made by tests/golden/make_golden.py from pagetopk + its compiled Cython backend):
  bit-exact for stats, norms, scores, bf16 keys, selections and attention;
* against the known-answer vectors of the reference's SPEC and unit tests;
* numpy's float64 summation order (the stats depend on it) against numpy itself.
CPU only.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def _count(prefix: str) -> int:
    return len({k.split("_")[0] for k in GOLD.files if k.startswith(prefix)})


def test_stats_golden(oracle):
    for i in range(_count("stats")):
        mean, std = oracle.compute_page_stats(GOLD[f"stats{i}_keys"])
        np.testing.assert_array_equal(mean, GOLD[f"stats{i}_mean"])
        assert np.float32(std) == GOLD[f"stats{i}_std"]


def test_scores_golden(oracle):
    for i in range(_count("score")):
        q = GOLD[f"score{i}_q"]
        norms = oracle.query_norms(q)
        np.testing.assert_array_equal(norms, GOLD[f"score{i}_norms"])
        s = oracle.fused_scores(q, norms, GOLD[f"score{i}_means"], GOLD[f"score{i}_stds"], 0.5)
        np.testing.assert_array_equal(s, GOLD[f"score{i}_f32"])
        np.testing.assert_array_equal(oracle.f32_to_bf16(s), GOLD[f"score{i}_bf16"])


def test_select_golden(oracle):
    for i in range(_count("select")):
        keys, k = GOLD[f"select{i}_keys"], int(GOLD[f"select{i}_k"])
        ids, thr, kp1, passes = oracle.radix_select_desc(keys, k)
        np.testing.assert_array_equal(np.sort(ids), GOLD[f"select{i}_ids"])
        assert [thr, kp1, passes] == GOLD[f"select{i}_meta"].tolist()


def test_attention_golden(oracle):
    for i in range(_count("attn")):
        o, lse = oracle.stream_attention(GOLD[f"attn{i}_q"], GOLD[f"attn{i}_K"], GOLD[f"attn{i}_V"],
                                         0.3, int(GOLD[f"attn{i}_block"]), GOLD[f"attn{i}_bias"])
        np.testing.assert_array_equal(o, GOLD[f"attn{i}_out"])
        assert lse == float(GOLD[f"attn{i}_lse"])


def test_decode_step_golden(oracle):
    for i in range(_count("decode")):
        n, d, s, hq, hkv, k = GOLD[f"decode{i}_shape"].tolist()
        kv = GOLD[f"decode{i}_kv"]  # [H, 2, n, d]
        P = -(-n // s)
        # pack each head's rows into its own pages (logical == physical order per head)
        kpool = np.zeros((hkv * P, s, d), np.float32)
        vpool = np.zeros_like(kpool)
        table = np.zeros((hkv, P), np.int32)
        for h in range(hkv):
            for p in range(P):
                r = min(s, n - p * s)
                kpool[h * P + p, :r] = kv[h, 0, p * s : p * s + r]
                vpool[h * P + p, :r] = kv[h, 1, p * s : p * s + r]
                table[h, p] = h * P + p
        seq = np.full(hkv, n, np.int32)
        means, stds = oracle.build_stats(kpool, table, seq, s)
        q = GOLD[f"decode{i}_q"].reshape(hkv, hq // hkv, d)
        r = oracle.decode_units(q, kpool, vpool, table, seq, means, stds, k, 0.5,
                                1.0 / np.sqrt(d), s)
        np.testing.assert_array_equal(r["out"].reshape(hq, d), GOLD[f"decode{i}_out"])
        np.testing.assert_array_equal(r["lse"].reshape(hq), GOLD[f"decode{i}_lse"])
        for h in range(hkv):
            logical = np.sort(r["sel"][h, : r["n_sel"][h]] - h * P)
            np.testing.assert_array_equal(logical, GOLD[f"decode{i}_sel"][h])


# ---------------------------------------------------------------------------
# known-answer vectors of the reference (SPEC.md, tests)
# ---------------------------------------------------------------------------
def test_spec_known_answers(oracle):
    mean, std = oracle.compute_page_stats(np.float32([[1, 0], [0, 1]]))
    np.testing.assert_array_equal(mean, np.float32([0.5, 0.5]))
    assert std == pytest.approx(0.70710677, rel=1e-7)
    q = np.float32([[1, 0]])  # SPEC.md:124 score of that page, lam 0.5
    s = oracle.fused_scores(q, oracle.query_norms(q), mean[None], np.float32([std]), 0.5)
    assert float(s[0]) == pytest.approx(0.85355341, rel=1e-7)
    keys = oracle.encode_ordered(oracle.f32_to_bf16(np.float32([3, 1, 4, 1, 5])))
    ids, thr, kp1, passes = oracle.radix_select_desc(keys, 2)
    assert set(ids.tolist()) == {2, 4} and passes == 3
    from paper_2605_27740_b200.bf16 import bf16_to_f32
    from paper_2605_27740_b200.select import decode_ordered

    assert float(bf16_to_f32(decode_ordered(np.uint16(thr)))) == 4.0
    assert float(bf16_to_f32(decode_ordered(np.uint16(kp1)))) == 3.0


BF16_KNOWN = [  # test_bf16.py:31-47
    (0.0, 0x0000), (-0.0, 0x8000), (1.0, 0x3F80), (-1.0, 0xBF80), (2.0, 0x4000),
    (1.00390625, 0x3F80), (1.01171875, 0x3F82), (1.0039066, 0x3F81),
    (3.4028234663852886e38, 0x7F80), (float("inf"), 0x7F80), (float("-inf"), 0xFF80),
]


def test_bf16_known_vectors(oracle):
    from paper_2605_27740_b200.bf16 import f32_to_bf16

    for v, bits in BF16_KNOWN:
        assert int(oracle.f32_to_bf16(np.float32([v]))[0]) == bits
        assert int(f32_to_bf16(np.float32([v]))[0]) == bits
    nan = oracle.f32_to_bf16(np.float32([np.nan]))[0]
    assert (nan & 0x7F80) == 0x7F80 and (nan & 0x7F)


def test_bf16_matches_ml_dtypes(oracle):
    ml = pytest.importorskip("ml_dtypes")
    rng = np.random.default_rng(2024)
    x = rng.standard_normal(20000).astype(np.float32)
    x *= np.float32(10.0) ** rng.integers(-18, 19, 20000).astype(np.float32)
    np.testing.assert_array_equal(oracle.f32_to_bf16(x), x.astype(ml.bfloat16).view(np.uint16))


def test_encode_order_exhaustive(oracle):
    from paper_2605_27740_b200.bf16 import EXPONENT_MASK, bf16_to_f32
    from paper_2605_27740_b200.select import decode_ordered, encode_ordered

    bits = np.arange(1 << 16, dtype=np.uint16)
    bits = bits[(bits & EXPONENT_MASK) != EXPONENT_MASK]
    keys = oracle.encode_ordered(bits)
    np.testing.assert_array_equal(keys, encode_ordered(bits))
    np.testing.assert_array_equal(decode_ordered(keys), bits)
    order = np.argsort(keys, kind="stable")
    vals = bf16_to_f32(bits[order]).astype(np.float64)
    assert np.all(np.diff(vals) >= 0)
    with pytest.raises(ValueError, match="NaN"):
        oracle.encode_ordered(np.uint16([0x7FC1]))


def test_numpy_summation_order(oracle):
    """The oracle's float64 reduction equals numpy's np.sum bit for bit."""
    rng = np.random.default_rng(0)
    for _ in range(2000):
        n = int(rng.integers(0, 600))
        a = rng.standard_normal(n) * 10.0 ** rng.integers(-4, 5, n)
        assert oracle.np_sum(a) == float(np.sum(a))


def test_radix_vs_stable_sort_random(oracle):
    """Criterion 2 of the reference acceptance suite, against a stable-sort oracle."""
    rng = np.random.default_rng(20241)
    for P in (128, 1024, 4096):
        for trial in range(60):
            vals = (rng.integers(-6, 7, P) if trial % 4 == 0 else
                    rng.standard_normal(P) * rng.choice([0.05, 1.0, 30.0])).astype(np.float32)
            keys = oracle.encode_ordered(oracle.f32_to_bf16(vals))
            ids, thr, kp1, _ = oracle.radix_select_desc(keys, 64)
            order = np.argsort(np.uint16(0xFFFF) - keys, kind="stable")
            np.testing.assert_array_equal(np.sort(ids), np.sort(order[:64]))
            assert thr == keys[order[63]] and kp1 == keys[order[64]]
