"""The oracle against the LIVE reference (build container only; skipped elsewhere).

Bit-exactness of oracle/pagetopk_oracle.c against the reference's own compiled
backend (pkg/src/pagetopk/_kernels_cy.pyx built into oracle/_ref) and its numpy
statistics, on randomized inputs -- the restatement is the checker for the GPU.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import reference

pytestmark = pytest.mark.skipif(not reference.available(), reason="/root/reference absent")


@pytest.fixture(scope="module")
def ref():
    pt = reference.load("cython")
    if pt.backend_name() != "cython":
        pytest.skip("reference compiled backend not built (make -C oracle ref)")
    return pt


def test_page_stats_bit_exact(ref, oracle):
    rng = np.random.default_rng(1)
    for _ in range(300):
        rows, d = int(rng.integers(1, 70)), int(rng.choice([4, 16, 24, 64, 128, 200]))
        keys = (rng.standard_normal((rows, d)) * 10.0 ** rng.integers(-3, 3)).astype(np.float32)
        st = ref.compute_page_stats(keys)
        mean, std = oracle.compute_page_stats(keys)
        np.testing.assert_array_equal(mean, st.mean)
        assert std == st.std


def test_kernels_bit_exact(ref, oracle):
    from pagetopk import _kernels_cy as cy

    rng = np.random.default_rng(2)
    for _ in range(100):
        g, p, d = int(rng.integers(1, 9)), int(rng.integers(1, 400)), int(rng.integers(1, 140))
        q = rng.standard_normal((g, d)).astype(np.float32)
        grp = ref.QueryGroup.from_queries(q)
        np.testing.assert_array_equal(oracle.query_norms(q), grp.norms)
        means = rng.standard_normal((p, d)).astype(np.float32)
        stds = np.abs(rng.standard_normal(p)).astype(np.float32)
        np.testing.assert_array_equal(oracle.fused_scores(q, grp.norms, means, stds, 0.5),
                                      cy.fused_scores(q, grp.norms, means, stds, np.float32(0.5)))
    for _ in range(100):
        p = int(rng.integers(2, 5000))
        k = int(rng.integers(1, p))
        vals = (rng.integers(-6, 7, p) if rng.random() < 0.3 else
                rng.standard_normal(p) * 30).astype(np.float32)
        keys = np.ascontiguousarray(ref.encode_ordered(ref.f32_to_bf16(vals)))
        a = oracle.radix_select_desc(keys, k)
        b = cy.radix_select_desc(keys, k)
        np.testing.assert_array_equal(a[0], b[0])  # same emission order
        assert a[1:] == tuple(b[1:])
    for _ in range(60):
        n, d, block = int(rng.integers(1, 500)), int(rng.integers(1, 130)), int(rng.integers(1, 33))
        q = rng.standard_normal(d).astype(np.float32)
        K = rng.standard_normal((n, d)).astype(np.float32)
        V = rng.standard_normal((n, d)).astype(np.float32)
        bias = rng.uniform(-3, 0, -(-n // block)).astype(np.float32)
        o, lse = oracle.stream_attention(q, K, V, 0.17, block, bias)
        o2, lse2 = cy.stream_attention(q, K, V, np.float32(0.17), block, bias)
        np.testing.assert_array_equal(o, o2)
        assert lse == lse2


def test_decode_step_bit_exact(ref, oracle):
    from pagetopk.harness.workload import WorkloadSpec, gen_workload

    rng = np.random.default_rng(3)
    for trial in range(8):
        hkv = int(rng.choice([1, 2, 4]))
        g = int(rng.choice([1, 2, 4]))
        s = int(rng.choice([8, 16, 32]))
        n = int(rng.integers(s, 3000))
        d = int(rng.choice([16, 64, 128]))
        k = int(rng.integers(1, 40))
        wl = gen_workload(WorkloadSpec(seed=100 + trial, n_tokens=n, head_dim=d, page_size=s,
                                       num_query_heads=hkv * g, num_kv_heads=hkv))
        c = wl.cache
        outs, sels = ref.decode_step(c, wl.queries, ref.DecodeConfig(k=k))
        kpool = np.stack(c._page_keys)
        vpool = np.stack(c._page_values)
        table = np.stack([c.table.mapping(h) for h in range(hkv)]).astype(np.int32)
        seq = np.full(hkv, n, np.int32)
        means, stds = oracle.build_stats(kpool, table, seq, s)
        for h in range(hkv):
            m, sd, _ = c.stats_arrays(h)
            np.testing.assert_array_equal(means[h], m)
            np.testing.assert_array_equal(stds[h], sd)
        r = oracle.decode_units(wl.queries.reshape(hkv, g, d), kpool, vpool, table, seq, means,
                                stds, k, 0.5, 1.0 / np.sqrt(d), s)
        for h in range(hkv):
            np.testing.assert_array_equal(r["sel"][h, : r["n_sel"][h]], sels[h].physical_ids)
        for i, o in enumerate(outs):
            np.testing.assert_array_equal(r["out"].reshape(-1, d)[i], o.out)
            assert r["lse"].reshape(-1)[i] == o.lse
