"""Generate tests/golden/golden.npz from the LIVE reference package (container only).

Run:  python tests/golden/make_golden.py     (needs /root/reference and oracle/_ref built)

Every vector is produced by the reference itself -- `pagetopk` imported from
/root/reference/pkg/src with its compiled Cython backend (oracle/_ref, built from
pkg/src/pagetopk/_kernels_cy.pyx by oracle/Makefile) -- so the committed fixtures pin
the oracle (and, through it, the GPU kernels) on boxes where the reference is absent.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import reference  # noqa: E402


def main() -> None:
    pt = reference.load("cython")
    assert pt.backend_name() == "cython", "build oracle/_ref first (make -C oracle ref)"
    from pagetopk import _kernels_cy as cy
    from pagetopk.harness.workload import WorkloadSpec, gen_workload

    rng = np.random.default_rng(20240)
    out: dict[str, np.ndarray] = {}

    # --- page statistics (kvcache.py:59-71)
    for i, (rows, d) in enumerate([(1, 16), (5, 16), (8, 24), (16, 128), (3, 128), (64, 64)]):
        keys = (rng.standard_normal((rows, d)) * rng.choice([0.01, 1.0, 50.0])).astype(np.float32)
        st = pt.compute_page_stats(keys)
        out[f"stats{i}_keys"] = keys
        out[f"stats{i}_mean"] = st.mean
        out[f"stats{i}_std"] = np.float32(st.std)

    # --- query norms + fused scores (scoring.py:39-47, _kernels_cy.pyx:19-43)
    for i, (g, p, d) in enumerate([(1, 37, 16), (4, 300, 128), (3, 64, 24), (8, 50, 64)]):
        q = rng.standard_normal((g, d)).astype(np.float32)
        grp = pt.QueryGroup.from_queries(q)
        means = rng.standard_normal((p, d)).astype(np.float32)
        stds = np.abs(rng.standard_normal(p)).astype(np.float32)
        sv = pt.score_pages_grouped(grp, (means, stds), 0.5)
        out[f"score{i}_q"] = q
        out[f"score{i}_norms"] = grp.norms
        out[f"score{i}_means"] = means
        out[f"score{i}_stds"] = stds
        out[f"score{i}_f32"] = sv.scores_f32
        out[f"score{i}_bf16"] = sv.scores_bf16

    # --- radix select (_kernels_cy.pyx:46-126), incl. dense ties
    for i, (p, k, kind) in enumerate([(5, 2, "spec"), (1024, 64, "ties"), (4096, 64, "normal"),
                                      (600, 599, "normal"), (2048, 128, "ties")]):
        if kind == "spec":
            vals = np.float32([3, 1, 4, 1, 5])
        elif kind == "ties":
            vals = rng.integers(-6, 7, p).astype(np.float32)
        else:
            vals = (rng.standard_normal(p) * 30).astype(np.float32)
        keys = pt.encode_ordered(pt.f32_to_bf16(vals))
        ids, thr, kp1, passes = cy.radix_select_desc(np.ascontiguousarray(keys), k)
        out[f"select{i}_keys"] = keys
        out[f"select{i}_k"] = np.int64(k)
        out[f"select{i}_ids"] = np.sort(ids)
        out[f"select{i}_meta"] = np.int64([thr, kp1, passes])

    # --- stream attention (_kernels_cy.pyx:129-172)
    for i, (n, d, block) in enumerate([(1, 24, 8), (65, 24, 8), (300, 64, 16), (123, 16, 7)]):
        q = rng.standard_normal(d).astype(np.float32)
        K = rng.standard_normal((n, d)).astype(np.float32)
        V = rng.standard_normal((n, d)).astype(np.float32)
        nb = -(-n // block)
        bias = rng.uniform(-3, 0, nb).astype(np.float32)
        o, lse = cy.stream_attention(q, K, V, np.float32(0.3), block, bias)
        out[f"attn{i}_q"], out[f"attn{i}_K"], out[f"attn{i}_V"] = q, K, V
        out[f"attn{i}_block"], out[f"attn{i}_bias"] = np.int64(block), bias
        out[f"attn{i}_out"], out[f"attn{i}_lse"] = o, np.float64(lse)

    # --- full decode_step (attention.py:110-147) on the reference workload generator
    for i, (n, d, s, hq, hkv, k) in enumerate([(400, 64, 16, 8, 2, 8), (333, 32, 8, 4, 1, 64)]):
        wl = gen_workload(WorkloadSpec(seed=31 + i, n_tokens=n, head_dim=d, page_size=s,
                                       num_query_heads=hq, num_kv_heads=hkv))
        outs, sels = pt.decode_step(wl.cache, wl.queries, pt.DecodeConfig(k=k))
        kv = np.stack([np.stack(wl.cache.full_kv(h)) for h in range(hkv)])  # [H, 2, n, d]
        out[f"decode{i}_shape"] = np.int64([n, d, s, hq, hkv, k])
        out[f"decode{i}_q"] = wl.queries
        out[f"decode{i}_kv"] = kv
        out[f"decode{i}_out"] = np.stack([o.out for o in outs])
        out[f"decode{i}_lse"] = np.float64([o.lse for o in outs])
        # logical ids of the selections (physical ids depend on allocation order)
        out[f"decode{i}_sel"] = np.stack([
            np.sort(wl.cache.table.to_logical(h, sels[h].physical_ids)) for h in range(hkv)])
        out[f"decode{i}_kth"] = np.float64([x.kth_score for x in sels])
        out[f"decode{i}_kp1"] = np.float64([np.nan if x.kplus1_score is None else x.kplus1_score
                                            for x in sels])
        # the reference's own cached page stats, and its UNQK snapshot of this cache
        # (kvcache.py:289-320): PagedKvCache.load must rebuild the same stats from it
        st = [wl.cache.stats_arrays(h) for h in range(hkv)]
        out[f"decode{i}_means"] = np.stack([x[0] for x in st])
        out[f"decode{i}_stds"] = np.stack([x[1] for x in st])
        out[f"decode{i}_counts"] = np.stack([x[2] for x in st]).astype(np.int64)
        snap = os.path.join(HERE, f"decode{i}.unqk")
        wl.cache.save(snap)
        # the reference's load -> save round trip is byte-identical
        rt = snap + ".rt"
        pt.PagedKvCache.load(snap).save(rt)
        with open(snap, "rb") as a, open(rt, "rb") as b:
            assert a.read() == b.read()
        os.remove(rt)

    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
