"""Generate tests/golden/softmask_golden.npz from the LIVE reference (container only).

Run:  python tests/golden/make_softmask_golden.py

Seeded small caches (the reference's own workload generator) and the reference's float64
decode_train_step (softmask.py:357-521) in soft and hard mode; the GPU training path
(paper_2605_27740_b200.softmask) must reproduce loss, outputs and every gradient to the
f32-vs-f64 tolerance stated in the test.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import reference  # noqa: E402

CASES = [  # seed, n_tokens, head_dim, page, q_heads, kv_heads, k, tau, mode, standardize
    (31, 150, 32, 8, 4, 2, 5, 1.0, "soft", True),
    (32, 203, 64, 16, 2, 2, 4, 0.5, "soft", False),
    (33, 120, 32, 8, 4, 2, 6, 1.0, "hard", True),
    (34, 64, 16, 8, 2, 1, 8, 1.0, "soft", True),   # P <= k: all gates one, no score gradient
]


def main() -> None:
    reference.load("cython")
    from pagetopk.harness.workload import WorkloadSpec, gen_workload
    from pagetopk.softmask import GateConfig, decode_train_step

    out: dict[str, np.ndarray] = {}
    for i, (seed, n, d, s, hq, hkv, k, tau, mode, std) in enumerate(CASES):
        wl = gen_workload(WorkloadSpec(seed=seed, n_tokens=n, head_dim=d, page_size=s,
                                       num_query_heads=hq, num_kv_heads=hkv))
        rng = np.random.default_rng(seed + 1000)
        target = rng.standard_normal((hq, d)).astype(np.float32)
        cfg = GateConfig(k=k, tau=tau, mode=mode, standardize=std)
        r = decode_train_step(wl.cache, wl.queries, cfg, target)
        out[f"c{i}_spec"] = np.array([seed, n, d, s, hq, hkv, k], dtype=np.int64)
        out[f"c{i}_cfg"] = np.array([tau, 1.0 if mode == "hard" else 0.0, 1.0 if std else 0.0])
        out[f"c{i}_q"] = wl.queries
        out[f"c{i}_target"] = target
        for h in range(hkv):
            kk, vv = wl.cache.full_kv(h)
            out[f"c{i}_k{h}"] = kk.astype(np.float32)
            out[f"c{i}_v{h}"] = vv.astype(np.float32)
            out[f"c{i}_dk{h}"] = r.d_keys[h]
            out[f"c{i}_dv{h}"] = r.d_values[h]
            out[f"c{i}_ds{h}"] = r.d_scores[h]
            out[f"c{i}_dm{h}"] = r.d_means[h]
            out[f"c{i}_dstd{h}"] = r.d_stds[h]
            out[f"c{i}_gates{h}"] = r.gates[h]
        out[f"c{i}_loss"] = np.float64(r.loss)
        out[f"c{i}_out"] = np.stack([o.out for o in r.outputs])
        out[f"c{i}_lse"] = np.array([o.lse for o in r.outputs])
        out[f"c{i}_dq"] = r.d_queries
    np.savez_compressed(os.path.join(HERE, "softmask_golden.npz"), **out)
    print("wrote softmask_golden.npz with", len(CASES), "cases")


if __name__ == "__main__":
    main()
