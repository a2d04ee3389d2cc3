"""Generate tests/golden/recall_golden.npz from the LIVE reference (container only).

Run:  python tests/golden/make_recall_golden.py     (needs /root/reference and oracle/_ref)

Seeded dilution workloads from the reference's own generator (harness/workload.py:60-98) and
the reference's eval_recall (harness/recall.py:71-102) for every method: the GPU harness
(paper_2605_27740_b200.recall) must reproduce page_recall / mass_recall / output_err on the
same keys, values and queries.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import reference  # noqa: E402

CASES = [  # seed, n_tokens, head_dim, page_size, planted_pages, gain, k
    (11, 2048, 64, 16, 4, 6.0, 8),
    (12, 2048, 64, 16, 4, 6.0, 16),
    (13, 4000, 128, 16, 8, 8.0, 16),
    (14, 1024, 32, 8, 0, 6.0, 12),
    (15, 3000, 64, 32, 3, 5.0, 6),
]


def main() -> None:
    pt = reference.load("cython")
    assert pt.backend_name() == "cython", "build oracle/_ref first (make -C oracle ref)"
    from pagetopk.harness.recall import RECALL_METHODS, eval_recall
    from pagetopk.harness.workload import WorkloadSpec, gen_workload

    out: dict[str, np.ndarray] = {}
    for i, (seed, n, d, s, planted, gain, k) in enumerate(CASES):
        spec = WorkloadSpec(seed=seed, n_tokens=n, head_dim=d, page_size=s,
                            planted_pages=planted, planted_gain=gain)
        wl = gen_workload(spec)
        keys, values = wl.cache.full_kv(0)
        out[f"c{i}_spec"] = np.array([seed, n, d, s, planted, k], dtype=np.int64)
        out[f"c{i}_gain"] = np.float64(gain)
        out[f"c{i}_keys"] = keys.astype(np.float32)
        out[f"c{i}_values"] = values.astype(np.float32)
        out[f"c{i}_q"] = wl.queries[0].astype(np.float32)
        rep = np.zeros((len(RECALL_METHODS), 3), dtype=np.float64)
        for m, method in enumerate(RECALL_METHODS):
            r = eval_recall(method, wl, k)
            rep[m] = (r.page_recall, r.mass_recall, r.output_err)
        out[f"c{i}_reports"] = rep
    out["methods"] = np.array(RECALL_METHODS)
    np.savez_compressed(os.path.join(HERE, "recall_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "recall_golden.npz"), len(CASES), "cases")


if __name__ == "__main__":
    main()
