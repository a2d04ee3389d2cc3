"""The multi-rank bench path on ONE GPU: bench.py --gpus 2 self-launches two ranks under
torch.distributed.run (gloo, both on cuda:0), shards the global batch by sequence, times
the step max-over-ranks, gathers the outputs -- and the gathered step equals the 1-rank
step bit for bit (same per-unit workload, deterministic kernels)."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp_path, gpus):
    out = tmp_path / f"out{gpus}.npy"
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus),
                        "--batch", "4", "--ctx", "8192", "--steps", "8", "--warmup", "3",
                        "--no-dense", "--no-cpu", "--dump-out", str(out)],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    return line, np.load(out)


def test_two_ranks_equal_one_rank(cuda, tmp_path):
    l1, o1 = _run(tmp_path, 1)
    l2, o2 = _run(tmp_path, 2)
    assert l1["n_gpus"] == 1 and l2["n_gpus"] == 2
    assert l2["scaling"] == "strong" and l2["config"]["units_per_gpu"] == 16
    assert l2["allgather_us"] is not None and l2["us_per_step_with_allgather"] is not None
    assert l2["weak"] is not None and l2["weak"]["batch_per_gpu"] == 4
    assert l2["value"] > 0 and l2["e2e"]["value"] > 0
    assert o1.shape == o2.shape == (4 * 32, 128)
    np.testing.assert_array_equal(o1, o2)
