"""The bench reference arm (the reference's own compiled kernels driven as decode_step,
oracle/ref_arm.py) agrees with the oracle port on the same batched workload."""

import math

import numpy as np
import pytest

from oracle import oracle as O
from oracle import ref_arm

pytestmark = pytest.mark.skipif(ref_arm.so_path() is None,
                                reason="oracle/_ref not built (make -C oracle ref)")


@pytest.mark.parametrize("n_tokens,k", [(1000, 8), (200, 16)])  # radix regime; P <= k take-all
def test_ref_arm_matches_port(n_tokens, k):
    rng = np.random.default_rng(101)
    U, G, D, S = 6, 4, 32, 16
    P = -(-n_tokens // S)
    kpool = rng.standard_normal((U * P, S, D)).astype(np.float32)
    vpool = rng.standard_normal((U * P, S, D)).astype(np.float32)
    perm = rng.permutation(U * P).astype(np.int32).reshape(U, P)
    seq = np.array([n_tokens - 3 * u for u in range(U)], np.int32)
    tab = perm.copy()
    for u in range(U):
        tab[u, -(-int(seq[u]) // S):] = -1
    means, stds = O.build_stats(kpool, tab, seq, S)
    q = rng.standard_normal((U, G, D)).astype(np.float32)
    arm = ref_arm.RefArm(q, kpool, vpool, tab, seq, means, stds, k, 0.5, S, nproc=2)
    try:
        res = arm.run()
    finally:
        arm.close()
    port = O.decode_units(q, kpool, vpool, tab, seq, means, stds, k, 0.5, 1.0 / math.sqrt(D), S)
    for u, (phys, out, lse) in enumerate(res):
        assert set(phys.tolist()) == set(port["sel"][u][: port["n_sel"][u]].tolist())
        np.testing.assert_allclose(out, port["out"][u], rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(lse, port["lse"][u], rtol=1e-6)
