"""Host-side gate pipeline of the soft-mask training path (softmask.py:60-131): boundary,
sigmoid gates, hard mask, standardised temperature -- against the reference where it is
importable (build container), and against closed forms everywhere."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2605_27740_b200 import softmask as sm


def test_gate_pipeline_closed_forms():
    s = np.array([3.0, 1.0, 4.0, 1.0, 5.0, 9.0, 2.0])
    assert sm.boundary(s, 2) == pytest.approx(0.5 * (5.0 + 4.0))
    g, theta, tau = sm.gate_pipeline(s, sm.GateConfig(k=2, tau=1.0, standardize=False))
    assert theta == pytest.approx(4.5) and tau == 1.0
    np.testing.assert_allclose(g, 1.0 / (1.0 + np.exp(-(s - 4.5))), rtol=1e-12)
    h, _, _ = sm.gate_pipeline(s, sm.GateConfig(k=3, mode="hard"))
    np.testing.assert_array_equal(h, [0, 0, 1, 0, 1, 1, 0])
    # ties go to the lower index
    np.testing.assert_array_equal(sm.hard_mask(np.array([1.0, 2.0, 2.0, 2.0]), 2), [0, 1, 1, 0])
    ones, th, _ = sm.gate_pipeline(s[:2], sm.GateConfig(k=4))
    assert th is None and np.all(ones == 1.0)
    tiny, _, _ = sm.gate_pipeline(np.array([0.0, 0.0, 1e6]), sm.GateConfig(k=1, tau=1e-3,
                                                                           standardize=False))
    assert tiny.min() >= sm.GATE_FLOOR
    with pytest.raises(ValueError):
        sm.GateConfig(mode="medium")
    with pytest.raises(ValueError):
        sm.boundary(s, 7)


def test_gate_pipeline_matches_reference():
    from oracle import reference

    if not reference.available():
        pytest.skip("/root/reference absent")
    reference.load("python")
    from pagetopk import softmask as ref

    rng = np.random.default_rng(5)
    for _ in range(50):
        n = int(rng.integers(2, 300))
        k = int(rng.integers(1, n + 3))
        s = rng.standard_normal(n) * 10.0 ** rng.integers(-2, 3)
        for mode in ("soft", "hard"):
            for std in (True, False):
                cfg_ours = sm.GateConfig(k=k, tau=0.7, mode=mode, standardize=std)
                cfg_ref = ref.GateConfig(k=k, tau=0.7, mode=mode, standardize=std)
                g0, t0, e0 = sm.gate_pipeline(s, cfg_ours)
                g1, t1, e1 = ref.gate_pipeline(s, cfg_ref)
                np.testing.assert_array_equal(g0, g1)
                assert t0 == t1 and e0 == e1
