"""The reference's kernel-backend module contract, served by the B200 library.

The reference selects its kernels through ``pagetopk.backend`` (backend.py:14-58):
a module exposing ``NAME`` plus ``fused_scores``, ``radix_select_desc`` and
``stream_attention`` with the signatures of ``_kernels_cy.pyx:19-172``.  This module
is that contract with host (numpy) buffers in and out, each call going through the
C ABI (include/pagetopk_b200.h section A) to the sm_100a kernels -- register it in
the reference as a third backend or call it directly.

There is exactly one implementation here; no dispatch, no CPU fallback.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

NAME = "b200"

__all__ = ["NAME", "fused_scores", "radix_select_desc", "stream_attention"]


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def fused_scores(queries, norms, means, stds, lam: float) -> np.ndarray:
    """Group-max criticality scores, one f32 score per page (_kernels_cy.pyx:19-43).

    Bit-identical to the reference's compiled backend.
    """
    q, nr, m, s = _f32(queries), _f32(norms), _f32(means), _f32(stds)
    if q.ndim != 2 or m.ndim != 2 or m.shape[1] != q.shape[1] or s.shape[0] != m.shape[0]:
        raise ValueError("fused_scores: queries (G, D), norms (G,), means (P, D), stds (P,)")
    out = np.empty(s.shape[0], dtype=np.float32)
    _lib.call("pt_fused_scores_host", q.ctypes.data, nr.ctypes.data, m.ctypes.data,
              s.ctypes.data, q.shape[0], s.shape[0], q.shape[1], float(lam), out.ctypes.data)
    return out


def radix_select_desc(keys, k: int) -> tuple[np.ndarray, int, int, int]:
    """k largest of P uint16 keys, lowest index winning ties (_kernels_cy.pyx:46-126).

    Returns (indices int64 -- ascending, i.e. unordered as in the reference contract,
    kth key, next key below the cut, 3).  Caller guarantees 1 <= k < len(keys).
    """
    kk = np.ascontiguousarray(keys, dtype=np.uint16)
    ids = np.empty(int(k), dtype=np.int64)
    thr, kp1 = ctypes.c_int(), ctypes.c_int()
    _lib.call("pt_radix_select_desc_host", kk.ctypes.data, kk.shape[0], int(k), ids.ctypes.data,
              ctypes.addressof(thr), ctypes.addressof(kp1))
    return ids, int(thr.value), int(kp1.value), 3


def stream_attention(q, keys, values, scale: float, block: int, block_bias) -> tuple[np.ndarray, float]:
    """Streaming softmax attention with a per-block additive bias (_kernels_cy.pyx:129-172)."""
    qq, kk, vv = _f32(q), _f32(keys), _f32(values)
    n, d = kk.shape
    bias = None if block_bias is None else _f32(block_bias)
    out = np.empty(d, dtype=np.float32)
    lse = ctypes.c_double()
    _lib.call("pt_stream_attention_host", qq.ctypes.data, kk.ctypes.data, vv.ctypes.data, n, d,
              float(scale), int(block), None if bias is None else bias.ctypes.data,
              out.ctypes.data, ctypes.addressof(lse))
    return out, float(lse.value)
