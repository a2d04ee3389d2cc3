"""The reference's OWN compiled kernels as the bench reference arm -- TEST INFRASTRUCTURE ONLY.

``oracle/_ref/_kernels_cy*.so`` is the reference backend (``pkg/src/pagetopk/_kernels_cy.pyx``)
compiled from the reference sources by ``make -C oracle ref`` (container only; the built .so
travels to the GPU box with the snapshot, the sources do not).  This module drives those
kernels exactly as the reference's ``decode_step`` does (``attention.py:110-147``), one
(sequence, kv-head) unit per task:

* ``QueryGroup.from_queries`` norms (``scoring.py:39-47``);
* ``fused_scores`` then RNE to bf16 bits (``scoring.py:108-124``, ``bf16.py:18-33``);
* ``encode_ordered`` (``select.py:51-57``), ``_take_all`` when P <= k (``select.py:75-84``),
  else ``radix_select_desc`` and ``mapping[ids]`` (``select.py:87-115``);
* per query head: ``gather_pages`` in selection order, partial tail page trimmed
  (``kvcache.py:266-280``), then ``stream_attention`` with block = page size and a zero
  block bias (``attention.py:57-75,94-107``).

With ``k_new`` / ``v_new`` a step first appends one K/V row per unit at position n (the
same slot every step, so the state a step sees is constant: n + 1 tokens) and refreshes the
tail page's stats with the reference's numpy ``compute_page_stats`` (``kvcache.py:59-71,
185-208``) -- the decode step of a serving loop, as the B200 arm's step does.

The compiled kernels hold the GIL (no ``nogil`` in the .pyx), so the units fan out over a
fork-started process pool, one worker per host core (SURVEY §8(d) CPU baseline (ii)).
Only ``bench.py --impl reference`` and tests use this module.
"""

from __future__ import annotations

import glob
import importlib.util
import math
import multiprocessing as mp
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_K = None  # the loaded reference kernel module (per process)
_W = None  # workload arrays shared with forked workers


def so_path() -> str | None:
    so = sorted(glob.glob(os.path.join(_HERE, "_ref", "_kernels_cy*.so")))
    return so[0] if so else None


def kernels():
    global _K
    if _K is None:
        p = so_path()
        if p is None:
            raise ImportError("oracle/_ref holds no compiled reference kernels (make -C oracle ref)")
        spec = importlib.util.spec_from_file_location("_kernels_cy", p)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _K = mod
    return _K


def _f32_to_bf16(a: np.ndarray) -> np.ndarray:
    bits = np.asarray(a, dtype=np.float32).view(np.uint32)
    out = ((bits + np.uint32(0x7FFF) + ((bits >> 16) & np.uint32(1))) >> 16).astype(np.uint16)
    nan = np.isnan(a)
    if np.any(nan):
        out = np.where(nan, ((bits >> 16) | np.uint32(0x40)).astype(np.uint16), out)
    return out


def _encode(bits: np.ndarray) -> np.ndarray:
    b = bits.astype(np.uint16)
    neg = (b & np.uint16(0x8000)) != 0
    return np.where(neg, ~b, b | np.uint16(0x8000)).astype(np.uint16)


def compute_page_stats(rows: np.ndarray):
    """kvcache.py:59-71 (numpy, float64 accumulation, f32 results)."""
    r = np.asarray(rows, dtype=np.float64)
    mean = r.mean(axis=0)
    var = np.mean((r - mean) ** 2, axis=0)
    return mean.astype(np.float32), float(np.float32(np.sqrt(var.sum())))


def append_unit(w, u: int) -> int:
    """kvcache.py:185-208 for unit u: the step's row lands at position n (the tail page has
    room: the workload keeps a spare page), the page's stats are recomputed; returns n + 1."""
    S = w["S"]
    n = int(w["seq"][u])
    lp, row = n // S, n % S
    pid = int(w["tab"][u, lp])
    w["kpool"][pid, row] = w["kn"][u]
    w["vpool"][pid, row] = w["vn"][u]
    mean, std = compute_page_stats(w["kpool"][pid, : row + 1])
    w["means"][u, lp] = mean
    w["stds"][u, lp] = std
    return n + 1


def appended(w):
    """(kpool, vpool, means, stds, seq) of the workload after one append per unit (for the
    port / cross-checks; the workload dict itself is not modified)."""
    v = dict(w)
    U, D = w["q"].shape[0], w["q"].shape[2]
    v["kpool"], v["vpool"] = w["kpool"].copy(), w["vpool"].copy()
    v["means"] = w["means"].reshape(U, -1, D).copy()
    v["stds"] = w["stds"].reshape(U, -1).copy()
    seq = np.array([append_unit(v, u) for u in range(U)], dtype=np.int32)
    return v["kpool"], v["vpool"], v["means"], v["stds"], seq


def decode_unit(u: int):
    """decode_step for one unit on the reference kernels; returns (phys ids, out [G,D], lse [G])."""
    K = kernels()
    w = _W
    q = np.ascontiguousarray(w["q"][u], dtype=np.float32)
    G, D = q.shape
    S = w["S"]
    n = append_unit(w, u) if w.get("kn") is not None else int(w["seq"][u])
    P = -(-n // S)
    norms = np.sqrt(np.sum(q.astype(np.float64) ** 2, axis=1)).astype(np.float32)
    means = np.ascontiguousarray(w["means"][u, :P])
    stds = np.ascontiguousarray(w["stds"][u, :P])
    scores = K.fused_scores(q, norms, means, stds, float(w["lam"]))
    keys = _encode(_f32_to_bf16(np.asarray(scores)))
    mapping = w["tab"][u, :P].astype(np.int64)
    k = w["k"]
    if P <= k:
        ids = np.arange(P, dtype=np.int64)
    else:
        ids, _, _, _ = K.radix_select_desc(np.ascontiguousarray(keys), k)
        ids = np.asarray(ids, dtype=np.int64)
    phys = mapping[ids]
    tail_rows = n - (P - 1) * S
    ks, vs = [], []
    for lid, pid in zip(ids.tolist(), phys.tolist()):
        rows = tail_rows if lid == P - 1 else S
        ks.append(w["kpool"][pid, :rows])
        vs.append(w["vpool"][pid, :rows])
    kk = np.ascontiguousarray(np.concatenate(ks, axis=0), dtype=np.float32)
    vv = np.ascontiguousarray(np.concatenate(vs, axis=0), dtype=np.float32)
    bias = np.zeros(-(-kk.shape[0] // S), dtype=np.float32)
    out = np.empty((G, D), np.float32)
    lse = np.empty(G, np.float64)
    for g in range(G):
        o, l = K.stream_attention(q[g], kk, vv, float(w["scale"]), S, bias)
        out[g] = np.asarray(o)
        lse[g] = l
    return phys, out, lse


class RefArm:
    """Fork-started worker pool over units running the reference kernels."""

    def __init__(self, q, kpool, vpool, page_table, seq_len, means, stds, k, lam, page_size,
                 nproc: int, k_new=None, v_new=None):
        global _W
        kernels()  # load (and fail loudly) before forking
        U, G, D = q.shape
        _W = dict(q=np.ascontiguousarray(q, dtype=np.float32), kpool=kpool, vpool=vpool,
                  tab=page_table, seq=seq_len, means=means.reshape(U, -1, D),
                  stds=stds.reshape(U, -1), k=int(k), lam=float(lam), S=int(page_size),
                  scale=1.0 / math.sqrt(D), kn=k_new, vn=v_new)
        self.U = U
        self.nproc = max(1, min(nproc, U))
        self.pool = mp.get_context("fork").Pool(self.nproc)

    def run(self):
        return self.pool.map(decode_unit, range(self.U), chunksize=1)

    def close(self):
        self.pool.terminate()
        self.pool.join()
