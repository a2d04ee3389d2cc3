"""ctypes front end of ``liboracle.so`` (pagetopk_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Each function mirrors one reference routine (paths relative to
``/root/reference/pkg/src/pagetopk/``) with identical arguments and results,
so parity tests read like the reference's own tests:

* ``compute_page_stats``  -> kvcache.py:59-71
* ``query_norms``         -> scoring.py:39-47 (QueryGroup.from_queries)
* ``fused_scores``        -> _kernels_cy.pyx:19-43
* ``f32_to_bf16``         -> bf16.py:18-33
* ``encode_ordered``      -> select.py:51-57
* ``radix_select_desc``   -> _kernels_cy.pyx:46-126
* ``stream_attention``    -> _kernels_cy.pyx:129-172
* ``decode_units``        -> attention.py:110-147 batched over (batch, kv-head) units
* ``dense_units``         -> attention.py:78-91 over every unit's full context
* ``build_stats``         -> kvcache.py:178-183/210-233 over a paged pool
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_c = ctypes


def build() -> str:
    """Compile liboracle.so with the committed Makefile (and the reference's own
    Cython kernels into oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    if os.path.isdir("/root/reference/pkg/src/pagetopk"):
        subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=False)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.or_f32_to_bf16.argtypes = [_f32p, _u16p, _c.c_int64]
        L.or_encode_ordered.argtypes = [_u16p, _u16p, _c.c_int64]
        L.or_encode_ordered.restype = _c.c_int
        L.or_np_sum.argtypes = [_f64p, _c.c_int64]
        L.or_np_sum.restype = _c.c_double
        L.or_page_stats.argtypes = [_f32p, _c.c_int, _c.c_int, _f32p, _f32p]
        L.or_query_norms.argtypes = [_f32p, _c.c_int, _c.c_int, _f32p]
        L.or_fused_scores.argtypes = [_f32p, _f32p, _f32p, _f32p, _c.c_int, _c.c_int64,
                                      _c.c_int, _c.c_float, _f32p]
        L.or_radix_select_desc.argtypes = [_u16p, _c.c_int64, _c.c_int64, _i64p,
                                           _c.POINTER(_c.c_int), _c.POINTER(_c.c_int)]
        L.or_radix_select_desc.restype = _c.c_int
        L.or_stream_attention.argtypes = [_f32p, _f32p, _f32p, _c.c_int64, _c.c_int,
                                          _c.c_float, _c.c_int64, _c.c_void_p, _f32p,
                                          _c.POINTER(_c.c_double)]
        L.or_build_stats.argtypes = [_f32p, _i32p, _i32p, _c.c_int, _c.c_int, _c.c_int,
                                     _c.c_int, _f32p, _f32p, _c.c_int]
        L.or_decode_units.argtypes = [_c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_int,
                                      _c.c_int64, _f32p, _f32p, _f32p, _i32p, _i32p, _f32p,
                                      _f32p, _c.c_float, _c.c_float, _c.c_int, _f32p, _f64p,
                                      _i32p, _i32p, _i32p, _i32p, _c.c_void_p, _c.c_void_p]
        L.or_decode_units.restype = _c.c_int
        L.or_dense_units.argtypes = [_c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_int, _f32p,
                                     _f32p, _f32p, _i32p, _i32p, _c.c_float, _c.c_int, _f32p,
                                     _f64p]
        L.or_max_threads.restype = _c.c_int
        _lib = L
    return _lib


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def max_threads() -> int:
    return int(lib().or_max_threads())


def f32_to_bf16(x) -> np.ndarray:
    x = _f32(x).reshape(-1)
    out = np.empty(x.shape[0], np.uint16)
    lib().or_f32_to_bf16(x, out, x.shape[0])
    return out


def encode_ordered(bits) -> np.ndarray:
    bits = np.ascontiguousarray(bits, dtype=np.uint16).reshape(-1)
    out = np.empty_like(bits)
    if lib().or_encode_ordered(bits, out, bits.shape[0]) != 0:
        raise ValueError("cannot order NaN scores")
    return out


def np_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().or_np_sum(a, a.shape[0]))


def compute_page_stats(keys) -> tuple[np.ndarray, float]:
    keys = _f32(keys)
    if keys.ndim != 2 or keys.shape[0] == 0:
        raise ValueError("keys must be a non-empty (count, head_dim) array")
    mean = np.empty(keys.shape[1], np.float32)
    std = np.empty(1, np.float32)
    lib().or_page_stats(keys, keys.shape[0], keys.shape[1], mean, std)
    return mean, float(std[0])


def query_norms(q) -> np.ndarray:
    q = _f32(q)
    if q.ndim == 1:
        q = q[None, :]
    out = np.empty(q.shape[0], np.float32)
    lib().or_query_norms(q, q.shape[0], q.shape[1], out)
    return out


def fused_scores(queries, norms, means, stds, lam: float) -> np.ndarray:
    queries, norms, means, stds = _f32(queries), _f32(norms), _f32(means), _f32(stds)
    out = np.empty(stds.shape[0], np.float32)
    lib().or_fused_scores(queries, norms, means, stds, queries.shape[0], stds.shape[0],
                          queries.shape[1], float(lam), out)
    return out


def radix_select_desc(keys, k: int) -> tuple[np.ndarray, int, int, int]:
    keys = np.ascontiguousarray(keys, dtype=np.uint16)
    ids = np.empty(k, np.int64)
    thr, kp1 = _c.c_int(), _c.c_int()
    lib().or_radix_select_desc(keys, keys.shape[0], k, ids, _c.byref(thr), _c.byref(kp1))
    return ids, int(thr.value), int(kp1.value), 3


def stream_attention(q, keys, values, scale: float, block: int, block_bias=None):
    q, keys, values = _f32(q), _f32(keys), _f32(values)
    out = np.empty(keys.shape[1], np.float32)
    lse = _c.c_double()
    bias = None if block_bias is None else _f32(block_bias)
    lib().or_stream_attention(q, keys, values, keys.shape[0], keys.shape[1], float(scale),
                              int(block), None if bias is None else bias.ctypes.data, out,
                              _c.byref(lse))
    return out, float(lse.value)


def build_stats(kpool, page_table, seq_len, page_size: int, nthreads: int = 0):
    kpool = _f32(kpool)
    page_table = np.ascontiguousarray(page_table, dtype=np.int32)
    seq_len = np.ascontiguousarray(seq_len, dtype=np.int32)
    U, Pmax = page_table.shape
    D = kpool.shape[-1]
    means = np.zeros((U, Pmax, D), np.float32)
    stds = np.zeros((U, Pmax), np.float32)
    lib().or_build_stats(kpool, page_table, seq_len, U, page_size, D, Pmax, means, stds,
                         nthreads)
    return means, stds


def decode_units(q, kpool, vpool, page_table, seq_len, means, stds, k: int, lam: float,
                 scale: float, page_size: int, nthreads: int = 0, want_scores: bool = False):
    """Batched reference decode step. q: [U, G, D]; returns a dict of numpy arrays."""
    q = _f32(q)
    U, G, D = q.shape
    page_table = np.ascontiguousarray(page_table, dtype=np.int32)
    seq_len = np.ascontiguousarray(seq_len, dtype=np.int32)
    Pmax = page_table.shape[1]
    means = _f32(means).reshape(U, Pmax, D)
    stds = _f32(stds).reshape(U, Pmax)
    out = np.zeros((U, G, D), np.float32)
    lse = np.zeros((U, G), np.float64)
    sel = np.full((U, k), -1, np.int32)
    n_sel = np.zeros(U, np.int32)
    kth = np.zeros(U, np.int32)
    kp1 = np.zeros(U, np.int32)
    scores = np.zeros((U, Pmax), np.float32) if want_scores else None
    keys = np.zeros((U, Pmax), np.uint16) if want_scores else None
    rc = lib().or_decode_units(U, G, D, page_size, Pmax, k, q, _f32(kpool), _f32(vpool),
                               page_table, seq_len, means, stds, float(lam), float(scale),
                               nthreads, out, lse, sel, n_sel, kth, kp1,
                               None if scores is None else scores.ctypes.data,
                               None if keys is None else keys.ctypes.data)
    if rc != 0:
        raise ValueError("cannot order NaN scores")
    res = dict(out=out, lse=lse, sel=sel, n_sel=n_sel, kth=kth, kplus1=kp1)
    if want_scores:
        res["scores"] = scores
        res["keys"] = keys
    return res


def dense_units(q, kpool, vpool, page_table, seq_len, scale: float, page_size: int,
                nthreads: int = 0):
    q = _f32(q)
    U, G, D = q.shape
    page_table = np.ascontiguousarray(page_table, dtype=np.int32)
    seq_len = np.ascontiguousarray(seq_len, dtype=np.int32)
    out = np.zeros((U, G, D), np.float32)
    lse = np.zeros((U, G), np.float64)
    lib().or_dense_units(U, G, D, page_size, page_table.shape[1], q, _f32(kpool), _f32(vpool),
                         page_table, seq_len, float(scale), nthreads, out, lse)
    return out, lse
