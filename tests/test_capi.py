"""The C-ABI boundary without a GPU: the library loads, exports exactly what
include/pagetopk_b200.h declares, and maps status codes onto the reference's errors."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pagetopk_b200.h")


def declared_symbols() -> set[str]:
    src = open(HEADER).read()
    return set(re.findall(r"PT_API\s+[\w\s\*]+?\b(pt_\w+)\s*\(", src))


def test_header_declares_the_contract():
    syms = declared_symbols()
    # the reference backend contract (backend.py:14-58) + the batched device API
    for name in ("pt_fused_scores_host", "pt_radix_select_desc_host", "pt_stream_attention_host",
                 "pt_page_stats", "pt_append", "pt_score", "pt_topk", "pt_attend"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_2605_27740_b200 import _lib

    L = _lib.load()
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert set(_lib.EXPORTED) == declared_symbols()
    # the reference package's own names are not exported by accident
    assert not hasattr(ctypes.CDLL(_lib.lib_path()), "fused_scores")


def test_library_is_sm100a_only():
    from paper_2605_27740_b200 import _lib

    data = open(_lib.lib_path(), "rb").read()
    assert b"sm_100a" in data


def test_version_and_status_strings():
    from paper_2605_27740_b200 import _lib

    assert _lib.load().pt_version() >= 100
    assert _lib.status_string(_lib.PT_OK) == "ok"
    assert "k must be at least 1" in _lib.status_string(_lib.PT_ERR_K)
    assert "exhausted" in _lib.status_string(_lib.PT_ERR_CAPACITY)
    with pytest.raises(ValueError, match="k must be at least 1"):
        _lib.check(_lib.PT_ERR_K)
    with pytest.raises(ValueError, match="no pages to select from"):
        _lib.check(_lib.PT_ERR_EMPTY)
    with pytest.raises(_lib.CapacityError):
        _lib.check(_lib.PT_ERR_CAPACITY)
    with pytest.raises(NotImplementedError):
        _lib.check(_lib.PT_ERR_UNSUPPORTED)


def test_invalid_arguments_rejected_without_touching_a_device():
    """Precondition checks run before any CUDA call (null pointers, k < 1)."""
    from paper_2605_27740_b200 import _lib

    L = _lib.load()
    assert L.pt_topk(None, None, None, 1, 16, 32, 4, None, None, None, None, None, None) == \
        _lib.PT_ERR_INVALID
    assert L.pt_score(None, 0, None, None, 0, None, None, 1, 4, 128, 16, 32, 0.5, None, None,
                      None, None, None) == _lib.PT_ERR_INVALID
    assert L.pt_select_attend(None, None, None, None, None, None, None, None, 1, 0, 1, 16, 32, 4, None,
                              None, None, None, None, None, 1, None, None, 1, 8, 4, 128, 0.1, None,
                              None, None, 0, None, None) == _lib.PT_ERR_INVALID
    assert L.pt_score_bounded(None, 1, None, None, None, None, None, 1, 0, 1, 4, 128, 16, 32, None,
                              None, None, None) == _lib.PT_ERR_INVALID
    assert L.pt_mirror_bytes(2, 64, 128) == 2 * 64 * 128 * 6 + 2 * 64 * 4
    assert L.pt_radix_select_desc_host(None, 10, 2, None, None, None) == _lib.PT_ERR_INVALID
    keys = (ctypes.c_uint16 * 4)()
    ids = (ctypes.c_int64 * 4)()
    t, k1 = ctypes.c_int(), ctypes.c_int()
    assert L.pt_radix_select_desc_host(keys, 4, 0, ids, ctypes.byref(t), ctypes.byref(k1)) == \
        _lib.PT_ERR_K
    assert L.pt_radix_select_desc_host(keys, 0, 1, ids, ctypes.byref(t), ctypes.byref(k1)) == \
        _lib.PT_ERR_EMPTY


def test_no_cpu_fallback_without_a_device(monkeypatch):
    """Compute entry points fail loudly when no CUDA device is present."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2605_27740_b200 as pt

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        pt.PagedKvCache(pt.CacheLayout(num_kv_heads=1, head_dim=16))
    with pytest.raises(RuntimeError):
        pt.compute_page_stats([[1.0, 0.0, 0.0, 0.0]])
