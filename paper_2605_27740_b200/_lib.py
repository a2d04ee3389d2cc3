"""ctypes binding of ``libpagetopk_b200.so`` (include/pagetopk_b200.h).

There is no CPU fallback: if the sm_100a library is missing or no CUDA device is
visible, every compute entry point raises.  Status codes map onto the reference's
exception types and messages (select.py:94-99, kvcache.py:164-166).
"""

from __future__ import annotations

import ctypes
import os

from . import _build

PT_F32 = 0
PT_BF16 = 1

PT_OK = 0
PT_ERR_INVALID = 1
PT_ERR_UNSUPPORTED = 2
PT_ERR_K = 3
PT_ERR_EMPTY = 4
PT_ERR_CAPACITY = 5
PT_ERR_CUDA_BASE = 1000

_lib: ctypes.CDLL | None = None

_c = ctypes
_vp = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64
_f = ctypes.c_float
_sz = ctypes.c_size_t

# name -> (restype, argtypes)
_PROTOS = {
    "pt_version": (_i, []),
    "pt_status_string": (ctypes.c_char_p, [_i]),
    "pt_fused_scores_host": (_i, [_vp, _vp, _vp, _vp, _i, _i64, _i, _f, _vp]),
    "pt_radix_select_desc_host": (_i, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "pt_stream_attention_host": (_i, [_vp, _vp, _vp, _i64, _i, _f, _i64, _vp, _vp, _vp]),
    "pt_mirror_bytes": (_sz, [_i, _i, _i]),
    "pt_page_stats": (_i, [_vp, _i, _vp, _vp, _vp, _i, _i, _i, _i, _vp, _i, _vp, _vp, _vp]),
    "pt_append": (_i, [_vp, _vp, _vp, _vp, _i, _vp, _vp, _i, _i, _i, _i, _vp, _i, _vp, _vp,
                       _vp, _vp, _vp, _vp]),
    "pt_write_rows": (_i, [_vp, _vp, _i, _vp, _vp, _vp, _vp, _i, _vp, _i, _i, _i, _i, _vp]),
    "pt_extend": (_i, [_vp, _vp, _i, _vp, _vp, _vp, _vp, _i, _vp, _i, _i, _i, _i, _vp, _i, _vp,
                       _vp, _vp]),
    "pt_score": (_i, [_vp, _i, _vp, _vp, _i, _vp, _vp, _i, _i, _i, _i, _i, _f, _vp, _vp, _vp, _vp,
                      _vp]),
    "pt_lam_norms": (_i, [_vp, _i, _vp, _i, _i, _i, _f, _vp, _vp, _vp]),
    "pt_lam_norms_chained": (_i, [_vp, _i, _vp, _i, _i, _i, _f, _vp, _vp, _vp]),
    "pt_score_bounded": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp,
                              _vp, _vp]),
    "pt_score_bounded_step": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _vp, _vp,
                                   _vp, _vp, _vp, _vp]),
    "pt_append_step": (_i, [_vp, _vp, _vp, _vp, _i, _vp, _vp, _i, _i, _i, _i, _vp, _i, _vp, _vp,
                            _vp, _vp, _vp, _vp, _vp]),
    "pt_score_prenorm": (_i, [_vp, _i, _vp, _vp, _i, _vp, _vp, _i, _i, _i, _i, _i, _vp, _vp, _vp,
                              _vp]),
    "pt_topk": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pt_score_select": (_i, [_vp, _i, _vp, _vp, _i, _vp, _vp, _vp, _i, _i, _i, _i, _i, _f, _i, _vp,
                             _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pt_attend_workspace_bytes": (_sz, [_i, _i, _i, _i]),
    "pt_attend": (_i, [_vp, _i, _vp, _vp, _i, _i, _vp, _i, _vp, _vp, _vp, _i, _i, _i, _i, _i, _vp,
                       _f, _vp, _vp, _vp, _sz, _vp, _i, _vp]),
    "pt_select_attend": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp,
                              _vp, _vp, _i, _vp,
                              _vp, _i, _i, _i, _i, _f, _vp, _vp, _vp, _sz, _vp, _vp]),
    "pt_debug_sa_prof": (_i, [_vp, _i]),
    "pt_debug_append_prof": (_i, [_vp, _i]),
    "pt_debug_sb_prof": (_i, [_vp, _i]),
    "pt_gated_attend_bwd": (_i, [_vp, _i, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _i, _i,
                                 _i, _f, _vp, _vp, _vp, _vp, _vp]),
    "pt_gate_bias": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp, _vp]),
    "pt_tile_means": (_i, [_vp, _i, _i, _i, _i, _vp, _i, _vp]),
    "pt_keys_max": (_i, [_vp, _vp, _i64, _vp]),
    "pt_pipe_create": (_i, [_vp, _vp, _vp, _i, _vp]),
    "pt_pipe_submit": (_i, [_vp, _i, _vp, _vp, _vp, _sz, _vp, _vp, _sz]),
    "pt_pipe_wait": (_i, [_vp, _i]),
    "pt_pipe_destroy": (_i, [_vp]),
}

EXPORTED = tuple(_PROTOS)


class CapacityError(RuntimeError):
    """Raised when the physical page pool is exhausted (kvcache.py:30-31)."""


def lib_path() -> str:
    return _build.LIB_PATH


def load() -> ctypes.CDLL:
    """Load the library (does not need a GPU; symbols only)."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} is missing: the sm_100a kernels are not built "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`); "
                "there is no CPU fallback"
            )
        L = ctypes.CDLL(path)
        for name, (res, args) in _PROTOS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def status_string(rc: int) -> str:
    return load().pt_status_string(rc).decode()


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI status onto the reference's exception types."""
    if rc == PT_OK:
        return
    if rc == PT_ERR_K:
        raise ValueError("k must be at least 1")
    if rc == PT_ERR_EMPTY:
        raise ValueError("no pages to select from")
    if rc == PT_ERR_CAPACITY:
        raise CapacityError("page pool exhausted")
    msg = status_string(rc)
    if rc == PT_ERR_UNSUPPORTED:
        raise NotImplementedError(f"{what}: {msg}")
    if rc >= PT_ERR_CUDA_BASE:
        raise RuntimeError(f"{what}: CUDA error: {msg}")
    raise ValueError(f"{what}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
