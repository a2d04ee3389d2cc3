"""Device plumbing shared by the host mirror: dtype codes, pointers, streams.

PyTorch provides device memory and streams only; all arithmetic on the hot path
runs in the sm_100a kernels of ``libpagetopk_b200.so``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2605_27740_b200 needs a CUDA (sm_100a) device; there is no CPU fallback"
        )
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return _lib.PT_F32
    if dt == torch.bfloat16:
        return _lib.PT_BF16
    raise NotImplementedError(f"element type {dt} (supported: float32, bfloat16)")


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def to_device(a, dtype: torch.dtype, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=device, dtype=dtype).contiguous()


def stats_vec(stats_dtype: torch.dtype) -> int:
    """Elements per 16-byte vector of the page-interleaved means layout."""
    return 4 if stats_dtype == torch.float32 else 8


def untile_means(tiled: torch.Tensor, U: int, Pmax: int, D: int, stats_dtype) -> torch.Tensor:
    """Tiled means [U][Pmax/32][D/V][32][V] -> row-major [U][Pmax][D] (readback only)."""
    V = stats_vec(stats_dtype)
    t = tiled.view(U, Pmax // 32, D // V, 32, V).permute(0, 1, 3, 2, 4)
    return t.reshape(U, Pmax, D)
