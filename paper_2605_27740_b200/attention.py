"""Decode-side attention: dense, sparse over selected pages, and the scored decode
step (reference attention.py:1-147), on the B200 kernels.

* ``dense_attention`` / the backend ``stream_attention`` contract -> K4 over
  contiguous rows served as pages;
* ``sparse_attention`` -> K4 over one head's selected pages straight from the
  paged pool (no host gather);
* ``decode_step`` -> the batched engine (K2 score -> K3 select -> K4 attend for
  every kv head at once), returned in the reference's per-head types.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from . import _lib
from . import backend
from .engine import DecodeEngine
from .kvcache import PagedKvCache
from .select import STAGED_MAX_PAGES, TopKSelection, _regime, key_to_score

__all__ = [
    "AttentionOutput",
    "DecodeConfig",
    "decode_step",
    "decode_step_batched",
    "dense_attention",
    "sparse_attention",
]


@dataclass
class AttentionOutput:
    """Attention result for one query: output vector and log-sum-exp (attention.py:23-28)."""

    out: np.ndarray  # (head_dim,) f32
    lse: float


@dataclass(frozen=True)
class DecodeConfig:
    """Page budget k, spread weight lam, logit scale (None -> 1/sqrt(D)) (attention.py:31-54)."""

    k: int = 64
    lam: float = 0.5
    scale: float | None = None

    def __post_init__(self) -> None:
        if self.k < 1:
            raise ValueError("k must be at least 1")

    @classmethod
    def from_budget(cls, budget_tokens: int, page_size: int, **kw) -> "DecodeConfig":
        """Token budget -> page budget, rounded up."""
        if budget_tokens < 1:
            raise ValueError("budget_tokens must be positive")
        return cls(k=(budget_tokens + page_size - 1) // page_size, **kw)

    def resolve_scale(self, head_dim: int) -> float:
        return 1.0 / math.sqrt(head_dim) if self.scale is None else self.scale


def dense_attention(q, keys, values, scale: float | None = None,
                    block_size: int = 8) -> AttentionOutput:
    """Softmax attention of one query over a full context (attention.py:78-91)."""
    keys = np.asarray(keys)
    if keys.ndim != 2 or keys.shape[0] == 0:
        raise ValueError("attention over an empty context is undefined")
    if scale is None:
        scale = 1.0 / math.sqrt(keys.shape[1])
    n_blocks = -(-keys.shape[0] // block_size)
    out, lse = backend.stream_attention(q, keys, values, float(scale), block_size,
                                        np.zeros(n_blocks, dtype=np.float32))
    return AttentionOutput(out=out, lse=lse)


def sparse_attention(q, cache: PagedKvCache, head: int, selection: TopKSelection,
                     scale: float | None = None) -> AttentionOutput:
    """Attention restricted to one head's selected pages (attention.py:94-107)."""
    if len(selection) == 0:
        raise ValueError("attention over an empty selection is undefined")
    cache.table.to_logical(head, selection.physical_ids)  # ownership check (LookupError)
    if scale is None:
        scale = 1.0 / math.sqrt(cache.layout.head_dim)
    d = cache.device
    D, S = cache.layout.head_dim, cache.layout.page_size
    qt = dev.to_device(np.asarray(q, np.float32).reshape(1, D), torch.float32, d)
    sel = torch.from_numpy(np.asarray(selection.physical_ids, dtype=np.int32)).to(d)
    n_sel = torch.tensor([sel.numel()], dtype=torch.int32, device=d)
    out = torch.empty(1, D, dtype=torch.float32, device=d)
    lse = torch.empty(1, dtype=torch.float32, device=d)
    ws = torch.empty(_lib.load().pt_attend_workspace_bytes(1, 1, D, sel.numel()),
                     dtype=torch.uint8, device=d)
    tickets = torch.zeros(1, dtype=torch.int32, device=d)
    # address unit `head` by offsetting the per-unit arrays
    pt_row = cache.page_table[head]
    seq = cache.seq_lens[head : head + 1]
    _lib.call("pt_attend", qt.data_ptr(), _lib.PT_F32, cache.k_pool.data_ptr(),
              cache.v_pool.data_ptr(), cache.kv_code, cache.layout.max_pages, sel.data_ptr(),
              sel.numel(),
              n_sel.data_ptr(), pt_row.data_ptr(), seq.data_ptr(), 1, 1, D, S, cache.Pmax, None,
              float(scale), out.data_ptr(), lse.data_ptr(), ws.data_ptr(), ws.numel(),
              tickets.data_ptr(), 0, dev.stream_handle())
    return AttentionOutput(out=out[0].cpu().numpy(), lse=float(lse.item()))


def _engine_for(cache: PagedKvCache, G: int, cfg: DecodeConfig) -> DecodeEngine:
    key = (G, cfg.k, float(cfg.lam), cfg.resolve_scale(cache.layout.head_dim))
    eng = getattr(cache, "_engines", {}).get(key)
    if eng is None:
        eng = DecodeEngine(cache, G, cfg.k, lam=cfg.lam,
                           scale=cfg.resolve_scale(cache.layout.head_dim))
        if not hasattr(cache, "_engines"):
            cache._engines = {}
        cache._engines[key] = eng
    return eng


def decode_step_batched(cache: PagedKvCache, queries: torch.Tensor,
                        cfg: DecodeConfig = DecodeConfig()):
    """Device-resident decode step for all units: returns (out [U*G, D], lse [U*G]) tensors
    plus the engine holding the selections (sel / n_sel / kth / kplus1)."""
    n_q = queries.reshape(-1, cache.layout.head_dim).shape[0]
    if n_q % cache.num_units:
        raise ValueError(f"{n_q} query heads not divisible by {cache.num_units} KV heads")
    eng = _engine_for(cache, n_q // cache.num_units, cfg)
    out, lse = eng.step(queries)
    return out, lse, eng


def decode_step(cache: PagedKvCache, queries, cfg: DecodeConfig = DecodeConfig()):
    """One sparse decode step for all query heads (attention.py:110-147).

    Returns one AttentionOutput per query head (row order of ``queries``) and one
    TopKSelection per KV head (unit).
    """
    q = np.asarray(queries, dtype=np.float32) if not isinstance(queries, torch.Tensor) else queries
    if q.ndim != 2:
        raise ValueError("queries must be (num_query_heads, head_dim)")
    n_heads, n_kv = q.shape[0], cache.num_units
    if n_heads % n_kv != 0:
        raise ValueError(f"{n_heads} query heads not divisible by {n_kv} KV heads")
    for h in range(n_kv):
        if cache.num_pages(h) == 0:
            raise ValueError("no pages to select from")
    qt = dev.to_device(q, torch.float32, cache.device)
    out, lse, eng = decode_step_batched(cache, qt, cfg)
    out_h = out.cpu().numpy()
    lse_h = lse.cpu().numpy().astype(np.float64)
    sel = eng.sel.cpu().numpy()
    n_sel = eng.n_sel.cpu().numpy()
    kth = eng.kth.cpu().numpy()
    kp1 = eng.kplus1.cpu().numpy()
    outputs = [AttentionOutput(out=out_h[i].copy(), lse=float(lse_h[i])) for i in range(n_heads)]
    selections = []
    for u in range(n_kv):
        P = cache.num_pages(u)
        take_all = kp1[u] < 0
        beyond = P > STAGED_MAX_PAGES
        selections.append(TopKSelection(
            physical_ids=sel[u, : n_sel[u]].astype(np.int64),
            kth_score=key_to_score(int(kth[u])),
            kplus1_score=None if take_all else key_to_score(int(kp1[u])),
            regime="fallback" if (beyond and not take_all) else _regime(P),
            passes=1 if take_all else (None if beyond else 3),
        ))
    return outputs, selections
