"""Selection-quality harness at GPU scale (reference harness/recall.py:36-102, baselines.py:35-57,
harness/workload.py:60-98): page recall, attention-mass recall and output error of the unique
scorer, the mean-only scorer and the Quest min/max bound, for many single-query units at once.

Per unit u (one kv head with one query, G = 1, as the reference's recall evaluation):

* oracle (recall.py:36-57): the true attention mass of every page, from a dense float64
  softmax over the unit's keys; ranked descending, ties to the lower logical page;
* method scores: ``unique`` = K2 with lambda, ``mean_only`` = K2 with lambda = 0
  (baselines.py:60-62), ``quest`` = sum_d max(q_d * min_d, q_d * max_d) over each page's
  elementwise key bounds (baselines.py:35-57), all reduced to the same ordered bf16 keys;
* selection: K3 (pt_topk) -- the same top-k as the decode path;
* page_recall = |oracle top-k ∩ selected| / k, mass_recall = oracle mass of the selection,
  output_err = max |sparse - dense| with K4 over the selection and K4 dense mode
  (recall.py:71-102).

The scoring / selection / attention run on the package's kernels; the oracle and the Quest
bounds are evaluation-only arithmetic on torch (float64 for the oracle, float32 for Quest as
the reference).  ``gen_units_workload`` restates gen_workload's dilution construction on the
device (one key per planted page aligned with the unit's query).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from .engine import DecodeEngine
from .kvcache import CacheLayout, PagedKvCache

__all__ = ["RecallReport", "RECALL_METHODS", "UnitsWorkload", "gen_units_workload",
           "oracle_page_masses", "eval_recall_units"]

RECALL_METHODS = ("unique", "mean_only", "quest")


@dataclass
class RecallReport:
    method: str
    budget_tokens: int
    page_recall: float
    mass_recall: float
    output_err: float


@dataclass
class UnitsWorkload:
    cache: PagedKvCache
    queries: torch.Tensor          # [U, D] f32 on the device (one query per unit)
    planted: list[np.ndarray]      # per unit, logical indices of planted pages


def gen_units_workload(n_units: int, n_tokens: int, head_dim: int, page_size: int = 16,
                       planted_pages: int = 0, planted_gain: float = 6.0, key_scale: float = 1.0,
                       seed: int = 0, dtype=torch.float32, device=None) -> UnitsWorkload:
    """workload.py:60-98 on the device for n_units independent (kv head, query) units."""
    d = device or dev.require_cuda()
    g = torch.Generator(device=d)
    g.manual_seed(seed)
    n_pages = -(-n_tokens // page_size)
    layout = CacheLayout(num_kv_heads=n_units, head_dim=head_dim, page_size=page_size,
                         max_pages=n_units * n_pages)
    cache = PagedKvCache(layout, batch=1, dtype=dtype, max_pages_per_head=n_pages, device=d)
    q = torch.randn(n_units, head_dim, generator=g, device=d)
    planted: list[np.ndarray] = []
    chunk = max(1, min(n_tokens, (1 << 26) // (n_units * head_dim)))
    direction = q.double() / torch.linalg.vector_norm(q.double(), dim=1, keepdim=True)
    full_pages = n_tokens // page_size
    plant_rows = None
    if planted_pages > 0:
        rng = np.random.default_rng(seed)
        rows = []
        for u in range(n_units):
            pages = np.sort(rng.choice(full_pages, size=planted_pages, replace=False))
            slots = pages * page_size + rng.integers(page_size, size=planted_pages)
            planted.append(pages.astype(np.int64))
            rows.append(slots)
        plant_rows = torch.from_numpy(np.stack(rows)).to(d)  # [U, planted]
    else:
        planted = [np.empty(0, np.int64) for _ in range(n_units)]
    done = 0
    while done < n_tokens:
        n = min(chunk, n_tokens - done)
        kk = torch.randn(n_units, n, head_dim, generator=g, device=d) * key_scale
        vv = torch.randn(n_units, n, head_dim, generator=g, device=d) * key_scale
        if plant_rows is not None:
            for u in range(n_units):
                sel = (plant_rows[u] >= done) & (plant_rows[u] < done + n)
                for r in plant_rows[u][sel].tolist():
                    res = torch.randn(head_dim, generator=g, device=d, dtype=torch.float64)
                    res -= (res @ direction[u]) * direction[u]
                    kk[u, r - done] = (key_scale * (planted_gain * direction[u] + res)).float()
        cache.extend_units(kk.to(dtype), vv.to(dtype))
        done += n
    return UnitsWorkload(cache=cache, queries=q, planted=planted)


def _unit_keys(cache: PagedKvCache, u: int) -> torch.Tensor:
    """The unit's keys [n, D] (gathered from its pages), float64."""
    n = cache.seq_len(u)
    P = cache.num_pages(u)
    pids = cache.page_table[u, :P].long()
    return cache.k_pool[pids].reshape(-1, cache.layout.head_dim)[:n].double()


def oracle_page_masses(cache: PagedKvCache, queries: torch.Tensor) -> list[torch.Tensor]:
    """Per unit, the dense float64 softmax mass of every logical page (recall.py:36-57)."""
    S = cache.layout.page_size
    out = []
    for u in range(cache.num_units):
        keys = _unit_keys(cache, u)
        q64 = queries[u].double()
        logits = keys @ q64 / math.sqrt(q64.shape[0])
        w = torch.exp(logits - logits.max())
        w = w / w.sum()
        P = cache.num_pages(u)
        pad = P * S - w.shape[0]
        out.append(torch.nn.functional.pad(w, (0, pad)).view(P, S).sum(dim=1))
    return out


def _ordered_keys(scores: torch.Tensor) -> torch.Tensor:
    """f32 scores -> RNE bf16 -> order-preserving u16 keys (bf16.py:18-33, select.py:51-64),
    held as int16 bit patterns."""
    b = scores.to(torch.bfloat16).view(torch.int16).int() & 0xFFFF
    neg = (b & 0x8000) != 0
    key = torch.where(neg, (~b) & 0xFFFF, b | 0x8000)
    return key.to(torch.int32).to(torch.int16)


def _quest_scores(cache: PagedKvCache, queries: torch.Tensor) -> torch.Tensor:
    """baselines.py:35-57 over every page of every unit: [U, Pmax] (pads = -inf)."""
    U, S, D = cache.num_units, cache.layout.page_size, cache.layout.head_dim
    out = torch.full((U, cache.Pmax), -math.inf, device=queries.device)
    for u in range(U):
        n, P = cache.seq_len(u), cache.num_pages(u)
        pids = cache.page_table[u, :P].long()
        rows = cache.k_pool[pids].float()                       # [P, S, D]
        valid = (torch.arange(P * S, device=rows.device) < n).view(P, S, 1)
        mins = torch.where(valid, rows, torch.full_like(rows, math.inf)).amin(dim=1)
        maxs = torch.where(valid, rows, torch.full_like(rows, -math.inf)).amax(dim=1)
        q32 = queries[u].float()
        out[u, :P] = torch.maximum(q32 * mins, q32 * maxs).sum(dim=1)
    return out


def eval_recall_units(cache: PagedKvCache, queries: torch.Tensor, k: int,
                      methods=RECALL_METHODS, lam: float = 0.5,
                      masses: list[torch.Tensor] | None = None) -> dict[str, list[RecallReport]]:
    """eval_recall (recall.py:71-102) for every unit of ``cache`` (one query per unit)."""
    U = cache.num_units
    if queries.shape[0] != U:
        raise ValueError("recall evaluation expects one query per unit (G = 1)")
    for u in range(U):
        if k < 1 or k > cache.num_pages(u):
            raise ValueError("k must lie in [1, n_pages]")
    if masses is None:
        masses = oracle_page_masses(cache, queries)
    q = queries.to(cache.dtype).contiguous()
    eng = DecodeEngine(cache, 1, k, lam=lam, keep_logical=True)
    dense_out, _ = eng.dense(q)
    dense_out = dense_out.clone()
    reports: dict[str, list[RecallReport]] = {}
    for method in methods:
        if method == "unique":
            eng.lam = float(lam)
            eng.score(q)
        elif method == "mean_only":
            eng.lam = 0.0
            eng.score(q)
        elif method == "quest":
            eng.keys.copy_(_ordered_keys(_quest_scores(cache, queries)))
        else:
            raise ValueError(f"unknown method {method!r}")
        eng.select()
        eng.attend(q)
        torch.cuda.synchronize()
        sel = eng.sel_logical.cpu().numpy()
        err = (eng.out.float() - dense_out.float()).abs().amax(dim=1).cpu().numpy()
        rows = []
        for u in range(U):
            m = masses[u]
            ranked = torch.sort(m, descending=True, stable=True).indices[:k].cpu().numpy()
            picked = sel[u, :k]
            rows.append(RecallReport(
                method=method, budget_tokens=k * cache.layout.page_size,
                page_recall=len(set(ranked.tolist()) & set(picked.tolist())) / k,
                mass_recall=float(m[torch.from_numpy(picked.astype(np.int64)).to(m.device)].sum()),
                output_err=float(err[u])))
        reports[method] = rows
    eng.lam = float(lam)
    return reports
