"""Differentiable page gating for training the criticality scorer (reference softmask.py),
with the attention forward and backward on the B200 kernels.

At train time every page takes part in attention, weighted by a sigmoid gate on its score
relative to the selection boundary (the midpoint of the k-th and (k+1)-th score); the gate
enters the softmax as an additive log-bias, so the gradient reaching each score is
d_scores_p = dL/dg_p * g_p (1 - g_p) / tau (softmask.py:1-22).  Hard mode keeps the top-k
pages (binary mask, ties to the lower page) and defines d_scores = 0.

Split of the work:
* the gate pipeline (boundary / sigmoid / standardisation, softmask.py:60-117) is P-sized
  float64 host arithmetic per unit, as the reference;
* the gated attention forward over every token is K4 in dense mode with a per-page bias
  log(gate) (soft) or K4 over the kept pages (hard) -- ``pt_attend``;
* its backward (softmask.py:178-217: dq, dK, dV, dgate per page, flash-style recomputation)
  is ``pt_gated_attend_bwd`` (csrc/gated_bwd.cu): one pass that reads K and V once and writes
  dK and dV once, for all G heads of a unit;
* the score path of the training step (float64 page statistics, group max, and the chain
  d_scores -> d_means / d_stds -> d_keys, softmask.py:438-464) runs on the device in float64.
The kernels compute in f32 where the reference computes in float64: parity is to a stated
tolerance (tests/test_gpu_parity.py::test_softmask_train_step_matches_reference).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .kvcache import CacheLayout, PagedKvCache

__all__ = [
    "GATE_FLOOR", "GateConfig", "boundary", "soft_gate", "gate_derivative", "hard_mask",
    "effective_tau", "gate_pipeline", "GatedOutput", "GateGradients", "GateTape",
    "gated_attention_forward", "gated_attention_backward", "gated_forward", "gated_backward",
    "FrozenConstants", "TrainStepResult", "decode_train_loss", "decode_train_step",
]

# smallest gate emitted (softmask.py:34-36): log(GATE_FLOOR) ~ -691 is a finite bias
GATE_FLOOR = 1e-300


@dataclass(frozen=True)
class GateConfig:
    """Page budget, temperature, mode, score standardisation (softmask.py:39-56)."""

    k: int = 64
    tau: float = 1.0
    mode: str = "soft"  # "soft" | "hard"
    standardize: bool = True

    def __post_init__(self) -> None:
        if self.mode not in ("soft", "hard"):
            raise ValueError(f"unknown gate mode {self.mode!r}")
        if self.tau <= 0:
            raise ValueError("tau must be positive")
        if self.k < 1:
            raise ValueError("k must be at least 1")


def _sigmoid(x):
    return 0.5 * (1.0 + np.tanh(0.5 * x))


def boundary(scores, k: int) -> float:
    """Midpoint of the k-th and (k+1)-th largest score (softmask.py:61-69)."""
    s = np.asarray(scores, dtype=np.float64)
    if k < 1:
        raise ValueError("k must be at least 1")
    if s.shape[0] <= k:
        raise ValueError("boundary undefined: need more than k scores")
    top = -np.sort(-s)
    return float(0.5 * (top[k - 1] + top[k]))


def soft_gate(scores, theta: float, tau: float) -> np.ndarray:
    return _sigmoid((np.asarray(scores, dtype=np.float64) - theta) / tau)


def gate_derivative(scores, theta: float, tau: float) -> np.ndarray:
    g = soft_gate(scores, theta, tau)
    return g * (1.0 - g) / tau


def hard_mask(scores, k: int) -> np.ndarray:
    """Binary top-k mask, ties to the lower page index (softmask.py:84-94)."""
    s = np.asarray(scores, dtype=np.float64)
    gates = np.zeros(s.shape[0], dtype=np.float64)
    if s.shape[0] <= k:
        gates[:] = 1.0
        return gates
    gates[np.argsort(-s, kind="stable")[:k]] = 1.0
    return gates


def effective_tau(scores, cfg: GateConfig) -> float:
    """tau times the score standard deviation when standardising (softmask.py:97-102)."""
    if not cfg.standardize:
        return cfg.tau
    sigma = float(np.std(np.asarray(scores, dtype=np.float64)))
    return cfg.tau * sigma if sigma > 0.0 else cfg.tau


def gate_pipeline(scores, cfg: GateConfig, theta: float | None = None,
                  tau_eff: float | None = None) -> tuple[np.ndarray, float | None, float]:
    """Scores -> (gates, theta, tau_eff) (softmask.py:105-131)."""
    s = np.asarray(scores, dtype=np.float64)
    if cfg.mode == "hard":
        return hard_mask(s, cfg.k), None, cfg.tau
    if s.shape[0] <= cfg.k:
        return np.ones(s.shape[0], dtype=np.float64), None, cfg.tau
    if tau_eff is None:
        tau_eff = effective_tau(s, cfg)
    if theta is None:
        theta = boundary(s, cfg.k)
    return np.maximum(soft_gate(s, theta, tau_eff), GATE_FLOOR), theta, tau_eff


# ---------------------------------------------------------------------------
# batched device forward / backward over a paged cache
# ---------------------------------------------------------------------------
def _gates_tensor(cache: PagedKvCache, gates) -> torch.Tensor:
    """Per-unit gate vectors -> f32 [U][Pmax] (pads 0)."""
    U, d = cache.num_units, cache.device
    g = torch.zeros(U, cache.Pmax, dtype=torch.float64, device=d)
    for u in range(U):
        gu = torch.as_tensor(np.asarray(gates[u], dtype=np.float64), device=d)
        g[u, : gu.shape[0]] = gu
    return g


def gated_forward(cache: PagedKvCache, queries: torch.Tensor, gates, scale: float | None = None,
                  mode: str = "soft") -> tuple[torch.Tensor, torch.Tensor]:
    """Attention of every query head over all pages of its unit with log-gate biases
    (softmask.py:108-176), batched: queries [U*G, D]; gates: per unit (P_u,) float64.
    Returns (out f32 [U*G, D], lse f32 [U*G])."""
    U, D, S = cache.num_units, cache.layout.head_dim, cache.layout.page_size
    q = queries.reshape(-1, D).contiguous()
    G = q.shape[0] // U
    if scale is None:
        scale = 1.0 / math.sqrt(D)
    g64 = gates if isinstance(gates, torch.Tensor) and gates.dim() == 2 else _gates_tensor(cache, gates)
    npages = np.array([cache.num_pages(u) for u in range(U)])  # host mirror: no device work
    if int(npages.min()) == 0:
        raise ValueError("attention over an empty context is undefined")
    if mode == "soft":
        # range check of the live gates and the f32 log-gate bias in one kernel, one flag read
        g64 = g64.to(cache.device, torch.float64).contiguous()
        bias = torch.empty(U, cache.Pmax, dtype=torch.float32, device=cache.device)
        flag = torch.empty(1, dtype=torch.int32, device=cache.device)
        _lib.call("pt_gate_bias", g64.data_ptr(), cache.seq_lens.data_ptr(), U, S, cache.Pmax,
                  bias.data_ptr(), flag.data_ptr(), dev.stream_handle())
        if int(flag.item()):
            raise ValueError("soft gates must lie in (0, 1]")
    elif mode == "hard":
        pages = torch.as_tensor(npages, device=cache.device)
        live = torch.arange(cache.Pmax, device=cache.device)[None, :] < pages[:, None]
        flags = torch.stack([(((g64 != 0) & (g64 != 1)) & live).any(),
                             (((g64 == 1) & live).sum(dim=1) == 0).any()]).cpu()
        if bool(flags[0]):
            raise ValueError("hard gates must be binary")
        if bool(flags[1]):
            raise ValueError("hard mask keeps no pages")
    else:
        raise ValueError(f"unknown gate mode {mode!r}")
    out = torch.empty(U * G, D, dtype=torch.float32, device=cache.device)
    lse = torch.empty(U * G, dtype=torch.float32, device=cache.device)
    ws = torch.empty(_lib.load().pt_attend_workspace_bytes(U, G, D, cache.Pmax), dtype=torch.uint8,
                     device=cache.device)
    tickets = torch.zeros(U, dtype=torch.int32, device=cache.device)
    qc = dev.dtype_code(q.dtype)
    if mode == "soft":
        _lib.call("pt_attend", q.data_ptr(), qc, cache.k_pool.data_ptr(), cache.v_pool.data_ptr(),
                  cache.kv_code, cache.layout.max_pages, cache.page_table.data_ptr(), cache.Pmax,
                  None, cache.page_table.data_ptr(), cache.seq_lens.data_ptr(), U, G, D, S,
                  cache.Pmax, bias.data_ptr(), float(scale), out.data_ptr(), lse.data_ptr(),
                  ws.data_ptr(), ws.numel(), tickets.data_ptr(), 0, dev.stream_handle())
    else:  # the kept pages only (a masked page carries exactly no weight)
        keep = g64 == 1
        n_sel = keep.sum(dim=1).to(torch.int32)
        k = int(n_sel.max().item())
        order = torch.argsort((~keep).to(torch.int8), dim=1, stable=True)[:, :k]
        sel = torch.gather(cache.page_table, 1, order).to(torch.int32).contiguous()
        _lib.call("pt_attend", q.data_ptr(), qc, cache.k_pool.data_ptr(), cache.v_pool.data_ptr(),
                  cache.kv_code, cache.layout.max_pages, sel.data_ptr(), k, n_sel.data_ptr(),
                  cache.page_table.data_ptr(), cache.seq_lens.data_ptr(), U, G, D, S, cache.Pmax,
                  None, float(scale), out.data_ptr(), lse.data_ptr(), ws.data_ptr(), ws.numel(),
                  tickets.data_ptr(), 0, dev.stream_handle())
    return out, lse


def gated_backward(cache: PagedKvCache, queries: torch.Tensor, gates, out: torch.Tensor,
                   lse: torch.Tensor, d_out: torch.Tensor, scale: float | None = None):
    """softmask.py:178-217 for every unit: returns (dq f32 [U*G, D], dk_pool f32, dv_pool f32
    ([pages][S][D]), dgates f32 [U][Pmax])."""
    U, D, S = cache.num_units, cache.layout.head_dim, cache.layout.page_size
    q = queries.reshape(-1, D).contiguous()
    G = q.shape[0] // U
    if scale is None:
        scale = 1.0 / math.sqrt(D)
    g64 = gates if isinstance(gates, torch.Tensor) and gates.dim() == 2 else _gates_tensor(cache, gates)
    g32 = g64.to(torch.float32).contiguous()
    d = cache.device
    dq = torch.zeros(U * G, D, dtype=torch.float32, device=d)
    # every row of every page of every unit is written by the kernel (zeros where no gradient)
    dk = torch.empty(cache.layout.max_pages, S, D, dtype=torch.float32, device=d)
    dv = torch.empty_like(dk)
    dg = torch.zeros(U, cache.Pmax, dtype=torch.float32, device=d)
    _lib.call("pt_gated_attend_bwd", q.data_ptr(), dev.dtype_code(q.dtype), cache.k_pool.data_ptr(),
              cache.v_pool.data_ptr(), cache.kv_code, cache.page_table.data_ptr(),
              cache.seq_lens.data_ptr(), g32.data_ptr(), out.contiguous().data_ptr(),
              lse.contiguous().data_ptr(), d_out.to(torch.float32).contiguous().data_ptr(), U, G, D,
              S, cache.Pmax, float(scale), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), dg.data_ptr(),
              dev.stream_handle())
    return dq, dk, dv, dg


# ---------------------------------------------------------------------------
# single-query API of the reference (softmask.py:108-217), on a one-unit device cache
# ---------------------------------------------------------------------------
@dataclass
class GatedOutput:
    out: np.ndarray
    lse: float


@dataclass
class GateGradients:
    d_q: np.ndarray
    d_keys: list
    d_values: list
    d_gates: np.ndarray
    d_scores: np.ndarray


@dataclass
class GateTape:
    cache: PagedKvCache
    q: torch.Tensor
    gates: np.ndarray
    scale: float
    tau_eff: float
    mode: str
    theta: float | None
    counts: list
    out: torch.Tensor = field(default=None)
    lse: torch.Tensor = field(default=None)


def _one_unit_cache(page_keys, page_values) -> tuple[PagedKvCache, list]:
    counts = [int(np.asarray(kp).shape[0]) for kp in page_keys]
    D = int(np.asarray(page_keys[0]).shape[1])
    S = max(counts)
    if any(c != S for c in counts[:-1]):
        raise ValueError("pages must be full except the last")
    layout = CacheLayout(num_kv_heads=1, head_dim=D, page_size=S, max_pages=len(counts))
    cache = PagedKvCache(layout, batch=1, dtype=torch.float32, max_pages_per_head=len(counts))
    k = np.concatenate([np.asarray(kp, np.float32) for kp in page_keys])[None]
    v = np.concatenate([np.asarray(vp, np.float32) for vp in page_values])[None]
    cache.extend_units(torch.from_numpy(k), torch.from_numpy(v))
    return cache, counts


def gated_attention_forward(q, page_keys, page_values, gates, scale: float | None = None,
                            mode: str = "soft", tau_eff: float = 1.0, theta: float | None = None,
                            scores=None) -> tuple[GatedOutput, GateTape]:
    """One query over per-page key/value arrays (softmask.py:108-176), on the device."""
    gates = np.asarray(gates, dtype=np.float64)
    if len(page_keys) != gates.shape[0] or len(page_values) != gates.shape[0]:
        raise ValueError("one gate per page required")
    if gates.shape[0] == 0:
        raise ValueError("attention over an empty context is undefined")
    cache, counts = _one_unit_cache(page_keys, page_values)
    qt = torch.as_tensor(np.asarray(q, np.float32)[None], device=cache.device)
    if scale is None:
        scale = 1.0 / math.sqrt(qt.shape[1])
    out, lse = gated_forward(cache, qt, [gates], scale, mode)
    tape = GateTape(cache=cache, q=qt, gates=gates, scale=float(scale), tau_eff=float(tau_eff),
                    mode=mode, theta=theta, counts=counts, out=out, lse=lse)
    return GatedOutput(out=out[0].double().cpu().numpy(), lse=float(lse[0])), tape


def gated_attention_backward(tape: GateTape, d_out) -> GateGradients:
    """Exact gradients of the gated forward (softmask.py:178-217), on the device."""
    cache = tape.cache
    do = torch.as_tensor(np.asarray(d_out, np.float32)[None], device=cache.device)
    dq, dk, dv, dg = gated_backward(cache, tape.q, [tape.gates], tape.out, tape.lse, do, tape.scale)
    P = len(tape.counts)
    pids = cache.page_table[0, :P].long()
    dk_p = dk[pids].double().cpu().numpy()
    dv_p = dv[pids].double().cpu().numpy()
    d_gates = dg[0, :P].double().cpu().numpy()
    if tape.mode == "hard":
        d_scores = np.zeros(P)
        d_gates = np.zeros(P)
    else:
        d_scores = d_gates * tape.gates * (1.0 - tape.gates) / tape.tau_eff
    return GateGradients(d_q=dq[0].double().cpu().numpy(),
                         d_keys=[dk_p[p, : tape.counts[p]] for p in range(P)],
                         d_values=[dv_p[p, : tape.counts[p]] for p in range(P)],
                         d_gates=d_gates, d_scores=d_scores)


# ---------------------------------------------------------------------------
# the gated decode training step (softmask.py:220-521), all units at once
# ---------------------------------------------------------------------------
@dataclass
class FrozenConstants:
    thetas: list
    tau_effs: list
    norms: list


@dataclass
class TrainStepResult:
    outputs: list
    loss: float
    d_queries: np.ndarray
    d_keys: list
    d_values: list
    d_scores: list
    d_means: list
    d_stds: list
    gates: list
    frozen: FrozenConstants


def _unit_rows(cache: PagedKvCache, pool: torch.Tensor, u: int) -> torch.Tensor:
    n, P = cache.seq_len(u), cache.num_pages(u)
    pids = cache.page_table[u, :P].long()
    return pool[pids].reshape(-1, pool.shape[-1])[:n]


def _train_forward(cache, queries, cfg, lam, target, scale, frozen):
    U, D, S = cache.num_units, cache.layout.head_dim, cache.layout.page_size
    q64 = torch.as_tensor(np.asarray(queries, np.float64), device=cache.device).reshape(-1, D)
    tgt = torch.as_tensor(np.asarray(target, np.float64), device=cache.device)
    if q64.shape[0] % U:
        raise ValueError(f"{q64.shape[0]} query heads not divisible by {U} KV heads")
    if tuple(tgt.shape) != (q64.shape[0], D):
        raise ValueError("target must be (num_query_heads, head_dim)")
    G = q64.shape[0] // U
    if scale is None:
        scale = 1.0 / math.sqrt(D)
    per_unit, gates_all = [], []
    for u in range(U):
        keys = _unit_rows(cache, cache.k_pool, u).double()
        n, P = keys.shape[0], cache.num_pages(u)
        counts = torch.full((P,), S, dtype=torch.float64, device=cache.device)
        counts[-1] = n - (P - 1) * S
        padded = torch.nn.functional.pad(keys, (0, 0, 0, P * S - n)).view(P, S, D)
        valid = (torch.arange(P * S, device=cache.device) < n).view(P, S, 1)
        means = padded.sum(dim=1) / counts[:, None]
        centred = torch.where(valid, padded - means[:, None, :], torch.zeros_like(padded))
        stds = torch.sqrt(((centred ** 2).sum(dim=1) / counts[:, None]).sum(dim=1))
        qg = q64[u * G:(u + 1) * G]
        norms = (torch.as_tensor(frozen.norms[u], device=cache.device)
                 if frozen is not None and frozen.norms[u] is not None
                 else torch.sqrt((qg ** 2).sum(dim=1)))
        score_mat = qg @ means.T + lam * norms[:, None] * stds[None, :]
        argmax_head = torch.argmax(score_mat, dim=0)  # first max: lowest head wins ties
        scores = score_mat.gather(0, argmax_head[None])[0]
        gates, theta, tau_eff = gate_pipeline(
            scores.cpu().numpy(), cfg,
            theta=frozen.thetas[u] if frozen is not None else None,
            tau_eff=frozen.tau_effs[u] if frozen is not None else None)
        gates_all.append(gates)
        per_unit.append(dict(keys=keys, padded=padded, valid=valid, means=means, stds=stds,
                             counts=counts, norms=norms, argmax_head=argmax_head,
                             scores=scores, gates=gates, theta=theta, tau_eff=tau_eff))
    qdev = q64.to(torch.float32)
    out, lse = gated_forward(cache, qdev, gates_all, scale, cfg.mode)
    diff = out.double() - tgt
    loss = float((diff * diff).sum())
    return per_unit, gates_all, qdev, out, lse, tgt, loss, G, float(scale)


def decode_train_loss(cache: PagedKvCache, queries, cfg: GateConfig, target, lam: float = 0.5,
                      scale: float | None = None, frozen: FrozenConstants | None = None) -> float:
    """Squared-error loss of one gated decode step (softmask.py:338-354)."""
    return _train_forward(cache, queries, cfg, lam, target, scale, frozen)[6]


def decode_train_step(cache: PagedKvCache, queries, cfg: GateConfig, target, lam: float = 0.5,
                      scale: float | None = None) -> TrainStepResult:
    """Gated decode step plus exact gradients (softmask.py:357-521)."""
    per_unit, gates_all, qdev, out, lse, tgt, loss, G, scale_v = _train_forward(
        cache, queries, cfg, lam, target, scale, None)
    U, D = cache.num_units, cache.layout.head_dim
    q64 = qdev.double()
    d_out = 2.0 * (out.double() - tgt)
    dq, dk_pool, dv_pool, dg = gated_backward(cache, qdev, gates_all, out, lse, d_out, scale_v)
    d_queries = dq.double()
    res = dict(d_keys=[], d_values=[], d_scores=[], d_means=[], d_stds=[])
    for u in range(U):
        st = per_unit[u]
        P = cache.num_pages(u)
        d_keys = _unit_rows(cache, dk_pool, u).double()
        d_values = _unit_rows(cache, dv_pool, u).double()
        gates = torch.as_tensor(st["gates"], device=cache.device)
        if cfg.mode == "hard" or P <= cfg.k:
            d_scores = torch.zeros(P, dtype=torch.float64, device=cache.device)
        else:
            d_scores = dg[u, :P].double() * gates * (1.0 - gates) / st["tau_eff"]
        d_means = torch.zeros(P, D, dtype=torch.float64, device=cache.device)
        d_stds = torch.zeros(P, dtype=torch.float64, device=cache.device)
        if bool((d_scores != 0).any()):
            win = st["argmax_head"]
            qw = q64[u * G + win]                                   # [P, D] winning heads
            d_queries.index_add_(0, u * G + win, d_scores[:, None] * st["means"])
            d_means = d_scores[:, None] * qw
            d_stds = d_scores * lam * st["norms"][win]
            cnt = st["counts"]
            chain = (d_means / cnt[:, None])[:, None, :].expand(P, cache.layout.page_size, D)
            ok = (st["stds"] > 0) & (d_stds != 0)
            coef = torch.where(ok, d_stds / (cnt * st["stds"]), torch.zeros_like(d_stds))
            cent = torch.where(st["valid"], st["padded"] - st["means"][:, None, :],
                               torch.zeros_like(st["padded"]))
            chain = chain + coef[:, None, None] * cent
            d_keys = d_keys + chain.reshape(-1, D)[: d_keys.shape[0]]
        res["d_keys"].append(d_keys.cpu().numpy())
        res["d_values"].append(d_values.cpu().numpy())
        res["d_scores"].append(d_scores.cpu().numpy())
        res["d_means"].append(d_means.cpu().numpy())
        res["d_stds"].append(d_stds.cpu().numpy())
    outs = [GatedOutput(out=out[i].double().cpu().numpy(), lse=float(lse[i])) for i in range(U * G)]
    frozen = FrozenConstants(thetas=[st["theta"] for st in per_unit],
                             tau_effs=[st["tau_eff"] for st in per_unit],
                             norms=[st["norms"].cpu().numpy() for st in per_unit])
    return TrainStepResult(outputs=outs, loss=loss, d_queries=d_queries.cpu().numpy(),
                           d_keys=res["d_keys"], d_values=res["d_values"],
                           d_scores=res["d_scores"], d_means=res["d_means"], d_stds=res["d_stds"],
                           gates=gates_all, frozen=frozen)
