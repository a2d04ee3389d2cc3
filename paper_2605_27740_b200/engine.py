"""Batched decode engine: the B200 hot path of attention.py:110-147 over all units.

One decode step for every (sequence, kv-head) unit of a :class:`PagedKvCache`:

    append K/V row    (K1b: pt_append)        kvcache.py:185-208
    lambda * ||q||    (pt_lam_norms_chained)  scoring.py:39-47        (runs beside the append)
    score             (K2b: pt_score_bounded) scoring.py:108-124 -> bf16 -> ordered keys, as
                                              [lower, upper] key intervals from the bf16 mirror
                                              of the f32 means (+ per-32-page tile maxima);
                      (K2: pt_score_prenorm)  exact keys from the f32 means (no mirror, f32 q)
    select + attend   (K3+K4: pt_select_attend) select.py:87-115 + page-table translation,
                                              then attention.py:94-107 for the G heads

All launches go on device-resident buffers with no host synchronisation (programmatic
dependent launch between consecutive kernels), so a step can be captured once and replayed as
a CUDA graph (:meth:`DecodeEngine.capture`).  ``select`` / ``attend`` are the same stages as
separate launches (pt_topk / pt_attend); ``score_select`` is an alternative K2+K3 launch.
``dense`` runs K4 over every page (attention.py:78-91), the speed-up denominator.
"""

from __future__ import annotations

import math
import os

import torch

from . import _device as dev
from . import _lib
from .kvcache import PagedKvCache

__all__ = ["DecodeEngine"]


class DecodeEngine:
    def __init__(
        self,
        cache: PagedKvCache,
        group_size: int,
        k: int,
        lam: float = 0.5,
        scale: float | None = None,
        keep_scores: bool = False,
        keep_logical: bool = False,
    ) -> None:
        if k < 1:
            raise ValueError("k must be at least 1")
        if group_size < 1:
            raise ValueError("group_size must be positive")
        self.cache = cache
        self.G = group_size
        self.k = int(k)
        self.lam = float(lam)
        D = cache.layout.head_dim
        self.scale = 1.0 / math.sqrt(D) if scale is None else float(scale)
        U, Pmax, d = cache.num_units, cache.Pmax, cache.device
        self.U, self.D = U, D
        self.keys = torch.zeros(U, Pmax, dtype=torch.int16, device=d)  # u16 bit patterns
        self.tile_max = torch.zeros(U, Pmax // 32, dtype=torch.int16, device=d)  # per 32 pages
        self.scores = torch.zeros(U, Pmax, dtype=torch.float32, device=d) if keep_scores else None
        self.sel = torch.zeros(U, self.k, dtype=torch.int32, device=d)
        self.sel_logical = (torch.zeros(U, self.k, dtype=torch.int32, device=d)
                            if keep_logical else None)
        self.n_sel = torch.zeros(U, dtype=torch.int32, device=d)
        self.kth = torch.zeros(U, dtype=torch.int32, device=d)
        self.kplus1 = torch.zeros(U, dtype=torch.int32, device=d)
        self.out = torch.zeros(U * self.G, D, dtype=torch.float32, device=d)
        self.lse = torch.zeros(U * self.G, dtype=torch.float32, device=d)
        self.dense_out = torch.zeros_like(self.out)
        self.dense_lse = torch.zeros_like(self.lse)
        wsb = _lib.load().pt_attend_workspace_bytes(U, self.G, D, max(self.k, Pmax))
        self.ws = torch.zeros(wsb, dtype=torch.uint8, device=d)
        self.tickets = torch.zeros(U, dtype=torch.int32, device=d)
        self.score_counters = torch.zeros(U, dtype=torch.int32, device=d)
        self.lamnorm = torch.zeros(U * 8, dtype=torch.float32, device=d)
        # bounded scoring (cache.mirror): upper keys of the score intervals and ||q|| bounds;
        # the selection resolves the straddling pages exactly
        self.bounded = (cache.mirror is not None and not keep_scores
                        and os.environ.get("PT_NO_BOUNDED", "") != "1" and self._bounded_pays(cache))
        self.keys_hi = torch.zeros(U, Pmax, dtype=torch.int16, device=d) if self.bounded else None
        self.qnorm = torch.zeros(U * 8, dtype=torch.float32, device=d) if self.bounded else None
        self._step_bounded = False  # the keys of the last scoring are intervals
        # K2 streaming kernel + K3 (two launches) is the default; the one-launch fused
        # score+select CTA kernel (pt_score_select) is kept as an alternative
        self.fused_select = False
        # K3 + K4 fused (pt_select_attend) is the default after K2
        self.fused_attend = True
        self.dense_tickets = torch.zeros(U, dtype=torch.int32, device=d)
        self.graph: torch.cuda.CUDAGraph | None = None
        self._side = torch.cuda.Stream(device=d)
        # append -> norms -> score as one PDL chain (PT_NO_PDL=1: the fork/join instead)
        self.chain_norms = os.environ.get("PT_NO_PDL", "") != "1" and os.environ.get("PT_NORMS_FORK", "") != "1"
        # half-batch pipelining of score -> select+attend (bounded mode, >= 128 units; split at
        # a sequence boundary when possible): opt-in (PT_SPLIT=1) -- measured slower at cfg3
        # (203 vs 168.5 us/step: the second half's select+attend runs alone at half occupancy,
        # and the first half's CTAs delay the second scorer's static tile ranges)
        h = U // 2
        H = cache.layout.num_kv_heads
        if U % H == 0 and (U // H) % 2 == 0:
            h = (U // H // 2) * H
        self.split_at = h
        self.split = self.bounded and U >= 128 and os.environ.get("PT_SPLIT", "") == "1"
        # decode steps with an append: norms -> append -> bounded scorer, the scorer streaming
        # every tile but the units' tail tiles while the append runs (pt_append_step /
        # pt_score_bounded_step; PT_EARLY=0: append -> norms -> scorer, one PDL chain)
        self.early = (self.bounded and self.chain_norms and os.environ.get("PT_EARLY", "1") != "0"
                      and self.G <= 8 and D in (64, 128) and U <= 2048)
        self.step_sync = torch.zeros(4, dtype=torch.int32, device=d)
        # GQA groups wider than the kernels' 8 heads (e.g. 128 q / 8 kv heads): sub-groups of
        # <= 8 heads, scored separately (exact keys) and combined by a key max, one shared
        # selection, attention per sub-group (see _step_wide)
        self.subgroups: list[tuple[int, int]] = []
        if self.G > 8:
            self.bounded = False
            nsub = -(-self.G // 8)
            base, extra = divmod(self.G, nsub)
            g0 = 0
            for i in range(nsub):
                g1 = g0 + base + (1 if i < extra else 0)
                self.subgroups.append((g0, g1))
                g0 = g1
            self._wide = []
            for (a, b) in self.subgroups:
                Gs = b - a
                self._wide.append(dict(
                    G=Gs, q=None,
                    lamnorm=torch.zeros(U * 8, dtype=torch.float32, device=d),
                    keys=torch.zeros(U, Pmax, dtype=torch.int16, device=d),
                    tile_max=torch.zeros(U, Pmax // 32, dtype=torch.int16, device=d),
                    out=torch.zeros(U * Gs, D, dtype=torch.float32, device=d),
                    lse=torch.zeros(U * Gs, dtype=torch.float32, device=d),
                    ws=torch.zeros(_lib.load().pt_attend_workspace_bytes(U, Gs, D, self.k),
                                   dtype=torch.uint8, device=d),
                    tickets=torch.zeros(U, dtype=torch.int32, device=d)))

    def _bounded_pays(self, cache: PagedKvCache) -> bool:
        """Bounded scoring halves the scorer's bytes but adds the resolve step to every
        selecting CTA and needs the CTA-per-unit selection: worth it when the f32-means bytes
        it saves (at ~6.5 TB/s) clearly exceed that (>= 25 us: cfg3 saves ~80 us; cfg2 (one
        sequence) < 1 us) and -- for the CTA-per-unit selection -- the tile-maximum bound
        applies (k < pages / 32; profiles/r02/sweep_r02b.jsonl) -- for the CTA-per-unit and
        the warp-per-unit selection alike (cfg4: 107.3 vs 118.5 us/step, r02g).  PT_BOUNDED=1
        forces it."""
        if os.environ.get("PT_BOUNDED", "") == "1":
            return True
        U, P, D = cache.num_units, cache.Pmax, cache.layout.head_dim
        saved_us = U * P * D * 2 / 6.5e6
        # the selection's lower bound needs k + 1 tiles of 32 pages (else every uncertain page
        # is resolved: k = ctx/8 at 32K-128K measured 1.4-1.8x slower than exact), and the
        # bounded selection's shared memory keeps two CTAs per SM up to 16384 pages
        tile_bound = P // 32 >= self.k + 1 and P <= 16384
        return tile_bound and saved_us >= 25.0

    # ------------------------------------------------------------------
    def _q(self, q: torch.Tensor) -> tuple[torch.Tensor, int]:
        """Queries as [U*G, D] (i.e. [batch, Hq, D] with contiguous GQA grouping)."""
        q2 = q.reshape(-1, self.D)
        if q2.shape[0] != self.U * self.G:
            raise ValueError(f"{q2.shape[0]} query heads do not form {self.U} groups of {self.G}")
        if not q2.is_cuda or not q2.is_contiguous():
            raise ValueError("queries must be a contiguous device tensor")
        return q2, dev.dtype_code(q2.dtype)

    def score(self, q: torch.Tensor, norms: torch.Tensor | None = None, stream=None) -> None:
        self._step_bounded = False
        q2, qc = self._q(q)
        c = self.cache
        _lib.call("pt_score", q2.data_ptr(), qc, dev.ptr(norms), c.means.data_ptr(), c.stats_code,
                  c.stds.data_ptr(), c.seq_lens.data_ptr(), self.U, self.G, self.D,
                  c.layout.page_size, c.Pmax, self.lam, self.keys.data_ptr(),
                  dev.ptr(self.scores), self.lamnorm.data_ptr(), self.tile_max.data_ptr(),
                  dev.stream_handle(stream))

    def lam_norms(self, q: torch.Tensor, norms: torch.Tensor | None = None, stream=None,
                  chained: bool = False) -> None:
        """fl(lam * ||q_g||) for every query row (scoring.py:39-47) into the [U][8] scratch read
        by :meth:`score_prenorm`.  ``chained``: pt_lam_norms_chained (runs beside the kernel
        launched before it, completes after it)."""
        q2, qc = self._q(q)
        _lib.call("pt_lam_norms_chained" if chained else "pt_lam_norms", q2.data_ptr(), qc,
                  dev.ptr(norms), self.U, self.G, self.D, self.lam, self.lamnorm.data_ptr(),
                  dev.ptr(self.qnorm), dev.stream_handle(stream))

    def score_bounded(self, q: torch.Tensor, stream=None, u0: int = 0, nu: int | None = None) -> bool:
        """K2b over the bf16 mirror (reads the norms of :meth:`lam_norms`): key intervals into
        keys / keys_hi for units [u0, u0 + nu); False when the shape needs the exact scorer."""
        if not self.bounded:
            return False
        q2, qc = self._q(q)
        c = self.cache
        nu = self.U - u0 if nu is None else nu
        rc = _lib.load().pt_score_bounded(
            q2.data_ptr(), qc, self.lamnorm.data_ptr(), self.qnorm.data_ptr(), c.mirror.data_ptr(),
            c.stds.data_ptr(), c.seq_lens.data_ptr(), self.U, u0, nu, self.G,
            self.D, c.layout.page_size, c.Pmax, self.keys.data_ptr(), self.keys_hi.data_ptr(),
            self.tile_max.data_ptr(), dev.stream_handle(stream))
        if rc == _lib.PT_ERR_UNSUPPORTED:
            return False
        _lib.check(rc, "pt_score_bounded")
        self._step_bounded = True
        return True

    def score_step(self, q: torch.Tensor, stream=None) -> None:
        """The scoring launch of :meth:`step` (after :meth:`lam_norms`): bounded where the
        shape allows, else the exact streaming scorer, else the CTA scorer."""
        self._step_bounded = False
        if self.score_bounded(q, stream=stream):
            return
        if not self.score_prenorm(q, stream=stream):
            self.score(q, stream=stream)

    def score_prenorm(self, q: torch.Tensor, stream=None) -> bool:
        """K2 reading the norms of :meth:`lam_norms`; False when the shape needs :meth:`score`."""
        self._step_bounded = False
        q2, qc = self._q(q)
        c = self.cache
        rc = _lib.load().pt_score_prenorm(
            q2.data_ptr(), qc, self.lamnorm.data_ptr(), c.means.data_ptr(), c.stats_code,
            c.stds.data_ptr(), c.seq_lens.data_ptr(), self.U, self.G, self.D, c.layout.page_size,
            c.Pmax, self.keys.data_ptr(), dev.ptr(self.scores), self.tile_max.data_ptr(),
            dev.stream_handle(stream))
        if rc == _lib.PT_ERR_UNSUPPORTED:
            return False
        _lib.check(rc, "pt_score_prenorm")
        return True

    def select(self, stream=None) -> None:
        c = self.cache
        _lib.call("pt_topk", self.keys.data_ptr(), c.seq_lens.data_ptr(), c.page_table.data_ptr(),
                  self.U, c.layout.page_size, c.Pmax, self.k, self.sel.data_ptr(),
                  dev.ptr(self.sel_logical), self.n_sel.data_ptr(), self.kth.data_ptr(),
                  self.kplus1.data_ptr(), dev.stream_handle(stream))

    def attend(self, q: torch.Tensor, stream=None, nsplit: int = 0) -> None:
        q2, qc = self._q(q)
        c = self.cache
        _lib.call("pt_attend", q2.data_ptr(), qc, c.k_pool.data_ptr(), c.v_pool.data_ptr(),
                  c.kv_code, c.layout.max_pages, self.sel.data_ptr(), self.k, self.n_sel.data_ptr(),
                  c.page_table.data_ptr(), c.seq_lens.data_ptr(), self.U, self.G, self.D,
                  c.layout.page_size, c.Pmax, None, self.scale, self.out.data_ptr(),
                  self.lse.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
                  self.tickets.data_ptr(), nsplit, dev.stream_handle(stream))

    def dense(self, q: torch.Tensor, stream=None, nsplit: int = 0):
        """Dense paged decode over every page of every unit (the speed-up denominator)."""
        q2, qc = self._q(q)
        c = self.cache
        _lib.call("pt_attend", q2.data_ptr(), qc, c.k_pool.data_ptr(), c.v_pool.data_ptr(),
                  c.kv_code, c.layout.max_pages, c.page_table.data_ptr(), c.Pmax, None, c.page_table.data_ptr(),
                  c.seq_lens.data_ptr(), self.U, self.G, self.D, c.layout.page_size, c.Pmax,
                  None, self.scale, self.dense_out.data_ptr(), self.dense_lse.data_ptr(),
                  self.ws.data_ptr(), self.ws.numel(), self.dense_tickets.data_ptr(), nsplit,
                  dev.stream_handle(stream))
        return self.dense_out, self.dense_lse

    def score_select(self, q: torch.Tensor, norms: torch.Tensor | None = None, stream=None) -> None:
        """K2 + K3 fused into one launch (pt_score_select); falls back to two launches when
        a unit's keys exceed the fused kernel's shared-memory envelope."""
        if self.fused_select:
            q2, qc = self._q(q)
            c = self.cache
            rc = _lib.load().pt_score_select(
                q2.data_ptr(), qc, dev.ptr(norms), c.means.data_ptr(), c.stats_code,
                c.stds.data_ptr(), c.seq_lens.data_ptr(), c.page_table.data_ptr(), self.U,
                self.G, self.D, c.layout.page_size, c.Pmax, self.lam, self.k,
                self.keys.data_ptr(), dev.ptr(self.scores), self.sel.data_ptr(),
                dev.ptr(self.sel_logical), self.n_sel.data_ptr(), self.kth.data_ptr(),
                self.kplus1.data_ptr(), self.score_counters.data_ptr(),
                dev.stream_handle(stream))
            if rc == _lib.PT_OK:
                return
            if rc != _lib.PT_ERR_UNSUPPORTED:
                _lib.check(rc, "pt_score_select")
            self.fused_select = False
        self.score(q, norms, stream=stream)
        self.select(stream=stream)

    def select_attend(self, q: torch.Tensor, stream=None, u0: int = 0, nu: int | None = None) -> bool:
        """K3 + K4 in one launch (pt_select_attend): per unit, select the top-k pages from the
        keys of :meth:`score`, then attend over them -- identical outputs to :meth:`select`
        followed by :meth:`attend`, which run instead outside the fused kernel's envelope.
        A unit range [u0, u0 + nu) runs only on the fused kernel (False when unsupported)."""
        bnd = self._step_bounded
        nu_ = self.U - u0 if nu is None else nu
        if u0 != 0 or nu_ != self.U:
            q2, qc = self._q(q)
            c = self.cache
            rc = _lib.load().pt_select_attend(
                self.keys.data_ptr(), self.tile_max.data_ptr(),
                self.keys_hi.data_ptr() if bnd else None, c.mirror.data_ptr() if bnd else None,
                c.stds.data_ptr() if bnd else None, self.lamnorm.data_ptr() if bnd else None,
                c.seq_lens.data_ptr(), c.page_table.data_ptr(), self.U, u0, nu_,
                c.layout.page_size, c.Pmax, self.k, self.sel.data_ptr(),
                dev.ptr(self.sel_logical), self.n_sel.data_ptr(), self.kth.data_ptr(),
                self.kplus1.data_ptr(), q2.data_ptr(), qc, c.k_pool.data_ptr(),
                c.v_pool.data_ptr(), c.kv_code, c.layout.max_pages, self.G, self.D, self.scale,
                self.out.data_ptr(), self.lse.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
                self.tickets.data_ptr(), dev.stream_handle(stream))
            if rc == _lib.PT_ERR_UNSUPPORTED:
                return False
            _lib.check(rc, "pt_select_attend")
            return True
        if self.fused_attend or bnd:
            q2, qc = self._q(q)
            c = self.cache
            rc = _lib.load().pt_select_attend(
                self.keys.data_ptr(), self.tile_max.data_ptr(),
                self.keys_hi.data_ptr() if bnd else None, c.mirror.data_ptr() if bnd else None,
                c.stds.data_ptr() if bnd else None, self.lamnorm.data_ptr() if bnd else None,
                c.seq_lens.data_ptr(), c.page_table.data_ptr(), self.U, 0, self.U,
                c.layout.page_size, c.Pmax, self.k, self.sel.data_ptr(),
                dev.ptr(self.sel_logical), self.n_sel.data_ptr(), self.kth.data_ptr(),
                self.kplus1.data_ptr(), q2.data_ptr(), qc, c.k_pool.data_ptr(),
                c.v_pool.data_ptr(), c.kv_code, c.layout.max_pages, self.G, self.D, self.scale,
                self.out.data_ptr(), self.lse.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
                self.tickets.data_ptr(), dev.stream_handle(stream))
            if rc == _lib.PT_OK:
                return True
            if rc != _lib.PT_ERR_UNSUPPORTED:
                _lib.check(rc, "pt_select_attend")
            if bnd:
                # interval keys need the fused kernel's resolution: rescore exactly instead
                self.bounded = self._step_bounded = False
                if not self.score_prenorm(q, stream=stream):
                    self.score(q, stream=stream)
                return self.select_attend(q, stream=stream)
            self.fused_attend = False
        self.select(stream=stream)
        self.attend(q, stream=stream)
        return True

    def _step_wide(self, q: torch.Tensor, k_new, v_new, stream=None):
        """The step for G > 8 query heads per unit: per sub-group of <= 8 heads (row gathers
        of q, output scatters), lam*||q|| and exact scores; keys combined by max (the group
        max of scoring.py:108-124 split over sub-groups); one selection (pt_topk); attention
        per sub-group over the shared selection (attention.py:143-146)."""
        q2, qc = self._q(q)
        U, D, G = self.U, self.D, self.G
        c = self.cache
        sh = dev.stream_handle(stream)
        if k_new is not None:
            c.append_batch(k_new, v_new, stream=stream)
        q3 = q2.view(U, G, D)
        for i, ((a, b), w) in enumerate(zip(self.subgroups, self._wide)):
            Gs = w["G"]
            if w["q"] is None or w["q"].dtype != q2.dtype:
                w["q"] = torch.empty(U * Gs, D, dtype=q2.dtype, device=q2.device)
            w["q"].view(U, Gs, D).copy_(q3[:, a:b])
            _lib.call("pt_lam_norms", w["q"].data_ptr(), qc, None, U, Gs, D, self.lam,
                      w["lamnorm"].data_ptr(), None, sh)
            keys = self.keys if i == 0 else w["keys"]
            tmax = self.tile_max if i == 0 else w["tile_max"]
            rc = _lib.load().pt_score_prenorm(
                w["q"].data_ptr(), qc, w["lamnorm"].data_ptr(), c.means.data_ptr(), c.stats_code,
                c.stds.data_ptr(), c.seq_lens.data_ptr(), U, Gs, D, c.layout.page_size, c.Pmax,
                keys.data_ptr(), None, tmax.data_ptr(), sh)
            if rc == _lib.PT_ERR_UNSUPPORTED:
                _lib.call("pt_score", w["q"].data_ptr(), qc, None, c.means.data_ptr(), c.stats_code,
                          c.stds.data_ptr(), c.seq_lens.data_ptr(), U, Gs, D, c.layout.page_size,
                          c.Pmax, self.lam, keys.data_ptr(), None, w["lamnorm"].data_ptr(),
                          tmax.data_ptr(), sh)
            else:
                _lib.check(rc, "pt_score_prenorm")
            if i > 0:
                _lib.call("pt_keys_max", self.keys.data_ptr(), keys.data_ptr(), self.keys.numel(), sh)
                _lib.call("pt_keys_max", self.tile_max.data_ptr(), tmax.data_ptr(),
                          self.tile_max.numel(), sh)
        self._step_bounded = False
        self.select(stream=stream)
        o3, l2 = self.out.view(U, G, D), self.lse.view(U, G)
        for (a, b), w in zip(self.subgroups, self._wide):
            Gs = w["G"]
            _lib.call("pt_attend", w["q"].data_ptr(), qc, c.k_pool.data_ptr(), c.v_pool.data_ptr(),
                      c.kv_code, c.layout.max_pages, self.sel.data_ptr(), self.k,
                      self.n_sel.data_ptr(), c.page_table.data_ptr(), c.seq_lens.data_ptr(), U, Gs,
                      D, c.layout.page_size, c.Pmax, None, self.scale, w["out"].data_ptr(),
                      w["lse"].data_ptr(), w["ws"].data_ptr(), w["ws"].numel(),
                      w["tickets"].data_ptr(), 0, sh)
            o3[:, a:b].copy_(w["out"].view(U, Gs, D))
            l2[:, a:b].copy_(w["lse"].view(U, Gs))
        return self.out, self.lse

    def step(self, q: torch.Tensor, k_new: torch.Tensor | None = None,
             v_new: torch.Tensor | None = None, stream=None):
        """One decode step: [append] -> score -> select+attend.  Returns (out, lse)."""
        if self.subgroups:
            if stream is not None:
                with torch.cuda.stream(stream):
                    return self._step_wide(q, k_new, v_new, stream)
            return self._step_wide(q, k_new, v_new)
        if self.fused_select:
            if k_new is not None:
                self.cache.append_batch(k_new, v_new, stream=stream)
            self.score_select(q, stream=stream)
            self.attend(q, stream=stream)
            return self.out, self.lse
        # the query norms do not depend on the append: with PDL they run beside it as the next
        # link of one chain (append -> norms -> score -> select+attend); without PDL, on a
        # side stream (a fork/join that CUDA-graph capture records as two parallel branches)
        main = stream if stream is not None else torch.cuda.current_stream()
        if (self.early and not self.split and k_new is not None and self.bounded
                and q.dtype == torch.bfloat16):
            # the norms first (they store after the previous step's select+attend), then the
            # append and the scorer that overlaps it -- a paired launch: nothing between them
            # may fail (shape checks above mirror pt_score_bounded's envelope)
            q2, qc = self._q(q)
            c = self.cache
            self.lam_norms(q, stream=main, chained=True)
            self.cache.append_batch(k_new, v_new, stream=main, step_sync=self.step_sync)
            _lib.call("pt_score_bounded_step", q2.data_ptr(), qc, self.lamnorm.data_ptr(),
                      self.qnorm.data_ptr(), c.mirror.data_ptr(), c.stds.data_ptr(),
                      c.seq_lens.data_ptr(), self.U, self.G, self.D, c.layout.page_size, c.Pmax,
                      self.keys.data_ptr(), self.keys_hi.data_ptr(), self.tile_max.data_ptr(),
                      c._slot.data_ptr(), self.step_sync.data_ptr(), dev.stream_handle(main))
            self._step_bounded = True
            self.select_attend(q, stream=main)
            return self.out, self.lse
        if self.chain_norms:
            if k_new is not None:
                self.cache.append_batch(k_new, v_new, stream=main)
            self.lam_norms(q, stream=main, chained=True)
        else:
            self._side.wait_stream(main)
            self.lam_norms(q, stream=self._side)
            if k_new is not None:
                self.cache.append_batch(k_new, v_new, stream=main)
            main.wait_stream(self._side)
        if self.split and self.bounded:
            # two half-batches: the first half's select+attend (side stream) runs beside the
            # second half's scorer -- its selection prologue no longer leaves HBM idle
            # (tools/probe_overlap.py: 143.5 vs 153 us for score + select+attend at cfg3)
            h = self.split_at
            self._step_bounded = False
            if self.score_bounded(q, stream=main, u0=0, nu=h):
                ev = torch.cuda.Event()
                ev.record(main)
                self._side.wait_event(ev)
                ok = self.select_attend(q, stream=self._side, u0=0, nu=h)
                ok = ok and self.score_bounded(q, stream=main, u0=h, nu=self.U - h)
                ok = ok and self.select_attend(q, stream=main, u0=h, nu=self.U - h)
                main.wait_stream(self._side)
                if ok:
                    return self.out, self.lse
                self.split = False  # outside the fused kernel's envelope: the one-range step
        self.score_step(q, stream=main)
        self.select_attend(q, stream=main)
        return self.out, self.lse

    # ------------------------------------------------------------------
    def capture(self, q: torch.Tensor, k_new: torch.Tensor | None = None,
                v_new: torch.Tensor | None = None) -> torch.cuda.CUDAGraph:
        """Capture one step (static input buffers q/k_new/v_new) as a CUDA graph.

        With appends, each replay advances every unit by one token (the host mirror of
        the sequence lengths is advanced by :meth:`replay`).
        """
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                self.step(q, k_new, v_new)
                if k_new is not None:
                    self.cache._seq_host -= 1  # replay() accounts for the captured append
        torch.cuda.current_stream().wait_stream(s)
        self.graph = g
        self._graph_appends = k_new is not None
        return g

    def replay(self) -> None:
        assert self.graph is not None, "capture() first"
        self.graph.replay()
        if self._graph_appends:
            self.cache._seq_host += 1
