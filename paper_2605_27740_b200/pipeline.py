"""Host-facing decode loop: pinned host buffers in, pinned host results out, overlapped.

The serving path around :class:`DecodeEngine` (attention.py:110-147 for every unit of a
:class:`PagedKvCache`, one decode token per sequence per step).  Each step takes the
step's inputs -- queries [U*G, D], new key and value rows [U, D], packed in one pinned
host block -- and produces the step's outputs [U*G, D] f32 in a pinned host buffer.

B200 structure: ``depth`` (default 2) engines over the same cache, each with its own
static device input block and a captured CUDA graph of the whole step.  Step n uses slot
n % depth:

    h2d stream     H2D of step n's inputs      (waits until step n - depth released the slot)
    compute stream graph replay of step n       (waits for its inputs and for the D2H of
                                                 step n - depth, which reads the same outputs)
    d2h stream     D2H of step n's outputs      (waits for the replay)

so the PCIe transfers of step n + 1 and step n - 1 run under the kernels of step n.  Steps
still execute in order on the compute stream (each appends one token to every unit).  The
per-step host work is one native call (runtime.cu pt_pipe_submit: the copies, the graph
launch and the event edges), so the host keeps ahead of a ~180 us device step.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .engine import DecodeEngine
from .kvcache import PagedKvCache

__all__ = ["PipelinedDecoder"]


class PipelinedDecoder:
    def __init__(self, cache: PagedKvCache, group_size: int, k: int, lam: float = 0.5,
                 scale: float | None = None, depth: int = 2) -> None:
        if depth < 1:
            raise ValueError("depth must be positive")
        self.cache = cache
        U, D = cache.num_units, cache.layout.head_dim
        G = group_size
        self.nq, self.nk = U * G * D, U * D
        self.in_numel = self.nq + 2 * self.nk
        self.out_shape = (U * G, D)
        self.depth = depth
        dev = cache.device
        self.engines = [DecodeEngine(cache, G, k, lam=lam, scale=scale) for _ in range(depth)]
        self.inputs = [torch.zeros(self.in_numel, dtype=cache.dtype, device=dev) for _ in range(depth)]
        self.compute = torch.cuda.current_stream(dev)
        self.h2d = torch.cuda.Stream(device=dev)
        self.d2h = torch.cuda.Stream(device=dev)
        h = ctypes.c_void_p()
        _lib.call("pt_pipe_create", self.compute.cuda_stream, self.h2d.cuda_stream,
                  self.d2h.cuda_stream, depth, ctypes.byref(h))
        self._pipe = h
        self._execs: list[int] = []
        self.steps = 0
        self._captured = False

    def __del__(self):
        pipe = getattr(self, "_pipe", None)
        if pipe is not None and pipe.value:
            try:
                self.synchronize()
                _lib.load().pt_pipe_destroy(pipe)
            except Exception:
                pass
            self._pipe = None

    def _views(self, i: int):
        x = self.inputs[i]
        U, D = self.cache.num_units, self.cache.layout.head_dim
        q = x[: self.nq].view(-1, D)
        kn = x[self.nq : self.nq + self.nk].view(U, D)
        vn = x[self.nq + self.nk :].view(U, D)
        return q, kn, vn

    def capture(self, warm_input: torch.Tensor | None = None) -> None:
        """Capture every slot's step graph (after one eager warm-up step per slot, which
        appends a token: warm_input, or the slot's current input block)."""
        for i, e in enumerate(self.engines):
            if warm_input is not None:
                self.inputs[i].copy_(warm_input)
            q, kn, vn = self._views(i)
            e.step(q, kn, vn)  # eager warm-up: kernel attributes, fused-path decisions
        torch.cuda.synchronize()
        self.cache.check_errors()
        for i, e in enumerate(self.engines):
            e.capture(*self._views(i))
        self._execs = [int(e.graph.raw_cuda_graph_exec()) for e in self.engines]
        self._captured = True

    def submit(self, host_in: torch.Tensor, host_out: torch.Tensor) -> int:
        """Queue one step: H2D of ``host_in`` (pinned, ``in_numel`` elements of the cache
        dtype: q | k_new | v_new), the step, D2H of its outputs into ``host_out`` (pinned f32
        [U*G, D]).  Returns the step's slot (``wait(slot)`` blocks until ``host_out`` holds
        the result)."""
        if not self._captured:
            raise RuntimeError("capture() first")
        if host_in.numel() != self.in_numel or host_out.shape != self.out_shape:
            raise ValueError("host buffers do not match the cache / group shape")
        i = self.steps % self.depth
        e = self.engines[i]
        if not (host_in.is_pinned() and host_out.is_pinned()) or host_in.dtype != self.cache.dtype \
                or host_out.dtype != torch.float32:
            raise ValueError("host buffers must be pinned, of the cache dtype (in) and f32 (out)")
        _lib.call("pt_pipe_submit", self._pipe, i, self._execs[i], self.inputs[i].data_ptr(),
                  host_in.data_ptr(), host_in.numel() * host_in.element_size(),
                  host_out.data_ptr(), e.out.data_ptr(), host_out.numel() * host_out.element_size())
        if e._graph_appends:
            self.cache._seq_host += 1  # the replayed step appended one token per unit
        self.steps += 1
        return i

    def wait(self, slot: int) -> None:
        """Block until the outputs of the last step submitted on ``slot`` are on the host."""
        _lib.call("pt_pipe_wait", self._pipe, slot)

    def synchronize(self) -> None:
        self.h2d.synchronize()
        self.compute.synchronize()
        self.d2h.synchronize()
