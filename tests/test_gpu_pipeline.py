"""PipelinedDecoder (the serving loop: pinned host inputs -> H2D -> captured step graph ->
D2H, double-buffered through runtime.cu's native pt_pipe_submit) against the eager engine:
over many steps with appends and a different query every step, every step's host output is
bit-identical to the eager step's on an identical cache, and the caches end identical."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _cache(seed, U, n, D, S):
    import paper_2605_27740_b200 as pt

    rng = np.random.default_rng(seed)
    Pcap = -(-n // S) + 8
    layout = pt.CacheLayout(num_kv_heads=2, head_dim=D, page_size=S, max_pages=U * Pcap)
    c = pt.PagedKvCache(layout, batch=U // 2, dtype=torch.bfloat16, max_pages_per_head=Pcap)
    K = rng.standard_normal((U, n, D)).astype(np.float32)
    V = rng.standard_normal((U, n, D)).astype(np.float32)
    c.extend_units(torch.from_numpy(K), torch.from_numpy(V))
    return c


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_pipelined_steps_equal_eager_steps(cuda, depth):
    import paper_2605_27740_b200 as pt

    U, D, S, G, k, n = 4, 128, 16, 4, 16, 16 * 200 + 3
    ca, cb = _cache(1, U, n, D, S), _cache(1, U, n, D, S)
    dec = pt.PipelinedDecoder(ca, G, k, depth=depth)
    eng = pt.DecodeEngine(cb, G, k)
    rng = np.random.default_rng(2)
    steps = 24
    host_in = [torch.from_numpy(rng.standard_normal(dec.in_numel).astype(np.float32))
               .to(torch.bfloat16).pin_memory() for _ in range(steps + depth)]
    # warm-up steps (one per slot) consume the first inputs on both sides
    for i in range(depth):
        x = host_in[i].cuda()
        q, kn, vn = x[: dec.nq].view(-1, D), x[dec.nq:dec.nq + dec.nk].view(U, D), x[dec.nq + dec.nk:].view(U, D)
        eng.step(q, kn, vn)
    # PipelinedDecoder.capture runs its own warm step per slot from each slot's input block
    for i in range(depth):
        dec.inputs[i].copy_(host_in[i].cuda())
    dec.capture()
    outs = [torch.empty(U * G, D, dtype=torch.float32).pin_memory() for _ in range(steps)]
    for t in range(steps):
        dec.submit(host_in[depth + t], outs[t])
    dec.synchronize()
    for t in range(steps):
        x = host_in[depth + t].cuda()
        q, kn, vn = x[: dec.nq].view(-1, D), x[dec.nq:dec.nq + dec.nk].view(U, D), x[dec.nq + dec.nk:].view(U, D)
        o, _ = eng.step(q, kn, vn)
        torch.testing.assert_close(outs[t], o.cpu(), rtol=0, atol=0)
    ca.check_errors()
    cb.check_errors()
    assert [ca.seq_len(u) for u in range(U)] == [cb.seq_len(u) for u in range(U)] == [n + depth + steps] * U
    assert torch.equal(ca.seq_lens, cb.seq_lens)
    assert torch.equal(ca.stds, cb.stds)


def test_submit_rejects_pageable_buffers(cuda):
    import paper_2605_27740_b200 as pt

    c = _cache(3, 2, 64, 128, 16)
    dec = pt.PipelinedDecoder(c, 4, 4)
    dec.capture()
    with pytest.raises(ValueError):
        dec.submit(torch.zeros(dec.in_numel, dtype=torch.bfloat16), torch.zeros(8, 128))
