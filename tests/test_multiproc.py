"""Multi-GPU sharding logic on CPU: world_size-2 gloo process group.

Each rank runs the decode step for its own unit shard (here through the CPU oracle,
the only compute available without a GPU) and the optional output all-gather
reassembles the full [B*Hq, D] result, which must equal the unsharded step exactly.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_27740_b200.shard import gather_outputs, shard_units


def test_shard_units_cover_every_unit_once():
    for batch in (1, 2, 3, 32, 64):
        for H in (1, 8, 16):
            for world in (1, 2, 3, 4, 8):
                seen = []
                for r in range(world):
                    s = shard_units(batch, H, 4, world, r)
                    seen.extend(range(s.u0, s.u1))
                    assert s.q_rows == (s.u0 * 4, s.u1 * 4)
                assert seen == list(range(batch * H))
                if batch % world == 0:  # whole sequences per rank
                    for r in range(world):
                        s = shard_units(batch, H, 4, world, r)
                        assert s.u0 % H == 0 and s.num_units == batch // world * H


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(seed=5, B=3, H=2, G=4, D=32, S=8, N=200, k=6):
    rng = np.random.default_rng(seed)
    U = B * H
    P = -(-N // S)
    kpool = rng.standard_normal((U * P, S, D)).astype(np.float32)
    vpool = rng.standard_normal((U * P, S, D)).astype(np.float32)
    table = np.arange(U * P, dtype=np.int32).reshape(U, P)
    seq = np.full(U, N, np.int32)
    q = rng.standard_normal((U, G, D)).astype(np.float32)
    return dict(B=B, H=H, G=G, D=D, S=S, k=k, kpool=kpool, vpool=vpool, table=table, seq=seq, q=q)


def _worker(rank, world, port, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O

    p = _problem()
    sh = shard_units(p["B"], p["H"], p["G"], world, rank)
    u = slice(sh.u0, sh.u1)
    means, stds = O.build_stats(p["kpool"], p["table"][u], p["seq"][u], p["S"])
    r = O.decode_units(p["q"][u], p["kpool"], p["vpool"], p["table"][u], p["seq"][u], means, stds,
                       p["k"], 0.5, 1 / np.sqrt(p["D"]), p["S"])
    local = torch.from_numpy(r["out"].reshape(-1, p["D"]))
    full = gather_outputs(local, sh, p["B"] * p["H"])
    # max-over-ranks timing reduction used by bench.py
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        result_q.put((full.numpy(), float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_step_gathers_to_the_unsharded_result(world):
    from oracle import oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    full, tmax = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    p = _problem()
    means, stds = O.build_stats(p["kpool"], p["table"], p["seq"], p["S"])
    r = O.decode_units(p["q"], p["kpool"], p["vpool"], p["table"], p["seq"], means, stds, p["k"],
                       0.5, 1 / np.sqrt(p["D"]), p["S"])
    np.testing.assert_array_equal(full, r["out"].reshape(-1, p["D"]))
    assert tmax == float(world)
