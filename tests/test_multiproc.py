"""Multi-GPU sharding logic on CPU: world_size-2 gloo process groups.

Each rank runs bench.py's multi-rank plumbing -- shard_units, the per-unit workload
generators, Ctx (rank / gloo / max-over-ranks) -- and computes its shard's decode step
(through the CPU oracle, the only compute available without a GPU); the optional output
all-gather reassembles the full [B*Hq, D] result, which must equal the unsharded step
exactly.  The same path on the GPU is tests/test_gpu_multirank.py.
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


def _args(batch=4):
    import bench

    return bench.parse(["--batch", str(batch), "--ctx", "200", "--q-heads", "8", "--kv-heads", "2",
                        "--head-dim", "32", "--page", "8", "--budget", "48"])


def _units_step(args, units, q_rows):
    """The decode step for global units ``units`` on the bench workload (bench.unit_rows /
    bench.step_inputs on the CPU generator), computed by the oracle (no GPU here)."""
    import bench
    from oracle import oracle as O

    D, S = args.head_dim, args.page
    G = args.q_heads // args.kv_heads
    ks, vs = [], []
    for kk, vv in bench.unit_rows(args, "cpu", bench.SEED, units, chunk=64):
        ks.append(kk.float().numpy())
        vs.append(vv.float().numpy())
    K, V = np.concatenate(ks, axis=1), np.concatenate(vs, axis=1)
    Ul, n = K.shape[0], K.shape[1]
    P = -(-n // S)
    kpool = np.zeros((Ul * P, S, D), np.float32)
    vpool = np.zeros((Ul * P, S, D), np.float32)
    for i in range(Ul):
        kpool[i * P:(i + 1) * P].reshape(-1, D)[:n] = K[i]
        vpool[i * P:(i + 1) * P].reshape(-1, D)[:n] = V[i]
    table = (np.arange(Ul)[:, None] * P + np.arange(P)[None, :]).astype(np.int32)
    seq = np.full(Ul, n, np.int32)
    qs, _, _ = bench.step_inputs(args, "cpu", NQ=1)
    q = qs[0][q_rows[0]:q_rows[1]].float().numpy().reshape(Ul, G, D)
    means, stds = O.build_stats(kpool, table, seq, S)
    k = -(-args.budget // S)
    r = O.decode_units(q, kpool, vpool, table, seq, means, stds, k, 0.5, 1 / np.sqrt(D), S)
    return r["out"].reshape(-1, D)


def _worker(rank, world, port, batch, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank), BENCH_DIST_BACKEND="gloo")
    import bench

    ctx = bench.Ctx()  # the bench's rank / collective plumbing (gloo here)
    args = _args(batch)
    G = args.q_heads // args.kv_heads
    sh = shard_units(args.batch, args.kv_heads, G, ctx.world, ctx.rank)
    local = torch.from_numpy(_units_step(args, range(sh.u0, sh.u1), sh.q_rows))
    full = gather_outputs(local, sh, args.batch * args.kv_heads)
    tmax = ctx.max(float(rank + 1))  # max-over-ranks timing reduction of bench.py
    if rank == 0:
        result_q.put((full.numpy(), tmax))
    ctx.barrier()
    ctx.close()


@pytest.mark.parametrize("world,batch", [(2, 4), (2, 3)])
def test_sharded_step_gathers_to_the_unsharded_result(world, batch):
    """world ranks on gloo run bench.py's sharding (shard_units), workload generation
    (unit_rows / step_inputs: per-unit generators) and collectives (Ctx, gather_outputs);
    the gathered step equals the unsharded one bit for bit (batch 3 over 2 ranks splits a
    sequence's kv-heads)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, batch, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    full, tmax = q.get(timeout=180)
    for pr in procs:
        pr.join(timeout=180)
        assert pr.exitcode == 0
    args = _args(batch)
    G = args.q_heads // args.kv_heads
    U = args.batch * args.kv_heads
    ref = _units_step(args, range(U), (0, U * G))
    np.testing.assert_array_equal(full, ref)
    assert tmax == float(world)


def test_unit_rows_are_shard_stable():
    """A shard's rows equal the corresponding rows of the unsharded workload."""
    import bench

    args = _args(4)
    whole = [k.float() for k, _ in bench.unit_rows(args, "cpu", bench.SEED, range(8), chunk=64)]
    part = [k.float() for k, _ in bench.unit_rows(args, "cpu", bench.SEED, range(3, 6), chunk=64)]
    for a, b in zip(whole, part):
        assert torch.equal(a[3:6], b)
