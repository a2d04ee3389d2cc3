"""Multi-GPU partition of the decode step: units (sequence, kv-head) across ranks.

Every unit's score -> select -> attend is independent (attention.py:137-146), so the
step shards with no data-path collective: rank r owns a contiguous range of units
``[u0, u1)`` (batch-major, so whole sequences stay together whenever the batch
divides evenly; kv-head granularity when there are fewer sequences than ranks).
Its query rows are the contiguous block ``[u0*G, u1*G)`` of the [B*Hq, D] query
matrix (contiguous GQA grouping), its KV pages live only in its own HBM.

The one optional collective is the output all-gather of the [B*Hq, D] result
(NCCL over NVLink/NVSwitch on GPUs; gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["UnitShard", "shard_units", "gather_outputs"]


@dataclass(frozen=True)
class UnitShard:
    rank: int
    world: int
    u0: int
    u1: int
    group_size: int

    @property
    def num_units(self) -> int:
        return self.u1 - self.u0

    @property
    def q_rows(self) -> tuple[int, int]:
        """Rows of the [U*G, D] query/output matrix owned by this rank."""
        return self.u0 * self.group_size, self.u1 * self.group_size

    def sequences(self, num_kv_heads: int) -> tuple[int, int]:
        """Sequence range touched by this shard (first, last+1)."""
        if self.num_units == 0:
            return (0, 0)
        return self.u0 // num_kv_heads, (self.u1 - 1) // num_kv_heads + 1


def shard_units(batch: int, num_kv_heads: int, group_size: int, world: int, rank: int) -> UnitShard:
    """Balanced contiguous split of the batch*num_kv_heads units over `world` ranks.

    Whole sequences per rank when ``batch % world == 0``; otherwise the split falls on
    kv-head boundaries (the remainder units go to the lowest ranks).
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    U = batch * num_kv_heads
    if batch % world == 0:
        per = batch // world
        return UnitShard(rank, world, rank * per * num_kv_heads, (rank + 1) * per * num_kv_heads,
                         group_size)
    base, extra = divmod(U, world)
    u0 = rank * base + min(rank, extra)
    u1 = u0 + base + (1 if rank < extra else 0)
    return UnitShard(rank, world, u0, u1, group_size)


def gather_outputs(local_out, shard: UnitShard, total_units: int, group=None):
    """All-gather each rank's [units*G, D] output block into the full [U*G, D] matrix.

    Uses torch.distributed (NCCL for CUDA tensors, gloo for CPU tensors); ranks may
    own different unit counts, so blocks are padded to the largest shard.
    """
    import torch
    import torch.distributed as dist

    G = shard.group_size
    world = shard.world
    sizes = [shard_units_size(total_units, world, r) for r in range(world)]
    width = max(sizes) * G
    pad = torch.zeros(width, *local_out.shape[1:], dtype=local_out.dtype, device=local_out.device)
    pad[: local_out.shape[0]] = local_out
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[: s * G] for b, s in zip(bufs, sizes)], dim=0)


def shard_units_size(total_units: int, world: int, rank: int) -> int:
    base, extra = divmod(total_units, world)
    return base + (1 if rank < extra else 0)
