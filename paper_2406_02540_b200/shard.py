"""Token-row sharding of the quantized-linear path across ranks.

Per-token activation params depend only on their own row (quant.cpp:70-73:
one group per row) and the integer dot is per (row, out-channel)
(qgemm.cpp:52-63), so rows shard with no collective inside the layer:
rank r owns rows [r*M/P, (r+1)*M/P) of every linear's activations; weights
(and s_w, sum w, smoothing, signs) are replicated.  The only collective is the
verification all-gather of outputs after timing.
"""
from __future__ import annotations

from typing import Callable


def row_range(M: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced row range of `rank` (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    return (M * rank) // world, (M * (rank + 1)) // world


def gather_rows(local, M: int, group=None):
    """All-gather row shards (uneven sizes allowed) into the full [M, ...]
    tensor on every rank.  Uses the process group's backend (NCCL over
    NVLink on the GPU box, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = row_range(M, rank, world)
    assert local.shape[0] == hi - lo
    size = max(row_range(M, r, world)[1] - row_range(M, r, world)[0] for r in range(world))
    pad = torch.zeros((size,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: hi - lo] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    out = []
    for r in range(world):
        a, b = row_range(M, r, world)
        out.append(parts[r][: b - a])
    return torch.cat(out, 0)


def sharded_apply(x, fn: Callable, group=None):
    """Apply a row-local function to this rank's row shard of the full input
    `x` and all-gather the result (the equality-check harness)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = row_range(x.shape[0], rank, world)
    return gather_rows(fn(x[lo:hi]), x.shape[0], group)
