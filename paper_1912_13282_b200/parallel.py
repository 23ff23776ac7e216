"""Multi-process sharding of the hot path (one process per GPU).

kNN, the shape solve and the CSR rows are independent per target, so they
shard by contiguous target blocks with no data-path collective (positions are
replicated).  The only exchange is the explicit apply / heat step on a
row-partitioned operator, which needs the field at every stencil column: one
all-gather of the field per application (NCCL over NVLink on GPUs; gloo in the
CPU tests).  These helpers hold that partition and exchange logic; the local
row application is the plan apply of the rank's own CSR block.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous block [lo, hi) of `total` items for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(int(total), world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass
class RowPartition:
    total: int
    world: int
    rank: int

    @property
    def bounds(self):
        return [shard_range(self.total, self.world, r) for r in range(self.world)]

    @property
    def lo(self) -> int:
        return self.bounds[self.rank][0]

    @property
    def hi(self) -> int:
        return self.bounds[self.rank][1]

    @property
    def counts(self):
        return [hi - lo for lo, hi in self.bounds]

    def targets(self) -> np.ndarray:
        """Target node indices this rank computes stencils/weights for."""
        return np.arange(self.lo, self.hi, dtype=np.int64)


def allgather_field(u_local: torch.Tensor, part: RowPartition, group=None) -> torch.Tensor:
    """Concatenate every rank's block of the field (rank order) on every rank."""
    counts = part.counts
    width = max(counts)
    if u_local.shape[0] != counts[part.rank]:
        raise ValueError("local block has the wrong length")
    padded = torch.zeros(width, dtype=u_local.dtype, device=u_local.device)
    padded[: u_local.shape[0]] = u_local
    gathered = torch.empty(part.world * width, dtype=u_local.dtype, device=u_local.device)
    if hasattr(dist, "all_gather_into_tensor") and u_local.is_cuda:
        dist.all_gather_into_tensor(gathered, padded, group=group)
    else:
        chunks = list(gathered.view(part.world, width).unbind(0))
        dist.all_gather(chunks, padded, group=group)
        gathered = torch.stack(chunks).reshape(-1)
    blocks = gathered.view(part.world, width)
    return torch.cat([blocks[r, :c] for r, c in enumerate(counts)])


def distributed_apply(local_apply, u_local: torch.Tensor, part: RowPartition, group=None) -> torch.Tensor:
    """y[lo:hi] = (A u)[lo:hi] for a row-partitioned operator.

    ``local_apply(u_full) -> y_block`` applies this rank's CSR rows (column
    indices are global) to the gathered field.
    """
    u_full = allgather_field(u_local, part, group)
    return local_apply(u_full)


def distributed_heat_steps(local_step, u_local: torch.Tensor, part: RowPartition, steps: int, group=None):
    """`steps` explicit steps, one field exchange per step (drivers.py:88-103 per block)."""
    for _ in range(steps):
        u_full = allgather_field(u_local, part, group)
        u_local = local_step(u_full, u_local)
    return u_local
