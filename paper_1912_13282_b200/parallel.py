"""Multi-process sharding of the hot path (one process per GPU).

kNN, the shape solve and the CSR rows are independent per target, so they
shard by contiguous target blocks with no data-path collective (positions are
replicated).  The only exchange is the explicit apply / heat step on a
row-partitioned operator, which needs the field at every stencil column: one
all-gather of the field per application (NCCL over NVLink on GPUs; gloo in the
CPU tests).  These helpers hold that partition and exchange logic; the local
row application is the rank's own CSR rows (global column indices) applied to
the gathered field on the GPU (``mf_apply`` on the canonical CSR slice, then
``mf_heat_rows`` for the explicit step).

``ShardedProblem`` is the product path: one node set, positions replicated,
the rank's target block through find_closest_stencils and compute_weights
(global pool, global columns), and ``ShardedOperator`` per family for the
exchanged application and the row-partitioned heat loop.
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes

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


def world_and_rank(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


class ShardedOperator:
    """This rank's rows [lo, hi) of one operator family, global columns.

    ``indptr`` is the N+1 canonical CSR row pointer whose rows outside [lo, hi)
    are empty, so the block is the pointer slice [lo, hi] with indices / data
    addressed absolutely (no copy).  ``local_apply(u_full) -> y_block`` defaults
    to the GPU CSR product (mf_apply); tests may inject a host one.
    """

    def __init__(self, indptr, indices, data, part: RowPartition, group=None, local_apply=None):
        self.part, self.group = part, group
        self.indptr, self.indices, self.data = indptr, indices, data
        self._local = local_apply or self._gpu_apply

    @classmethod
    def from_store(cls, store, key, part: RowPartition, group=None):
        mat = store.matrix(key)
        return cls(mat.indptr_device, mat.indices_device, mat.data_device, part, group)

    def _gpu_apply(self, u_full: torch.Tensor) -> torch.Tensor:
        from . import _lib

        lo, hi = self.part.lo, self.part.hi
        y = torch.empty(hi - lo, dtype=torch.float64, device=u_full.device)
        if hi > lo:
            ip = self.indptr[lo:]  # absolute offsets into indices / data
            _lib.check(_lib.load().mf_apply(ip.data_ptr(), self.indices.data_ptr(), self.data.data_ptr(),
                                            u_full.data_ptr(), y.data_ptr(), hi - lo, _lib.stream_ptr()),
                       "mf_apply")
        return y

    def apply(self, u_local: torch.Tensor) -> torch.Tensor:
        """(A u)[lo:hi] from this rank's block of u: one all-gather, then the rows."""
        return distributed_apply(self._local, u_local, self.part, self.group)


class ShardedProblem:
    """One node set sharded by target blocks over the process group.

    Positions (and the kNN pool) are replicated; each rank selects stencils and
    computes weights for its targets only, so the data path has no
    collective until an operator is applied.
    """

    def __init__(self, nodes, n, engine, families, *, group=None, part: RowPartition | None = None):
        from .stencils import find_closest_stencils
        from .storage import compute_weights

        world, rank = world_and_rank(group)
        self.part = part or RowPartition(len(nodes), world, rank)
        self.group = group
        targets = self.part.targets()
        self.nodes = find_closest_stencils(nodes, n, for_which=targets)
        self.store = compute_weights(self.nodes, engine, families, for_which=targets)
        self._ops = {}

    def operator(self, key) -> ShardedOperator:
        if key not in self._ops:
            self._ops[key] = ShardedOperator.from_store(self.store, key, self.part, self.group)
        return self._ops[key]

    def apply_all(self, key, u_local: torch.Tensor) -> torch.Tensor:
        return self.operator(key).apply(u_local)

    def heat_steps(self, u_local: torch.Tensor, *, dt, steps, interior, dirichlet, g_dirichlet,
                   diffusivity=1.0, source=None, key="laplacian"):
        """Row-partitioned forward Euler: per step one field exchange, the local
        Laplacian rows, and the fused update (mf_heat_rows).  Masks / values are
        this rank's blocks (device tensors).  Returns the block and the per-step
        peaks of |u| on this rank (IEEE bits)."""
        from . import _lib

        op = self.operator(key)
        lib = _lib.load()
        peaks = torch.zeros(max(int(steps), 1), dtype=torch.int64, device=u_local.device)
        out = torch.empty_like(u_local)
        for s_ in range(int(steps)):
            lap = op.apply(u_local)
            _lib.check(lib.mf_heat_rows(lap.data_ptr(), u_local.data_ptr(), interior.data_ptr(),
                                        dirichlet.data_ptr(), g_dirichlet.data_ptr(), _lib.ptr(source),
                                        float(dt), float(diffusivity), u_local.shape[0], out.data_ptr(),
                                        peaks[s_:].data_ptr(), _lib.stream_ptr()), "mf_heat_rows")
            u_local, out = out, u_local
        return u_local, peaks
