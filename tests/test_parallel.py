"""Row-partitioned exchange logic with gloo, world size 2, on CPU.

The local row operator here is a CPU reference product supplied by the test
(the product path applies its rows on the GPU); what is under test is the
partition, the all-gather with uneven blocks, and the per-step exchange.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1912_13282_b200.parallel import RowPartition, distributed_apply, distributed_heat_steps, shard_range


def test_shard_range_covers_everything():
    for total in (0, 1, 7, 10, 1001):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_range(total, world, r)
                seen.extend(range(lo, hi))
                assert hi - lo in (total // world, total // world + 1)
            assert seen == list(range(total))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, N, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    # random sparse operator with 5 entries per row, dense copy for the check
    cols = rng.integers(0, N, (N, 5))
    vals = rng.standard_normal((N, 5))
    A = np.zeros((N, N))
    for i in range(N):
        for c, v in zip(cols[i], vals[i]):
            A[i, c] += v
    u = rng.standard_normal(N)
    part = RowPartition(N, world, rank)
    block = torch.from_numpy(A[part.lo:part.hi])
    y_local = distributed_apply(lambda uf: block @ uf, torch.from_numpy(u[part.lo:part.hi]), part)
    ys = [None] * world
    dist.all_gather_object(ys, y_local.numpy())
    # three explicit steps u <- u + dt A u
    dt = 1e-2
    step = lambda uf, ul: ul + dt * (block @ uf)
    u_end = distributed_heat_steps(step, torch.from_numpy(u[part.lo:part.hi]), part, 3)
    us = [None] * world
    dist.all_gather_object(us, u_end.numpy())
    if rank == 0:
        ref = u.copy()
        for _ in range(3):
            ref = ref + dt * (A @ ref)
        out.put((np.allclose(np.concatenate(ys), A @ u, rtol=0, atol=1e-12),
                 np.allclose(np.concatenate(us), ref, rtol=0, atol=1e-12)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("N", [11, 64])
def test_gloo_world2_apply_and_heat(N):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, N, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    ok_apply, ok_heat = out.get(timeout=10)
    assert ok_apply and ok_heat
