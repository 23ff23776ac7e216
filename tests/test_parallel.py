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


def _sharded_worker(rank, world, port, N, out):
    """ShardedOperator over the canonical-CSR slice of each rank's rows (global
    columns), with a host product injected for the local rows (CPU test)."""
    import scipy.sparse

    from paper_1912_13282_b200.parallel import ShardedOperator

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(3)
    n = 7
    stencils = np.stack([np.concatenate([[i], rng.choice(np.delete(np.arange(N), i), n - 1, replace=False)])
                         for i in range(N)])
    vals = rng.standard_normal((N, n))
    part = RowPartition(N, world, rank)
    lo, hi = part.lo, part.hi
    # this rank's store: rows lo..hi only -> canonical N x N CSR with empty rows elsewhere
    rows = np.repeat(np.arange(lo, hi), n)
    A_loc = scipy.sparse.csr_matrix((vals[lo:hi].ravel(), (rows, stencils[lo:hi].ravel())), shape=(N, N))
    A_loc.sort_indices()
    ip, ix, da = (torch.from_numpy(A_loc.indptr.astype(np.int32)), torch.from_numpy(A_loc.indices.astype(np.int32)),
                  torch.from_numpy(A_loc.data))

    def host_rows(u_full):  # the rows lo..hi addressed through the slice, as mf_apply does
        ipl = ip[lo:].numpy()
        y = np.zeros(hi - lo)
        for k in range(hi - lo):
            acc = 0.0
            for p in range(ipl[k], ipl[k + 1]):
                acc = acc + da.numpy()[p] * u_full.numpy()[ix.numpy()[p]]
            y[k] = acc
        return torch.from_numpy(y)

    op = ShardedOperator(ip, ix, da, part, local_apply=host_rows)
    u = rng.standard_normal(N)
    y_loc = op.apply(torch.from_numpy(u[lo:hi]))
    ys = [None] * world
    dist.all_gather_object(ys, y_loc.numpy())
    if rank == 0:
        full = scipy.sparse.csr_matrix((vals.ravel(), (np.repeat(np.arange(N), n), stencils.ravel())), shape=(N, N))
        full.sort_indices()
        out.put(bool(np.array_equal(np.concatenate(ys), full @ u)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("N", [9, 50])
def test_gloo_world2_sharded_operator_slices(N):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, N, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert out.get(timeout=10)


@pytest.mark.gpu
def test_sharded_problem_emulated_two_ranks_bitwise():
    """Two partitions of one node set on one GPU (no process group): stencils,
    weights, the exchanged apply and the row-partitioned heat loop equal the
    unsharded run bitwise."""
    import paper_1912_13282_b200 as mf
    from paper_1912_13282_b200 import _lib
    from paper_1912_13282_b200.parallel import ShardedProblem

    rng = np.random.default_rng(4)
    N = 6000
    pts = rng.uniform(0, 1, (N, 2))
    types = np.ones(N, dtype=np.int64)
    types[np.min(np.minimum(pts, 1 - pts), axis=1) < 0.02] = -1
    nodes = mf.NodeSet(pts, types)
    eng = mf.RbfFd(mf.Polyharmonic(3), degree=2, scale="support", solver="lu")
    full = mf.compute_weights(mf.find_closest_stencils(nodes, 15), eng, ["laplacian"])
    u = rng.standard_normal(N)
    y_ref = full.apply_all("laplacian", u)
    shards = [ShardedProblem(nodes, 15, eng, ["laplacian"], part=RowPartition(N, 2, r)) for r in range(2)]
    u_d = _lib.to_device(u, torch.float64)
    ys = [sh.operator("laplacian")._local(u_d).cpu().numpy() for sh in shards]
    assert np.array_equal(np.concatenate(ys), y_ref)
    # heat: 5 steps, the exchange done by hand between the two partitions
    dt = 1e-6
    interior = torch.from_numpy((types > 0).astype(np.uint8)).cuda()
    dirichlet = torch.from_numpy((types == -1).astype(np.uint8)).cuda()
    g = torch.zeros(N, dtype=torch.float64, device="cuda")
    u0 = np.exp(-50 * np.sum((pts - 0.5) ** 2, axis=1))
    u0[types == -1] = 0.0
    ref = mf.run_heat_explicit(nodes, full, dt=dt, steps=5, dirichlet={-1: 0.0}, initial=u0)
    cur = _lib.to_device(u0, torch.float64)
    lib = _lib.load()
    for _ in range(5):
        nxt = torch.empty_like(cur)
        for sh in shards:
            lo, hi = sh.part.lo, sh.part.hi
            lap = sh.operator("laplacian")._local(cur)
            _lib.check(lib.mf_heat_rows(lap.data_ptr(), cur[lo:].data_ptr(), interior[lo:].data_ptr(),
                                        dirichlet[lo:].data_ptr(), g[lo:].data_ptr(), None, dt, 1.0, hi - lo,
                                        nxt[lo:].data_ptr(), None, _lib.stream_ptr()), "mf_heat_rows")
        cur = nxt
    assert np.array_equal(cur.cpu().numpy(), ref)
