"""Timings of the §8(f) rows on the GPU: implicit Poisson solve (assembly,
ILU(0) build, BiCGStab) on 2D/3D jittered grids, fill_interior on a 2D disk
with a hole, the general engine (qr) at C4 size.  One JSON line per case."""
import json
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1912_13282_b200 as mf  # noqa: E402
from paper_1912_13282_b200.drivers import assemble_poisson_system  # noqa: E402
from paper_1912_13282_b200.solve import Ilu0Preconditioner, SolverConfig, solve_sparse  # noqa: E402


def jittered(m, d, seed=0):
    h = 1.0 / m
    g = np.arange(h / 2, 1, h)
    P = np.stack(np.meshgrid(*([g] * d), indexing="ij"), -1).reshape(-1, d)
    P = P + np.random.default_rng(seed).uniform(-0.3 * h, 0.3 * h, P.shape)
    types = np.where(np.min(np.minimum(P, 1 - P), axis=1) < h, -1, 1).astype(np.int64)
    return P, types


def sync_t():
    torch.cuda.synchronize()
    return time.perf_counter()


which = sys.argv[1:] or ["implicit", "fill", "engine"]
if "implicit" in which:
    for m, d, n in [(500, 2, 15), (1000, 2, 15), (64, 3, 35)]:
        P, types = jittered(m, d)
        nodes = mf.find_closest_stencils(mf.NodeSet(P, types), n)
        store = mf.compute_weights(nodes, mf.RbfFd(mf.Polyharmonic(3), 2, "support", "lu"), ["laplacian"])
        f = lambda p: np.sin(3 * p[:, 0]) + 1.0
        for rep in range(2):
            t0 = sync_t()
            A, b = assemble_poisson_system(nodes, store, terms=[(-1.0, "laplacian")], rhs=f, dirichlet={-1: 0.0})
            t1 = sync_t()
            M = Ilu0Preconditioner(A)
            t2 = sync_t()
            res = solve_sparse(A, b, SolverConfig(), preconditioner=M)
            t3 = sync_t()
        print(json.dumps({"case": "implicit", "N": len(P), "d": d, "n": n, "assemble_ms": 1e3 * (t1 - t0),
                          "ilu0_ms": 1e3 * (t2 - t1), "colors": M.ncolors, "bicgstab_ms": 1e3 * (t3 - t2),
                          "iterations": res.iterations, "residual": res.residual}), flush=True)
if "fill" in which:
    for h in [0.01, 0.004, 0.002]:
        shape = mf.Ball([0.0, 0.0], 1.0) - mf.Ball([0.3, 0.1], 0.25, tag=-2)
        t = np.arange(0, 2 * np.pi, h)
        seeds = np.concatenate([np.stack([np.cos(t), np.sin(t)], 1),
                                np.stack([0.3 + 0.25 * np.cos(t[::4]), 0.1 + 0.25 * np.sin(t[::4])], 1)])
        nodes = mf.NodeSet(seeds, -np.ones(len(seeds), dtype=np.int64))
        t0 = sync_t()
        out = mf.fill_interior(nodes, shape, h)
        t1 = sync_t()
        print(json.dumps({"case": "fill", "h": h, "nodes": len(out), "ms": 1e3 * (t1 - t0),
                          "generations": len(out.fill_rounds), "max_rounds": max(out.fill_rounds)}), flush=True)
if "engine" in which:
    pts = np.random.default_rng(0).uniform(0, 1, (1_000_000, 2))
    nodes = mf.find_closest_stencils(mf.NodeSet(pts, np.ones(len(pts), dtype=np.int64)), 15)
    for eng in [mf.RbfFd(mf.Polyharmonic(3), 2), mf.RbfFd(mf.Polyharmonic(3), 2, solver="svd"),
                mf.WeightedLeastSquares(2)]:
        for rep in range(2):
            t0 = sync_t()
            st = mf.compute_weights(nodes, eng, ["laplacian", "gradient"])
            t1 = sync_t()
        print(json.dumps({"case": "engine", "engine": repr(eng), "N": len(pts), "ms": 1e3 * (t1 - t0)}), flush=True)
