"""Host-side profile of the public-API (e2e) C3 step: stage wall times with a
synchronize after each stage, then a cProfile of one step.  Diagnostics only."""

import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

import paper_1912_13282_b200 as mf  # noqa: E402
from bench import c3_positions  # noqa: E402

N, n = 1_000_000, 35
pts = c3_positions(N, 0)
pts_pin = torch.empty((N, 3), dtype=torch.float64, pin_memory=True).numpy()
pts_pin[:] = pts
u_pin = torch.empty(N, dtype=torch.float64, pin_memory=True).numpy()
u_pin[:] = np.random.default_rng(1).standard_normal(N)
types = np.ones(N, dtype=np.int64)
eng = mf.RbfFd(mf.Polyharmonic(3), degree=2, scale="support", solver="lu", mode="hybrid")


def step(sync):
    marks = [time.perf_counter()]
    nodes = mf.NodeSet(pts_pin, types)
    nodes = mf.find_closest_stencils(nodes, n)
    if sync:
        torch.cuda.synchronize()
    marks.append(time.perf_counter())
    store = mf.compute_weights(nodes, eng, ["laplacian"])
    if sync:
        torch.cuda.synchronize()
    marks.append(time.perf_counter())
    y = store.apply_all("laplacian", u_pin)
    torch.cuda.synchronize()
    marks.append(time.perf_counter())
    return y, np.diff(marks) * 1e3


for _ in range(2):
    step(True)
for _ in range(2):
    _, ms = step(True)
    print("stages ms (knn, weights, apply_all):", np.round(ms, 2), "total", round(float(ms.sum()), 2))
t0 = time.perf_counter()
step(False)
print("unsynced step ms", round((time.perf_counter() - t0) * 1e3, 2))
pr = cProfile.Profile()
pr.enable()
step(False)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
