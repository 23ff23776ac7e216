"""Host-side cost of the public API with an explicit target block (the sharded
path's e2e): times NodeSet, find_closest_stencils(for_which=block),
compute_weights(for_which=block) and the apply, each synchronised."""
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1912_13282_b200 as mf  # noqa: E402

N = 1_000_000
pts = np.random.default_rng(0).uniform(0, 1, (N, 3))
u = np.random.default_rng(1).standard_normal(N)
eng = mf.RbfFd(mf.Polyharmonic(3), degree=2, scale="support", solver="lu")
for rep in range(3):
    t = [time.perf_counter()]
    nodes = mf.NodeSet(pts, np.ones(N, dtype=np.int64)); torch.cuda.synchronize(); t.append(time.perf_counter())
    tg = np.arange(0, N, dtype=np.int64)
    nd = mf.find_closest_stencils(nodes, 35, for_which=tg); torch.cuda.synchronize(); t.append(time.perf_counter())
    st = mf.compute_weights(nd, eng, ["laplacian"], for_which=tg); torch.cuda.synchronize(); t.append(time.perf_counter())
    y = st.apply_all("laplacian", u); torch.cuda.synchronize(); t.append(time.perf_counter())
    nd2 = mf.find_closest_stencils(nodes, 35); torch.cuda.synchronize(); t.append(time.perf_counter())
    st2 = mf.compute_weights(nd2, eng, ["laplacian"]); torch.cuda.synchronize(); t.append(time.perf_counter())
    print(rep, "nodeset %.1f knn(for_which) %.1f weights(for_which) %.1f apply %.1f | knn(all) %.1f weights(all) %.1f ms"
          % tuple(1e3 * np.diff(t)), flush=True)
