import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1912_13282_b200 as mf
from paper_1912_13282_b200.stencils import knn_device
pts = np.random.default_rng(0).uniform(0, 1, (1_000_000, 3))
nodes = mf.NodeSet(pts, np.ones(len(pts), dtype=np.int64))
idx = np.arange(len(pts))
for _ in range(2):
    st, ns = knn_device(nodes, 35, idx, idx)
torch.cuda.synchronize()
t = time.perf_counter(); st, ns = knn_device(nodes, 35, idx, idx); torch.cuda.synchronize()
print("knn ms", 1e3 * (time.perf_counter() - t), "straddle", int(ns.item()))
