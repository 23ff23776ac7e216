"""C3 apply-plan build (Morton order + ELL structure and values) timed alone.
Usage: python tools/plan_only.py   (MF_PLAN_BUILD selects the ELL build kernel)"""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1912_13282_b200 as mf  # noqa: E402
from bench import c3_positions  # noqa: E402

N, n = 1_000_000, 35
pts = c3_positions(N, 0)
nodes = mf.find_closest_stencils(mf.NodeSet(pts, np.ones(N, dtype=np.int64)), n)
store = mf.compute_weights(nodes, mf.RbfFd(mf.Polyharmonic(3), degree=2, scale="support", solver="lu"), ["laplacian"])
mat = store.matrix("laplacian")
data = mat.data_device
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts, ref = [], None
for r in range(8):
    mat._s._plans.clear()
    flush.fill_(1)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    val = mat._s.plan_values(data, True)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e) * 1e3)
    idx = mat._s._plans[True][2]
    h = (int(torch.sum(idx.long())), float(torch.sum(val)))
    ref = ref or h
    assert h == ref
print(f"plan build (order + ELL) median {np.median(ts[2:]):.1f} us min {min(ts[2:]):.1f} us checksum {ref}")
