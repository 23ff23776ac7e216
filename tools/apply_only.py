"""C3 apply: CSR warp kernel (mf_apply) vs the Morton ELL plan (mf_plan_apply),
bitwise comparison and device times.  Usage: python tools/apply_only.py"""
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
u = torch.as_tensor(np.random.default_rng(1).standard_normal(N)).cuda()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=20):
    ts = []
    for _ in range(reps):
        flush.fill_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        y = fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return y, float(np.median(ts)), float(np.min(ts))


s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
mat.plan(True)
e.record()
torch.cuda.synchronize()
print(f"plan build {s.elapsed_time(e) * 1e3:.1f} us")
y1, m1, b1 = timed(lambda: mat.apply_csr_device(u))
y2, m2, b2 = timed(lambda: mat.apply_device(u))
print(f"csr apply  median {m1:.1f} us  min {b1:.1f} us")
print(f"plan apply median {m2:.1f} us  min {b2:.1f} us")
print("bitwise equal:", bool(torch.equal(y1.view(torch.int64), y2.view(torch.int64))))
