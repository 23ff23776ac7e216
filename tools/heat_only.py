"""Time the C4 heat loop alone (run_heat_explicit on the resident store, stable dt).
Usage: python tools/heat_only.py [steps]"""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1912_13282_b200 as mf  # noqa: E402
from paper_1912_13282_b200 import workloads  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
w = workloads.make("C4")
nodes = mf.find_closest_stencils(mf.NodeSet(w.positions, w.types), w.n)
eng = mf.RbfFd(mf.Polyharmonic(3), degree=w.degree, scale="support", solver="lu")
store = mf.compute_weights(nodes, eng, w.families)
p = w.positions
u0 = np.exp(-50 * ((p[:, 0] - 0.5) ** 2 + (p[:, 1] - 0.5) ** 2))
dt = 4.9739636729043925e-14
for r in range(int(os.environ.get("REPS", "3"))):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    u = mf.run_heat_explicit(nodes, store, dt=dt, steps=steps, dirichlet={-1: 0.0}, initial=u0)
    e.record()
    torch.cuda.synchronize()
    print(f"heat {steps} steps: {s.elapsed_time(e):.2f} ms ({1e3 * s.elapsed_time(e) / steps:.1f} us/step)")
