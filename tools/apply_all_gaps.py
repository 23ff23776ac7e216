"""Where the time of WeightStore.apply_all goes on C3 (public API, pinned field):
CUDA-event and host marks between its sub-steps.  Usage: python tools/apply_all_gaps.py"""
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1912_13282_b200 as mf  # noqa: E402
from paper_1912_13282_b200 import _lib  # noqa: E402
from paper_1912_13282_b200.storage import _to_host  # noqa: E402
from bench import c3_positions  # noqa: E402

N, n = 1_000_000, 35
pts = c3_positions(N, 0)
u_pin = torch.empty(N, dtype=torch.float64, pin_memory=True).numpy()
u_pin[:] = np.random.default_rng(1).standard_normal(N)
eng = mf.RbfFd(mf.Polyharmonic(3), degree=2, scale="support", solver="lu")
for rep in range(4):
    nodes = mf.find_closest_stencils(mf.NodeSet(pts, np.ones(N, dtype=np.int64)), n)
    store = mf.compute_weights(nodes, eng, ["laplacian"])
    torch.cuda.synchronize()
    marks = []

    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append((name, e, time.perf_counter()))

    mark("start")
    u_d, ready = _lib.to_device_async(u_pin, torch.float64)
    mark("h2d_enqueue")
    mat = store.matrix("laplacian")
    mark("csr")
    mat.plan(True)
    mark("plan")
    torch.cuda.current_stream().wait_event(ready)
    mark("wait_h2d")
    y = mat.apply_device(u_d)
    mark("apply")
    mat._s.check()
    mark("check")
    yh = _to_host(y)
    mark("d2h")
    torch.cuda.synchronize()
    if rep >= 2:
        print(f"rep {rep}: total host {1e3 * (marks[-1][2] - marks[0][2]):.3f} ms")
        for (na, ea, ha), (nb, eb, hb) in zip(marks[:-1], marks[1:]):
            print(f"  {nb:12s} gpu {ea.elapsed_time(eb):7.3f} ms   host {1e3 * (hb - ha):7.3f} ms")
