import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import paper_1912_13282_b200 as mf
from bench import c3_positions
N, n = 1_000_000, 35
pts = c3_positions(N, 0)
pts_pin = torch.empty((N, 3), dtype=torch.float64, pin_memory=True).numpy(); pts_pin[:] = pts
u_pin = torch.empty(N, dtype=torch.float64, pin_memory=True).numpy(); u_pin[:] = np.random.default_rng(1).standard_normal(N)
types = np.ones(N, dtype=np.int64)
eng = mf.RbfFd(mf.Polyharmonic(3), degree=2, scale="support", solver="lu", mode="hybrid")
_prime = torch.empty(8 << 30, dtype=torch.uint8, device="cuda"); del _prime
def step(rec):
    ev = []
    def mark(name):
        e = torch.cuda.Event(enable_timing=True); e.record(); ev.append((name, e, time.perf_counter()))
    mark("start")
    nodes = mf.NodeSet(pts_pin, types); mark("nodeset")
    nodes = mf.find_closest_stencils(nodes, n); mark("knn")
    store = mf.compute_weights(nodes, eng, ["laplacian"]); mark("weights")
    y = store.apply_all("laplacian", u_pin); mark("apply_all")
    torch.cuda.synchronize()
    return ev
for _ in range(3): step(False)
for _ in range(2):
    t0 = time.perf_counter()
    ev = step(True)
    t1 = time.perf_counter()
    print(f"total wall {1e3*(t1-t0):.2f} ms")
    for (na, ea, ha), (nb, eb, hb) in zip(ev[:-1], ev[1:]):
        print(f"  {nb:10s} gpu {ea.elapsed_time(eb):7.3f} ms   host {1e3*(hb-ha):7.3f} ms")
