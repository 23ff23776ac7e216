import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1912_13282_b200 as mf
from paper_1912_13282_b200 import workloads
from paper_1912_13282_b200.stencils import knn_device
from paper_1912_13282_b200.storage import expand_families, phs_weights_device
w = workloads.make("C2"); N, n, d = w.N, w.n, w.dim
nodes = mf.NodeSet(w.positions, w.types); pos_d = nodes.positions_device()
idx_d = torch.arange(N, dtype=torch.int64, device="cuda")
eng = mf.RbfFd(mf.Polyharmonic(3), degree=2, scale="support", solver="lu")
fams = expand_families(w.families, d)
st, _ = knn_device(nodes, n, idx_d, idx_d)
out, *_ = phs_weights_device(pos_d, idx_d, st, eng, fams, d)
for rep in range(3):
    vals = {k: out[:, f, :].contiguous() for f, k in enumerate(fams)}
    store = mf.WeightStore(N, np.arange(N), st, vals, n, rows_d=idx_d, positions_d=pos_d)
    torch.cuda.synchronize()
    for k in fams:
        t = time.perf_counter(); m = store.matrix(k); torch.cuda.synchronize(); t1 = time.perf_counter()
        m.plan(True); torch.cuda.synchronize(); t2 = time.perf_counter()
        print(rep, k, f"matrix {1e3*(t1-t):.2f} ms plan {1e3*(t2-t1):.2f} ms")
