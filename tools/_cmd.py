import sys, os, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1912_13282_b200 as mf
from paper_1912_13282_b200 import workloads
from paper_1912_13282_b200.stencils import knn_device
from paper_1912_13282_b200.storage import expand_families, phs_weights_device
w = workloads.make(sys.argv[1] if len(sys.argv) > 1 else "C2")
N, n, d = w.N, w.n, w.dim
nodes = mf.NodeSet(w.positions, w.types); pos_d = nodes.positions_device()
idx_d = torch.arange(N, dtype=torch.int64, device="cuda")
eng = mf.RbfFd(mf.Polyharmonic(3), degree=w.degree, scale="support", solver="lu")
fams = expand_families(w.families, d)
u_d = torch.from_numpy(np.ascontiguousarray(w.field)).cuda()
def ev(): e = torch.cuda.Event(enable_timing=True); e.record(); return e
for rep in range(4):
    if rep == 3: torch.cuda.empty_cache()
    st, _ = knn_device(nodes, n, idx_d, idx_d)
    out, status, ff, nrep = phs_weights_device(pos_d, idx_d, st, eng, fams, d)
    vals = {k: out[:, f, :].contiguous() for f, k in enumerate(fams)}
    store = mf.WeightStore(N, np.arange(N), st, vals, n, rows_d=idx_d, positions_d=pos_d)
    torch.cuda.synchronize()
    marks = [("start", ev(), time.perf_counter())]
    for k in fams:
        m = store.matrix(k); marks.append((f"matrix {k}", ev(), time.perf_counter()))
        p = m.plan(True); marks.append((f"plan {k}", ev(), time.perf_counter()))
    for k in fams:
        y = store.matrix(k).apply_device(u_d); marks.append((f"apply1 {k}", ev(), time.perf_counter()))
    for k in fams:
        y = store.matrix(k).apply_device(u_d); marks.append((f"apply2 {k}", ev(), time.perf_counter()))
    torch.cuda.synchronize()
    if rep >= 2:
        print('rep', rep)
        for (na, ea, ha), (nb, eb, hb) in zip(marks[:-1], marks[1:]):
            print(f"  {nb:22s} gpu {ea.elapsed_time(eb):8.3f} ms   host {1e3*(hb-ha):8.3f} ms")
