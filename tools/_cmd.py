import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1912_13282_b200 as mf
from paper_1912_13282_b200 import workloads
from paper_1912_13282_b200.stencils import knn_device
from paper_1912_13282_b200.storage import expand_families, phs_weights_device
rng = np.random.default_rng(3)
p = rng.uniform(-1, 1, (120_000, 3)); p = p[np.sum(p*p, 1) <= 1][:50_000]
N = len(p)
nodes = mf.NodeSet(p, np.ones(N, dtype=np.int64)); pos_d = nodes.positions_device()
idx_d = torch.arange(N, dtype=torch.int64, device="cuda")
st, _ = knn_device(nodes, 70, idx_d, idx_d)
eng = mf.RbfFd(mf.Polyharmonic(3), degree=4, scale="support", solver="lu")
fams = expand_families(["laplacian", "gradient"], 3)
full, status, ff, nrep = phs_weights_device(pos_d, idx_d, st, eng, fams, 3)
print("full", N, "replayed", int(nrep.item()))
bad = 0
for m in [1, 2, 3, 5, 147, 148, 149, 295, 296, 297, 593, 2367, 2368, 2369, 4737, 9999]:
    for off in (0, 12345):
        rows = idx_d[off:off + m].contiguous()
        out, s2, f2, n2 = phs_weights_device(pos_d, rows, st[off:off + m].contiguous(), eng, fams, 3)
        same = torch.equal(out, full[off:off + m])
        if not same:
            bad += 1
            print("MISMATCH m", m, "off", off, float((out - full[off:off+m]).abs().max()))
print("batch-size independence:", "ok" if bad == 0 else f"{bad} mismatches")
