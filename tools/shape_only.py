"""Run only the shape solve of one BASELINE config (for ncu captures of the
shape kernels).  Usage: python tools/shape_only.py [C3] [mode] [reps] [rows]
(rows: solve only the first `rows` stencils)."""

import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_1912_13282_b200 as mf  # noqa: E402
from paper_1912_13282_b200 import workloads  # noqa: E402
from paper_1912_13282_b200.stencils import knn_device  # noqa: E402
from paper_1912_13282_b200.storage import expand_families, phs_weights_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
mode = sys.argv[2] if len(sys.argv) > 2 else "hybrid"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
nrows = int(sys.argv[4]) if len(sys.argv) > 4 else 0
w = workloads.make(name)
nodes = mf.NodeSet(w.positions, w.types)
idx_d = torch.arange(w.N, dtype=torch.int64, device="cuda")
st, _ = knn_device(nodes, w.n, idx_d, idx_d)
eng = mf.RbfFd(mf.Polyharmonic(3), degree=w.degree, scale="support", solver="lu", mode=mode)
fams = expand_families(w.families, w.dim)
pos_d = nodes.positions_device()
if nrows:
    idx_d = idx_d[:nrows].contiguous()
    st = st[:nrows].contiguous()
for r in range(reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    out, status, ff, nrep = phs_weights_device(pos_d, idx_d, st, eng, fams, w.dim)
    e.record()
    torch.cuda.synchronize()
    print(f"{name} {mode} rep {r}: {s.elapsed_time(e):.3f} ms, replayed {int(nrep.item())}", flush=True)
print("checksum", float(out.double().abs().sum().item()), int(np.count_nonzero(status.cpu().numpy())))
