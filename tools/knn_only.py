"""Time the stencil selection alone (mf_knn through knn_device) on one BASELINE
config.  Usage: python tools/knn_only.py [C3] [reps]"""

import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_1912_13282_b200 as mf  # noqa: E402
from paper_1912_13282_b200 import workloads  # noqa: E402
from paper_1912_13282_b200.stencils import knn_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = workloads.make(name)
nodes = mf.NodeSet(w.positions, w.types)
idx_d = torch.arange(w.N, dtype=torch.int64, device="cuda")
ts = []
for r in range(reps + 1):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    st, _ = knn_device(nodes, w.n, idx_d, idx_d)
    e.record()
    torch.cuda.synchronize()
    if r:
        ts.append(s.elapsed_time(e))
print(f"{name} knn: best {min(ts):.3f} ms, mean {sum(ts) / len(ts):.3f} ms, checksum {int(st.long().sum().item())}")
