"""Time WeightStore.apply_families (one pass over the shared structure) on a
BASELINE config: python tools/apply_families_only.py [C5|C2|C3]."""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1912_13282_b200 as mf  # noqa: E402
from paper_1912_13282_b200 import workloads  # noqa: E402

w = workloads.make(sys.argv[1] if len(sys.argv) > 1 else "C5")
nodes = mf.find_closest_stencils(mf.NodeSet(w.positions, w.types), w.n)
store = mf.compute_weights(nodes, mf.RbfFd(mf.Polyharmonic(3), w.degree, "support", "lu"), w.families)
keys = store.families
u = torch.from_numpy(np.random.default_rng(1).standard_normal(w.N)).cuda()
ys = store.apply_families(keys, u)
ref = {k: store.apply_all(k, u) for k in keys}
assert all(torch.equal(ys[k], ref[k]) for k in keys), "apply_families differs from apply_all"
ts = []
for _ in range(6):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    store.apply_families(keys, u)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
r = len(keys)
B = w.N * w.n * (8 * r + 4) + w.N * 8 + r * w.N * 8 + (w.N + 1) * 4
print(f"{w.name} apply_families r={r}: " + " ".join(f"{t:.3f}" for t in ts) + f" ms; best {B / min(ts) / 1e6:.0f} GB/s")
