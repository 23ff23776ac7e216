"""Diagnostic (GPU box, ~5 min of host oracle): full C5 HYBRID weights vs the oracle."""
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
import oracle  # noqa: E402
import paper_1912_13282_b200 as mf  # noqa: E402
from paper_1912_13282_b200 import workloads  # noqa: E402
from paper_1912_13282_b200.storage import expand_families, phs_weights_device  # noqa: E402

w = workloads.make("C5")
N = w.N
nodes = mf.find_closest_stencils(mf.NodeSet(w.positions, w.types), w.n)
st_d = nodes.full_block_matrix()
eng = mf.RbfFd(mf.Polyharmonic(3), degree=w.degree, scale="support", solver="lu", mode="hybrid")
fams = expand_families(w.families, w.dim)
out, status, ff, nrep = phs_weights_device(nodes.positions_device(), torch.arange(N, device="cuda"), st_d, eng,
                                           fams, w.dim)
got = out.cpu().numpy()
st = st_d.cpu().numpy()
t = time.time()
ref, fail, _ = oracle.phs_weights(w.positions, np.arange(N), st, w.families, degree=w.degree,
                                  threads=os.cpu_count())
print("oracle s", time.time() - t, "fails", int(fail.sum()), "status mismatches",
      int(np.sum((status.cpu().numpy() != 0) != (fail != 0))), "replayed", int(nrep.item()))
err = np.zeros(N)
for f in range(ref.shape[1]):
    den = np.max(np.abs(ref[:, f, :]), axis=1)
    err = np.maximum(err, np.max(np.abs(got[:, f, :] - ref[:, f, :]), axis=1) / den)
print("max err", err.max(), "rows > 1e-9", int(np.sum(err > 1e-9)), "p99.99", np.quantile(err, 0.9999))
np.save(os.path.join(REPO, "gpurun_out", "c5_err.npy"), err)
