"""Diagnostic (GPU box): dump FAST-mode error vs estimator features for C4.

TEST INFRASTRUCTURE: writes gpurun_out/c4_diag.npz for offline analysis of the
HYBRID re-solve criterion.  Not part of the product path.
"""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
import oracle  # noqa: E402

import paper_1912_13282_b200 as mf  # noqa: E402
from paper_1912_13282_b200 import workloads  # noqa: E402
from paper_1912_13282_b200.storage import expand_families, phs_weights_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
w = workloads.make(name)
N = w.N
nodes = mf.find_closest_stencils(mf.NodeSet(w.positions, w.types), w.n)
st_d = nodes.stencil_matrix_device(np.arange(N))
eng = mf.RbfFd(mf.Polyharmonic(3), degree=w.degree, scale="support", solver="lu", mode="fast")
fams = expand_families(w.families, w.dim)
kappa = torch.empty(4 * N, dtype=torch.float64, device="cuda")
out, status, ff, _ = phs_weights_device(nodes.positions_device(), torch.arange(N, device="cuda"), st_d, eng,
                                        fams, w.dim, kappa=kappa)
fast = out.cpu().numpy()
st = st_d.cpu().numpy()
ref, fail, _ = oracle.phs_weights(w.positions, np.arange(N), st, w.families, degree=w.degree,
                                  threads=os.cpu_count())
err = np.zeros(N)
for f in range(ref.shape[1]):
    den = np.max(np.abs(ref[:, f, :]), axis=1)
    err = np.maximum(err, np.max(np.abs(fast[:, f, :] - ref[:, f, :]), axis=1) / den)
P = w.positions[st]  # (N, n, d)
loc = P - P[:, :1, :]
scale = np.sqrt(np.max(np.einsum("nkd,nkd->nk", loc, loc), axis=1))
dmin = np.full(N, np.inf)
for i in range(w.n):
    for j in range(i + 1, w.n):
        dd = P[:, i, :] - P[:, j, :]
        dmin = np.minimum(dmin, np.sqrt(np.einsum("nd,nd->n", dd, dd)))
wmax = np.max(np.abs(ref[:, -1, :]), axis=1)
np.savez_compressed(os.path.join(REPO, "gpurun_out", f"{name.lower()}_diag.npz"), err=err,
                    diag=kappa.cpu().numpy().reshape(N, 4), dmin_rel=dmin / scale, wmax=wmax)
print("saved", err.max())
