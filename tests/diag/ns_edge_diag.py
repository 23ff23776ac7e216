"""Diagnostic (GPU box): which degenerate-cloud stencils miss the parity bar, per mode."""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, os.path.join(REPO, "tests"))
import oracle  # noqa: E402
import paper_1912_13282_b200 as mf  # noqa: E402
from paper_1912_13282_b200.storage import expand_families, phs_weights_device  # noqa: E402
from test_ns_edge_cases import _cloud  # noqa: E402

pts = _cloud()
N = pts.shape[0]
st, _ = oracle.knn(pts, 35)
ref, fail, _ = oracle.phs_weights(pts, np.arange(N), st, ["laplacian"], degree=2)
pos_d = torch.from_numpy(pts).cuda()
rows_d = torch.arange(N, dtype=torch.int64, device="cuda")
st_d = torch.from_numpy(st.astype(np.int32)).cuda()
ok = fail == 0
for mode in ("hybrid", "fast", "replay"):
    eng = mf.RbfFd(mf.Polyharmonic(3), degree=2, scale="support", solver="lu", mode=mode)
    out, status, ff, nrep = phs_weights_device(pos_d, rows_d, st_d, eng, expand_families(["laplacian"], 3), 3)
    got = out.cpu().numpy()[:, 0, :]
    err = np.zeros(N)
    err[ok] = np.max(np.abs(got[ok] - ref[ok, 0]), axis=1) / np.max(np.abs(ref[ok, 0]), axis=1)
    bad = np.flatnonzero(err > 1e-9)
    print(mode, "replayed", int(nrep.item()), "status mismatches", int(np.sum((status.cpu().numpy() != 0) != (fail != 0))),
          "bad rows", bad.size, bad[:12], "max", err.max())
    if bad.size:
        P = pts[st[bad[0]]]
        d = np.sqrt(((P[:, None] - P[None]) ** 2).sum(-1)) + np.eye(35)
        print("   first bad row", bad[0], "min sep / radius", d.min() / np.sqrt(((P - P[0]) ** 2).sum(1)).max(),
              "ref max |w|", np.abs(ref[bad[0], 0]).max())
