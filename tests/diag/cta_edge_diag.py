"""Diagnostic (GPU box): large-stencil (n=70, deg 4) degenerate cloud, per mode."""
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

pts = _cloud(seed=5, near_offset=float(sys.argv[1]) if len(sys.argv) > 1 else 2e-3, patch=2)
N = pts.shape[0]
spec = ["laplacian", "gradient"]
st, _ = oracle.knn(pts, 70)
ref, fail, _ = oracle.phs_weights(pts, np.arange(N), st, spec, degree=4)
ok = fail == 0
args = (torch.from_numpy(pts).cuda(), torch.arange(N, dtype=torch.int64, device="cuda"),
        torch.from_numpy(st.astype(np.int32)).cuda())
for mode in ("hybrid", "replay", "fast"):
    eng = mf.RbfFd(mf.Polyharmonic(3), degree=4, scale="support", solver="lu", mode=mode)
    out, status, ff, nrep = phs_weights_device(*args, eng, expand_families(spec, 3), 3)
    got = out.cpu().numpy()
    err = np.zeros(N)
    for f in range(got.shape[1]):
        e = np.zeros(N)
        e[ok] = np.max(np.abs(got[ok, f] - ref[ok, f]), axis=1) / np.max(np.abs(ref[ok, f]), axis=1)
        err = np.maximum(err, e)
    bad = np.flatnonzero(err > 1e-9)
    print(mode, "replayed", int(nrep.item()), "bad", bad.size, bad[:10], "max", err.max())
    for b in bad[:3]:
        P = pts[st[b]]
        dd = np.sqrt(((P[:, None] - P[None]) ** 2).sum(-1)) + np.eye(70)
        print("   row", b, "err", err[b], "minsep/radius", dd.min() / np.sqrt(((P - P[0]) ** 2).sum(1)).max(),
              "max|w|", np.abs(ref[b]).max())
