"""Shape-solve time for shapes around the BASELINE ones (which kernel serves
each (d, n, degree, families) and how fast): prints one JSON line per case."""
import json
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1912_13282_b200 as mf  # noqa: E402
from paper_1912_13282_b200.stencils import knn_device  # noqa: E402
from paper_1912_13282_b200.storage import expand_families, phs_weights_device  # noqa: E402

CASES = [(3, 35, 2, ["laplacian"]), (3, 35, 2, ["laplacian", "gradient"]), (2, 15, 2, ["laplacian"]),
         (2, 15, 2, ["laplacian", "gradient"]), (2, 25, 2, ["laplacian", "gradient"]), (2, 13, 2, ["laplacian"]),
         (2, 21, 3, ["laplacian"]), (3, 30, 2, ["laplacian"]), (3, 40, 2, ["laplacian"]), (3, 45, 3, ["laplacian"]),
         (2, 12, 2, ["laplacian"]), (3, 36, 2, ["laplacian"])]
M = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
for d, n, deg, fams in CASES:
    pts = np.random.default_rng(0).uniform(0, 1, (M, d))
    nodes = mf.NodeSet(pts, np.ones(M, dtype=np.int64))
    idx = torch.arange(M, dtype=torch.int64, device="cuda")
    st, _ = knn_device(nodes, n, idx, idx)
    eng = mf.RbfFd(mf.Polyharmonic(3), degree=deg, scale="support", solver="lu")
    fm = expand_families(fams, d)
    pos = nodes.positions_device()
    ts = []
    for r in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out, status, ff, nrep = phs_weights_device(pos, idx, st, eng, fm, d)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    l = len(mf.graded_lex_exponents(d, deg))
    s = n + l
    F = (2 / 3) * s ** 3 + 2 * len(fm) * s * s
    t = min(ts)
    print(json.dumps({"d": d, "n": n, "deg": deg, "nf": len(fm), "ms": round(t, 3),
                      "Mst_per_s": round(M / t / 1e3, 2), "tflops": round(M * F / t / 1e9, 2),
                      "replayed": int(nrep.item())}), flush=True)
