"""Diagnose HYBRID misses: stencils whose first-pass weights exceed a tolerance
against the oracle (C4 at several seeds): min node separation / radius, and
whether the REPLAY kernel alone meets the bar.  Test infrastructure (imports
the oracle)."""
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
import oracle  # noqa: E402
import paper_1912_13282_b200 as mf  # noqa: E402
from paper_1912_13282_b200 import workloads  # noqa: E402

out = {}
for seed in [int(s) for s in sys.argv[1:]] or [0, 1, 2, 3]:
    w = workloads.c4(seed=seed)
    nodes = mf.find_closest_stencils(mf.NodeSet(w.positions, w.types), w.n)
    tg = np.arange(w.N)
    st = nodes.stencil_matrix_device(tg).cpu().numpy()
    ref, fail, keys = oracle.phs_weights(w.positions, tg, st, w.families, degree=2, threads=os.cpu_count())
    res = {}
    for mode in ["hybrid", "replay"]:
        store = mf.compute_weights(nodes, mf.RbfFd(mf.Polyharmonic(3), 2, "support", "lu", mode=mode), w.families)
        wv = store.values["laplacian"].reshape(-1, w.n)
        err = np.max(np.abs(wv - ref[:, 0]), 1) / np.max(np.abs(ref[:, 0]), 1)
        res[mode] = err
    bad = np.argsort(res["hybrid"])[::-1][:12]
    rows = []
    for r in bad:
        P = w.positions[st[r]]
        c = P[0]
        rad = np.max(np.linalg.norm(P - c, axis=1))
        dd = np.linalg.norm(P[:, None] - P[None], axis=2) + np.eye(w.n) * 1e9
        rows.append({"row": int(r), "hybrid": float(res["hybrid"][r]), "replay": float(res["replay"][r]),
                     "minsep_over_radius": float(dd.min() / rad)})
    out[seed] = {"hybrid_max": float(res["hybrid"].max()), "replay_max": float(res["replay"].max()),
                 "n_hybrid_gt_1e-10": int((res["hybrid"] > 1e-10).sum()), "worst": rows}
    print(seed, json.dumps(out[seed], indent=1))
os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(REPO, "gpurun_out", "hybrid_diag.json"), "w"), indent=1)
