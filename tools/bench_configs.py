"""Stage timings of the B200 path on all five BASELINE.json configurations.

Runs each config through the public API (inputs resident after the first
H2D), times every stage with CUDA events (best of three passes after one
warm-up pass), and prints one JSON line per config.  C4 also times the 1000-step stable heat loop
(dt = 0.1 h_min^2, SURVEY.md §8d variant 4b).  Not the driver's bench
(bench.py is); this is the per-config table quoted in DESIGN.md.

Usage: python tools/bench_configs.py [C1 C2 C3 C4 C5]   (one config per process gives every config the
same caching-allocator state: `for c in C1 C2 C3 C4 C5; do python tools/bench_configs.py $c; done`)
"""

from __future__ import annotations

import json
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


def timed(fn):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    out = fn()
    e.record()
    torch.cuda.synchronize()
    return out, s.elapsed_time(e)


def run(name):
    w = workloads.make(name)
    N, n, d = w.N, w.n, w.dim
    nodes = mf.NodeSet(w.positions, w.types)
    pos_d = nodes.positions_device()
    idx_d = torch.arange(N, dtype=torch.int64, device="cuda")
    eng = mf.RbfFd(mf.Polyharmonic(3), degree=w.degree, scale="support", solver="lu", mode="hybrid")
    fams = expand_families(w.families, d)
    u_d = torch.from_numpy(np.ascontiguousarray(w.field)).cuda()
    rec = {"config": name, "N": N, "n": n, "families": list(fams)}
    best = {}
    for rep in range(4):  # warm-up pass, then the best of three measured passes per stage
        (st, _), t_knn = timed(lambda: knn_device(nodes, n, idx_d, idx_d))
        (out, status, ff, nrep), t_phs = timed(lambda: phs_weights_device(pos_d, idx_d, st, eng, fams, d))
        vals = {k: out[:, f, :].contiguous() for f, k in enumerate(fams)}
        store = mf.WeightStore(N, np.arange(N), st, vals, n, rows_d=idx_d, positions_d=pos_d)
        # canonical CSR + the Morton-row apply plan a single apply reads (plan_direct)
        mats, t_csr = timed(lambda: [store.matrix(k).plan_direct() for k in fams])
        y, t_apply = timed(lambda: [store.matrix(k).apply_device(u_d) for k in fams])
        if rep:
            for k, t in (("knn", t_knn), ("phs", t_phs), ("csr", t_csr), ("apply", t_apply)):
                best[k] = min(best.get(k, t), t)
    t_knn, t_phs, t_csr, t_apply = best["knn"], best["phs"], best["csr"], best["apply"]
    s = n + len(mf.graded_lex_exponents(d, w.degree))
    r = len(fams)
    F = (2.0 / 3.0) * s**3 + 2.0 * r * s * s
    nnz = N * n
    b_apply = nnz * (8 * r + 4) + N * 8 + r * N * 8 + (N + 1) * 4
    rec.update(knn_ms=t_knn, shape_ms=t_phs, csr_plan_ms=t_csr, apply_ms=t_apply,
               shapes_per_s=N / (t_phs * 1e-3), shape_tflops=N * F / (t_phs * 1e-3) / 1e12,
               apply_gbs=b_apply / (t_apply * 1e-3) / 1e9, replayed=int(nrep.item()),
               failed=int(ff.item()) != 0x7F7F7F7F7F7F7F7F)
    if name == "C4":
        stn = st.cpu().numpy()
        dd = w.positions[stn[:, 1]] - w.positions
        hmin = float(np.sqrt(np.min(np.einsum("ij,ij->i", dd, dd))))
        dt = 0.1 * hmin * hmin
        nodes2 = nodes._with_device_stencils(np.arange(N), st)
        mf.run_heat_explicit(nodes2, store, dt=dt, steps=5, dirichlet={-1: 0.0}, initial=w.field)
        _, t_heat = timed(lambda: mf.run_heat_explicit(nodes2, store, dt=dt, steps=1000, dirichlet={-1: 0.0},
                                                       initial=w.field, return_device=True))
        b_step = nnz * 12 + N * 8 + N * 8 + (N + 1) * 4 + N
        rec.update(heat_1000_steps_ms=t_heat, heat_step_gbs=1000 * b_step / (t_heat * 1e-3) / 1e9, dt=dt)
    return rec


if __name__ == "__main__":
    names = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
    torch.cuda.set_device(0)
    mf._lib.load()
    _prime = torch.empty(16 << 30, dtype=torch.uint8, device="cuda")  # caching-allocator segment
    del _prime
    for nm in names:
        print(json.dumps(run(nm)), flush=True)
        torch.cuda.empty_cache()
