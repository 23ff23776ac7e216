"""Full-size parity of the CUDA path against the pinned oracle (BASELINE configs).

The oracle is bit-identical to the reference (tests/test_oracle_pins.py), so
at full size it stands in for the reference: stencils bitwise, weights within
1e-9 normwise per stencil and family, canonical CSR structure bitwise, and
the explicit apply bitwise given the same CSR -- for every family.  C4 is
also run on three more node-set seeds.  Stencils whose closest node pair is
nearer than 1e-3 of the stencil radius may exceed 1e-9 up to the reference's
own numba-vs-numpy spread (3.9e-9); they are listed in the
record.  C5 (4M nodes): stencils bitwise for
all 4M targets, canonical CSR and apply bitwise for all four families over
all 4M rows, weights against the oracle on a strided 20k-row subset (the
oracle's shape solve needs minutes for all 4M; the builder's full-C5 weight
run is profiles/r01_c5_full_parity.txt).  The worst error and the 99th
percentile per configuration and family are written to
gpurun_out/full_parity.json (committed as profiles/r02_full_parity.json).
"""

import json
import os

import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = os.cpu_count() or 1
RECORD = {}


def record(name, worst):
    RECORD[name] = {k: {"max": v[0], "p99": v[1]} for k, v in worst.items()}
    RECORD["_excused_near_coincident"] = EXCUSED
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "full_parity.json"), "w") as fh:
        json.dump(RECORD, fh, indent=1, sort_keys=True)


def normwise(w, ref):
    den = np.max(np.abs(ref), axis=1)
    return np.max(np.abs(w - ref), axis=1) / np.where(den > 0, den, 1.0)


def run_config(name, mode, rows_stride=1, n_rows=None, **kw):
    import paper_1912_13282_b200 as mf
    from paper_1912_13282_b200 import workloads

    w = workloads.make(name, **kw)
    N = w.N
    tg = np.arange(0, N, rows_stride, dtype=np.int64)[:n_rows]
    nodes = mf.find_closest_stencils(mf.NodeSet(w.positions, w.types), w.n, for_which=tg)
    st = nodes.stencil_matrix_device(tg).cpu().numpy()
    ref_st, nstr = oracle.knn(w.positions, w.n, tg, threads=THREADS)
    assert np.array_equal(st, ref_st), f"{name}: stencils differ"
    eng = mf.RbfFd(mf.Polyharmonic(3), degree=w.degree, scale="support", solver="lu", mode=mode)
    store = mf.compute_weights(nodes, eng, w.families, for_which=tg)
    ref_w, fail, keys = oracle.phs_weights(w.positions, tg, ref_st, w.families, degree=w.degree,
                                           threads=THREADS)
    assert not fail.any()
    worst = {}
    for f, key in enumerate(keys):
        err = normwise(store.values[key].reshape(-1, w.n), ref_w[:, f, :])
        worst[key] = (float(err.max()), float(np.percentile(err, 99)))
        check_bar(w.positions, ref_st, err, (name, key))
    return w, tg, store, ref_st, worst


# the reference's own numba and numpy backends differ by up to 3.9e-9 on C4
# (SURVEY §8c): below a node separation of 1e-3 of the stencil radius the
# weights' rounding noise exceeds 1e-9 and no implementation without glibc's
# pow tables can reproduce it ("Limit of the re-solve")
NOISE_FLOOR = 3.9e-9
MIN_SEP = 1e-3
EXCUSED = {}


def check_bar(pos, st, err, label):
    """1e-9 for every stencil; stencils whose closest node pair is nearer than
    MIN_SEP * radius may reach the reference's own backend spread."""
    over = np.flatnonzero(err > 1e-9)
    for r in over:
        P = pos[st[r]]
        rad = np.max(np.linalg.norm(P - P[0], axis=1))
        dd = np.linalg.norm(P[:, None] - P[None], axis=2)
        dd[np.eye(P.shape[0], dtype=bool)] = np.inf
        sep = float(dd.min() / rad)
        assert sep < MIN_SEP and err[r] <= NOISE_FLOOR, (label, int(r), float(err[r]), sep)
        EXCUSED.setdefault(str(label), []).append({"row": int(r), "err": float(err[r]), "minsep_over_radius": sep})


def check_csr_apply(w, tg, store, st):
    """canonical CSR + apply of every family, bitwise vs the oracle on the same weights"""
    u = w.field if w.field is not None else np.random.default_rng(1).standard_normal(w.N)
    for key in store.families:
        mat = store.matrix(key)
        ip, ix, da = oracle.csr_canonical(tg, st, store.values[key].reshape(-1, w.n), w.N)
        assert np.array_equal(mat.indptr, ip) and np.array_equal(mat.indices, ix), key
        assert np.array_equal(mat.data, da), key
        assert np.array_equal(store.apply_all(key, u), oracle.apply(ip, ix, da, u, threads=THREADS)), key


@pytest.mark.parametrize("name", ["C1", "C2", "C4", "C3"])
def test_full_config_hybrid(name):
    w, tg, store, st, worst = run_config(name, "hybrid")
    record(name, worst)
    check_csr_apply(w, tg, store, st)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_c4_hybrid_more_seeds(seed):
    _, _, _, _, worst = run_config("C4", "hybrid", seed=seed)
    record(f"C4_seed{seed}", worst)


def test_full_c3_replay_mode():
    _, _, _, _, worst = run_config("C3", "replay")
    record("C3_replay", worst)
    assert worst["laplacian"][0] <= 1e-11


def test_c5_full_structure_and_strided_weights():
    """C5 at full size: stencils of all 4M targets bitwise, every family's CSR and
    apply bitwise over all 4M rows; weights vs the oracle on 20k strided rows."""
    import paper_1912_13282_b200 as mf
    from paper_1912_13282_b200 import workloads

    w = workloads.c5()
    nodes = mf.find_closest_stencils(mf.NodeSet(w.positions, w.types), w.n)
    tg = np.arange(w.N, dtype=np.int64)
    st = nodes.stencil_matrix_device(tg).cpu().numpy()
    ref_st, _ = oracle.knn(w.positions, w.n, tg, threads=THREADS)
    assert np.array_equal(st, ref_st), "C5: stencils differ"
    del ref_st
    eng = mf.RbfFd(mf.Polyharmonic(3), degree=w.degree, scale="support", solver="lu")
    store = mf.compute_weights(nodes, eng, w.families)
    sub = np.arange(0, w.N, 200, dtype=np.int64)[:20_000]
    ref_w, fail, keys = oracle.phs_weights(w.positions, sub, st[sub], w.families, degree=w.degree,
                                           threads=THREADS)
    assert not fail.any()
    worst = {}
    for f, key in enumerate(keys):
        err = normwise(store.values_device(key)[sub].cpu().numpy(), ref_w[:, f, :])
        worst[key] = (float(err.max()), float(np.percentile(err, 99)))
        check_bar(w.positions, st[sub], err, ("C5", key))
    record("C5_subset20k", worst)
    check_csr_apply(w, tg, store, st)


def test_c4_heat_steps_bitwise_vs_oracle():
    import paper_1912_13282_b200 as mf
    from paper_1912_13282_b200 import workloads

    w = workloads.c4()
    nodes = mf.find_closest_stencils(mf.NodeSet(w.positions, w.types), w.n)
    store = mf.compute_weights(nodes, mf.RbfFd(mf.Polyharmonic(3), 2, "support", "lu"), ["laplacian"])
    # stable variant 4b: dt = 0.1 h_min^2
    st = nodes.stencil_matrix_device(np.arange(w.N)).cpu().numpy()
    pts = w.positions
    d = pts[st[:, 1]] - pts
    hmin = float(np.sqrt(np.min(np.einsum("ij,ij->i", d, d))))
    dt = 0.1 * hmin * hmin
    steps = 20
    u = mf.run_heat_explicit(nodes, store, dt=dt, steps=steps, dirichlet={-1: 0.0}, initial=w.field)
    mat = store.matrix("laplacian")
    ref, bad, _ = oracle.heat_steps(mat.indptr, mat.indices, mat.data, w.types > 0, w.types == -1,
                                    np.zeros(w.N), w.field, dt=dt, steps=steps, threads=THREADS)
    assert bad == 0
    assert np.array_equal(u, ref)
    # literal dt = 0.1 h^2 diverges; the failure is reproduced at the same step
    with pytest.raises(mf.InstabilityError) as exc:
        mf.run_heat_explicit(nodes, store, dt=w.extra["dt_literal"], steps=50, dirichlet={-1: 0.0},
                             initial=w.field)
    _, bad, peak = oracle.heat_steps(mat.indptr, mat.indices, mat.data, w.types > 0, w.types == -1,
                                     np.zeros(w.N), w.field, dt=w.extra["dt_literal"], steps=50,
                                     threads=THREADS)
    assert exc.value.step == bad
    assert f"field peak {peak:.2e}" in str(exc.value)
