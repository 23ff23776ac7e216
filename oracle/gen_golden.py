"""Generate tests/golden/*.npz from the LIVE reference (run in the build container).

TEST INFRASTRUCTURE.  Usage (the reference tree is read-only, numba needs a
writable cache):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python oracle/gen_golden.py

Every fixture is produced by calling the reference's own public API
(``find_closest_stencils``, ``compute_weights`` with the batched
``RbfFd(Polyharmonic(k), solver="lu")`` engine, ``WeightStore.matrix``,
``apply_all``, ``run_heat_explicit``) on seeded synthetic inputs.  The
environment versions are stored alongside (``meta`` entries).  The CPU tests
then pin the C oracle to these vectors bit-for-bit, and the GPU tests compare
the CUDA path with both.
"""

from __future__ import annotations

import os
import platform
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

import meshfree  # noqa: E402  (the reference, from PYTHONPATH)
import numba  # noqa: E402
import scipy  # noqa: E402
from meshfree import (  # noqa: E402
    InstabilityError,
    NodeSet,
    Polyharmonic,
    RbfFd,
    WeightError,
    compute_weights,
    find_closest_stencils,
)
from meshfree.drivers import run_heat_explicit  # noqa: E402

from paper_1912_13282_b200 import workloads  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")


def meta():
    return dict(
        meta_numpy=np.array(np.__version__),
        meta_scipy=np.array(scipy.__version__),
        meta_numba=np.array(numba.__version__),
        meta_python=np.array(platform.python_version()),
        meta_libc=np.array(" ".join(platform.libc_ver())),
        meta_backend=np.array(meshfree.backend_name()),
    )


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays, **meta())
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def cloud(n, d, seed, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, (n, d))


# -- kNN -------------------------------------------------------------------

def knn_cases():
    """Small clouds mirroring reference tests/test_stencils.py + edge cases."""
    cases = []

    def add(name, pts, n, types=None, for_which=None, search_among=None):
        N = pts.shape[0]
        types = np.ones(N, dtype=np.int64) if types is None else types
        nodes = NodeSet(pts, types)
        out = find_closest_stencils(nodes, n, for_which, search_among)
        tg = nodes.select(for_which)
        pool = nodes.select(search_among)
        st = np.stack([out.stencil(int(i)) for i in tg]) if tg.size else np.zeros((0, n), np.int64)
        cases.append(dict(name=name, pts=pts, types=types, n=n, targets=tg, pool=pool, stencils=st))

    add("random2d_60_n7", cloud(60, 2, 0), 7)
    add("random3d_40_n5", cloud(40, 3, 3), 5)
    g = np.stack(np.meshgrid(np.arange(5.0), np.arange(5.0), indexing="ij"), axis=-1).reshape(-1, 2)
    add("grid5x5_ties_n4", g, 4)
    g3 = np.stack(np.meshgrid(np.arange(4.0), np.arange(4.0), np.arange(4.0), indexing="ij"), axis=-1).reshape(-1, 3)
    add("grid4x4x4_ties_n9", g3, 9)
    add("grid4x4x4_ties_n27", g3, 27)
    types = np.ones(30, dtype=np.int64)
    types[:6] = -1
    add("for_which_interior", cloud(30, 2, 1), 4, types=types.copy(), for_which="interior")
    add("search_among_interior", cloud(30, 2, 2), 4, types=types.copy(), search_among="interior")
    idx = np.array([17, 3, 25, 3, 9], dtype=np.int64)
    add("explicit_targets_unsorted", cloud(30, 3, 4), 6, for_which=idx, search_among=np.arange(5, 30))
    for s in range(24):
        rng = np.random.default_rng(1000 + s)
        d = 2 + (s % 2)
        n = 1 + (s * 5) % 12
        add(f"prop_seed{s}_d{d}_n{n}", rng.uniform(-1, 1, (16, d)), n)
    # coincident nodes: self cannot lead by distance alone
    dup = cloud(20, 2, 7)
    dup[5] = dup[3]
    dup[6] = dup[3]
    dup[11] = dup[3]
    add("duplicates_n3", dup, 3)
    add("duplicates_n6", dup, 6)
    add("line1d_n5", np.sort(cloud(25, 1, 8), axis=0), 5)
    add("pool_equals_n", cloud(12, 2, 9), 12)
    add("single_n1", cloud(15, 3, 10), 1)
    return cases


def dump_knn():
    cases = knn_cases()
    arrs = {}
    for i, c in enumerate(cases):
        for k, v in c.items():
            arrs[f"c{i}_{k}"] = np.asarray(v)
    arrs["count"] = np.array(len(cases))
    save("knn_small.npz", **arrs)


def config_subset(w, n_targets, stride=1):
    nodes = NodeSet(w.positions, w.types)
    tg = np.arange(0, w.N, stride, dtype=np.int64)[:n_targets]
    nodes = find_closest_stencils(nodes, w.n, for_which=tg)
    st = np.stack([nodes.stencil(int(i)) for i in tg])
    return nodes, tg, st


def dump_configs():
    """Per-config stencils + weights for a prefix/strided subset of targets."""
    specs = [("C1", workloads.c1(), 2000, 1), ("C2", workloads.c2(), 400, 499),
             ("C3", workloads.c3(), 300, 3331), ("C4", workloads.c4(), 400, 2477),
             ("C5", workloads.c5(), 60, 66_667)]
    for name, w, cnt, stride in specs:
        nodes, tg, st = config_subset(w, cnt, stride)
        eng = RbfFd(Polyharmonic(3), degree=w.degree, scale="support", solver="lu")
        store = compute_weights(nodes, eng, w.families, for_which=tg)
        arrs = dict(targets=tg, stencils=st.astype(np.int32), n=np.array(w.n),
                    degree=np.array(w.degree), families=np.array(store.families))
        for f in store.families:
            arrs[f"w_{f}"] = store.values[f].reshape(len(tg), w.n)
        save(f"config_{name}.npz", **arrs)


# -- weight variants ---------------------------------------------------------

def dump_weight_variants():
    """Engine/family variants through the batched path (storage.py:310-322)."""
    arrs = {}
    variants = [
        # name, d, N, n, k, degree, scale, families
        ("k3_deg2_support_2d", 2, 400, 12, 3, 2, "support", ["laplacian", "gradient", "hessian", "identity"]),
        ("k3_deg2_nearest_2d", 2, 400, 12, 3, 2, "nearest", ["laplacian", "gradient"]),
        ("k3_deg2_none_2d", 2, 400, 12, 3, 2, "none", ["laplacian"]),
        ("k5_deg2_support_3d", 3, 500, 20, 5, 2, "support", ["laplacian", "gradient", "hessian"]),
        ("k4_even_deg1_2d", 2, 300, 9, 4, 1, "support", ["laplacian", "d1_0"]),
        ("k3_nodeg_2d", 2, 300, 9, 3, -1, "support", ["laplacian", "identity"]),
        ("k3_deg3_3d", 3, 600, 30, 3, 3, "support", ["laplacian", "d2_0_2"]),
        ("k7_deg2_1d", 1, 100, 7, 7, 2, "nearest", ["laplacian", "d1_0", "d2_0_0"]),
        ("k3_deg2_3d_n45", 3, 500, 45, 3, 2, "support", ["laplacian", "gradient"]),
        ("k3_deg2_2d_n31", 2, 500, 31, 3, 2, "support", ["laplacian"]),
    ]
    arrs["names"] = np.array([v[0] for v in variants])
    for vi, (name, d, N, n, k, deg, scale, fams) in enumerate(variants):
        pts = cloud(N, d, 500 + vi, 0.0, 1.0)
        nodes = find_closest_stencils(NodeSet(pts, np.ones(N, dtype=np.int64)), n)
        eng = RbfFd(Polyharmonic(k), degree=deg, scale=scale, solver="lu")
        store = compute_weights(nodes, eng, fams)
        arrs[f"{name}_pts"] = pts
        arrs[f"{name}_stencils"] = nodes.stencil_matrix().astype(np.int32)
        arrs[f"{name}_params"] = np.array([d, N, n, k, deg])
        arrs[f"{name}_scale"] = np.array(scale)
        arrs[f"{name}_families"] = np.array(fams)
        arrs[f"{name}_keys"] = np.array(store.families)
        for f in store.families:
            arrs[f"{name}_w_{f}"] = store.values[f].reshape(N, n)
    save("weight_variants.npz", **arrs)


def dump_weight_errors():
    """Degenerate stencils: the lowest failing row's node id and message."""
    arrs = {}
    pts = cloud(50, 2, 21, 0.0, 1.0)
    # node 13 and its stencil collapse onto one point -> scale degenerate
    pts[[13, 30, 31, 32, 33]] = pts[13]
    nodes = NodeSet(pts, np.ones(50, dtype=np.int64))
    nodes = find_closest_stencils(nodes, 5, for_which=np.arange(13, 50))
    eng = RbfFd(Polyharmonic(3), degree=1, scale="support", solver="lu")
    try:
        compute_weights(nodes, eng, ["laplacian"], for_which=np.arange(13, 50))
        msg = ""
    except WeightError as exc:
        msg = str(exc)
    arrs["scale_pts"] = pts
    arrs["scale_msg"] = np.array(msg)
    # collinear stencil with a 2D degree-1 basis -> singular system
    pts2 = cloud(40, 2, 22, 0.0, 1.0)
    pts2[:8, 1] = 0.5
    pts2[:8, 0] = np.linspace(0.1, 0.2, 8)
    nodes2 = find_closest_stencils(NodeSet(pts2, np.ones(40, dtype=np.int64)), 4, for_which=np.arange(8))
    try:
        compute_weights(nodes2, eng, ["laplacian"], for_which=np.arange(8))
        msg2 = ""
    except WeightError as exc:
        msg2 = str(exc)
    arrs["singular_pts"] = pts2
    arrs["singular_msg"] = np.array(msg2)
    save("weight_errors.npz", **arrs)


# -- CSR, apply, heat ----------------------------------------------------------

def dump_csr_apply():
    arrs = {}
    pts = cloud(700, 2, 31, 0.0, 1.0)
    types = np.ones(700, dtype=np.int64)
    types[::7] = -1
    nodes = find_closest_stencils(NodeSet(pts, types), 12)
    eng = RbfFd(Polyharmonic(3), degree=2, scale="support", solver="lu")
    # only interior rows stored: boundary rows of the CSR stay empty
    store = compute_weights(nodes, eng, ["laplacian", "gradient"], for_which="interior")
    u = np.random.default_rng(5).standard_normal(700)
    arrs["pts"] = pts
    arrs["types"] = types
    arrs["rows"] = store.rows
    arrs["stencils"] = np.stack([nodes.stencil(int(i)) for i in store.rows]).astype(np.int32)
    arrs["u"] = u
    for f in store.families:
        m = store.matrix(f)
        arrs[f"{f}_indptr"] = m.indptr
        arrs[f"{f}_indices"] = m.indices
        arrs[f"{f}_data"] = m.data
        arrs[f"{f}_w"] = store.values[f]
        arrs[f"{f}_y"] = store.apply_all(f, u)
    save("csr_apply.npz", **arrs)


def dump_heat():
    arrs = {}
    N = 3000
    pts = cloud(N, 2, 41, 0.0, 1.0)
    h = 1.0 / np.sqrt(N)
    edge = np.minimum(np.minimum(pts[:, 0], pts[:, 1]), np.minimum(1 - pts[:, 0], 1 - pts[:, 1]))
    types = np.where(edge < h, -1, 1).astype(np.int64)
    nodes = find_closest_stencils(NodeSet(pts, types), 15)
    eng = RbfFd(Polyharmonic(3), degree=2, scale="support", solver="lu")
    store = compute_weights(nodes, eng, ["laplacian"])
    d = pts - 0.5
    u0 = np.exp(-50.0 * (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]))
    from scipy.spatial import cKDTree
    hmin = float(cKDTree(pts).query(pts, k=2)[0][:, 1].min())
    dt = 0.1 * hmin * hmin
    u = run_heat_explicit(nodes, store, dt=dt, steps=40, dirichlet={-1: 0.0}, initial=u0)
    arrs.update(pts=pts, types=types, u0=u0, dt=np.array(dt), steps=np.array(40), u_final=u,
                stencils=nodes.stencil_matrix().astype(np.int32), w=store.values["laplacian"].reshape(N, 15))
    # source + diffusivity + a Dirichlet value != 0
    u2 = run_heat_explicit(nodes, store, dt=dt, steps=25, diffusivity=0.7, source=lambda p, t: 2.0,
                           dirichlet={-1: 0.25}, initial=u0)
    arrs["u_final_src"] = u2
    # literal dt = 0.1 h^2 diverges: parity of the failure
    try:
        run_heat_explicit(nodes, store, dt=0.1 * h * h, steps=400, dirichlet={-1: 0.0}, initial=u0)
        arrs["unstable_msg"] = np.array("")
        arrs["unstable_step"] = np.array(0)
    except InstabilityError as exc:
        arrs["unstable_msg"] = np.array(str(exc))
        arrs["unstable_step"] = np.array(exc.step)
    arrs["dt_literal"] = np.array(0.1 * h * h)
    try:
        run_heat_explicit(nodes, store, dt=0.5, steps=50, dirichlet={-1: 0.0}, initial=u0)
        arrs["unstable2_msg"] = np.array("")
    except InstabilityError as exc:
        arrs["unstable2_msg"] = np.array(str(exc))
    save("heat.npz", **arrs)


# -- vector operators and the explicit Neumann closure -----------

def square_set(m=48, seed=61):
    """Jittered grid on the unit square (jitter 0.2 h inside): interior +1;
    left edge x = 0 tagged -2 with outward normal (-1, 0), the other three
    edges -1 with their outward normals."""
    rng = np.random.default_rng(seed)
    h = 1.0 / (m - 1)
    g = np.arange(m) * h
    X, Y = np.meshgrid(g, g, indexing="ij")
    pts = np.stack([X.ravel(), Y.ravel()], 1)
    on_b = (pts[:, 0] == 0) | (pts[:, 0] == g[-1]) | (pts[:, 1] == 0) | (pts[:, 1] == g[-1])
    pts[~on_b] += rng.uniform(-0.2 * h, 0.2 * h, (int((~on_b).sum()), 2))
    types = np.where(on_b, -1, 1).astype(np.int64)
    left = pts[:, 0] == 0
    types[left] = -2
    normals = np.full(pts.shape, np.nan)
    normals[left] = (-1.0, 0.0)
    normals[(pts[:, 0] == g[-1]) & ~left] = (1.0, 0.0)
    normals[(pts[:, 1] == 0) & (types == -1) & (pts[:, 0] != g[-1])] = (0.0, -1.0)
    normals[(pts[:, 1] == g[-1]) & (types == -1) & (pts[:, 0] != g[-1])] = (0.0, 1.0)
    return pts, types, normals


def dump_vector_ops():
    arrs = {}
    pts, types, normals = square_set()
    N = pts.shape[0]
    nodes = find_closest_stencils(NodeSet(pts, types, normals), 15)
    eng = RbfFd(Polyharmonic(3), degree=2, scale="support", solver="lu")
    store = compute_weights(nodes, eng, ["laplacian", "gradient", "hessian"])
    rng = np.random.default_rng(62)
    u = rng.standard_normal(N)
    vec = rng.standard_normal((N, 2))
    sample = np.sort(rng.choice(N, 300, replace=False))
    arrs.update(pts=pts, types=types, normals=normals, u=u, vec=vec, sample=sample,
                stencils=nodes.stencil_matrix().astype(np.int32))
    for f in store.families:
        arrs[f"w_{f}"] = store.values[f].reshape(N, 15)
        arrs[f"y_{f}"] = store.apply_all(f, u)
    arrs["apply_lap"] = np.array([store.apply("laplacian", u, int(i)) for i in sample])
    arrs["gradient"] = np.stack([store.gradient(u, int(i)) for i in sample])
    arrs["divergence"] = np.array([store.divergence(vec, int(i)) for i in sample])
    arrs["vector_laplacian"] = np.stack([store.vector_laplacian(vec, int(i)) for i in sample])
    arrs["grad_div"] = np.stack([store.grad_div(vec, int(i)) for i in sample])
    bnd = np.flatnonzero(types < 0)
    gn = np.linspace(-0.5, 0.5, bnd.size)
    arrs["neumann_nodes"] = bnd
    arrs["neumann_gn"] = gn
    arrs["neumann_values"] = np.array([store.neumann_value(u, int(i), normals[i], g) for i, g in zip(bnd, gn)])
    arrs["normal_comb"] = np.stack([store.normal_combination(int(i), normals[i]) for i in bnd[:40]])
    # heat with Neumann on the hole and Dirichlet on the outer circle (drivers.py:99-102)
    from scipy.spatial import cKDTree
    hmin = float(cKDTree(pts).query(pts, k=2)[0][:, 1].min())
    dt = 0.1 * hmin * hmin
    u0 = np.exp(-4.0 * np.sum((pts - 0.3) ** 2, axis=1))
    arrs["heat_dt"] = np.array(dt)
    arrs["heat_u0"] = u0
    arrs["heat_neumann"] = run_heat_explicit(nodes, store, dt=dt, steps=30, dirichlet={-1: 0.0},
                                             neumann={-2: 0.3}, initial=u0)
    arrs["heat_neumann_fn"] = run_heat_explicit(nodes, store, dt=dt, steps=20, diffusivity=0.5,
                                                dirichlet={-1: lambda p, t: p[:, 0] * (1.0 + t)},
                                                neumann={-2: lambda p, t: p[:, 1] + t}, initial=u0)
    save("vector_ops.npz", **arrs)


# -- general engines (the reference's per-node loop, storage.py:325-339) --------

from gen_golden_specs import ENGINE_ERRORS, ENGINE_VARIANTS, family_specs  # noqa: E402


def dump_engines():
    arrs = {}
    arrs["names"] = np.array([v[0] for v in ENGINE_VARIANTS])
    for vi, (name, d, N, n, eng_expr, fams) in enumerate(ENGINE_VARIANTS):
        pts = cloud(N, d, 700 + vi, 0.0, 1.0)
        nodes = find_closest_stencils(NodeSet(pts, np.ones(N, dtype=np.int64)), n)
        eng = eval(eng_expr, vars(meshfree))
        store = compute_weights(nodes, eng, family_specs(meshfree, fams))
        arrs[f"{name}_pts"] = pts
        arrs[f"{name}_stencils"] = nodes.stencil_matrix().astype(np.int32)
        arrs[f"{name}_keys"] = np.array(store.families)
        for f in store.families:
            arrs[f"{name}_w_{f}"] = store.values[f].reshape(N, n)
    arrs["errors"] = np.array([v[0] for v in ENGINE_ERRORS])
    for vi, (name, d, N, n, eng_expr, fams, mutate) in enumerate(ENGINE_ERRORS):
        pts = cloud(N, d, 800 + vi, 0.0, 1.0)
        if mutate == "coincide":
            pts[[17, 40, 41, 42, 43, 44]] = pts[17]
        nodes = find_closest_stencils(NodeSet(pts, np.ones(N, dtype=np.int64)), n)
        try:
            compute_weights(nodes, eval(eng_expr, vars(meshfree)), family_specs(meshfree, fams))
            msg = ""
        except WeightError as exc:
            msg = str(exc)
        arrs[f"err_{name}_pts"] = pts
        arrs[f"err_{name}_msg"] = np.array(msg)
        print(name, "->", msg)
    save("engines.npz", **arrs)


# -- implicit consumer (SparseSystem, solve_sparse, solve_poisson_implicit) -------

def jittered(m, d, seed):
    """m^d jittered grid nodes in the unit cube; the band within h of x = 0/1 is
    Dirichlet (-1), the band within h of the other faces Neumann (-2, outward
    axis normals), everything else interior (+1)."""
    rng = np.random.default_rng(seed)
    h = 1.0 / m
    g = np.arange(h / 2, 1, h)
    P = np.stack(np.meshgrid(*([g] * d), indexing="ij"), -1).reshape(-1, d)
    P = P + rng.uniform(-0.3 * h, 0.3 * h, P.shape)
    types = np.ones(P.shape[0], dtype=np.int64)
    normals = np.full(P.shape, np.nan)
    for a in range(1, d):
        lo, hi = P[:, a] < h, P[:, a] > 1 - h
        types[lo | hi] = -2
        normals[lo] = 0.0
        normals[hi] = 0.0
        normals[lo, a] = -1.0
        normals[hi, a] = 1.0
    xb = (P[:, 0] < h) | (P[:, 0] > 1 - h)
    types[xb] = -1
    return P, types, normals


def dump_implicit():
    from meshfree import SparseSystem
    from meshfree.drivers import solve_poisson_implicit
    from meshfree.solve import SolverConfig, solve_sparse

    arrs = {}
    cases = [
        # name, m, d, n, families, terms, neumann?
        ("dir2d", 64, 2, 15, ["laplacian"], [(-1.0, "laplacian")], False),
        ("neu2d", 56, 2, 15, ["laplacian", "gradient", "identity"], [(1.0, "laplacian"), (-0.5, "identity")], True),
        ("dir3d", 15, 3, 35, ["laplacian"], [(-1.0, "laplacian")], False),
    ]
    arrs["names"] = np.array([c[0] for c in cases])
    for ci, (name, m, d, n, fams, terms, neu) in enumerate(cases):
        pts, types, normals = jittered(m, d, 900 + ci)
        if not neu:
            types[types == -2] = -1
        nodes = find_closest_stencils(NodeSet(pts, types, normals), n)
        store = compute_weights(nodes, RbfFd(Polyharmonic(3), degree=2, scale="support", solver="lu"), fams)
        out = []
        f = lambda p: np.sin(3 * p[:, 0]) + p[:, 1] ** 2
        res = solve_poisson_implicit(nodes, store, terms=terms, rhs=f,
                                     dirichlet={-1: lambda p: p[:, 0] * p[:, 1]},
                                     neumann={-2: 0.25} if neu else None, system_out=out)
        mat, rhs = out[0]
        arrs[f"{name}_pts"] = pts
        arrs[f"{name}_types"] = types
        arrs[f"{name}_normals"] = normals
        arrs[f"{name}_stencils"] = nodes.stencil_matrix().astype(np.int32)
        for k in store.families:
            arrs[f"{name}_w_{k}"] = store.values[k].reshape(-1, n)
        arrs[f"{name}_indptr"] = mat.indptr
        arrs[f"{name}_indices"] = mat.indices
        arrs[f"{name}_data"] = mat.data
        arrs[f"{name}_rhs"] = rhs
        arrs[f"{name}_u"] = res.u
        arrs[f"{name}_iters"] = np.array(res.iterations)
        arrs[f"{name}_residual"] = np.array(res.residual)
        print(name, len(nodes), "iters", res.iterations, "residual", res.residual)
    # per-row SparseSystem: rows committed out of order, then finalize
    rng = np.random.default_rng(950)
    sysm = SparseSystem(6)
    order = [3, 0, 5, 1, 4, 2]
    for i in order:
        cols = rng.permutation(6)[: 3]
        if i not in cols:
            cols[0] = i
        sysm.add_row(i, cols, rng.standard_normal(3) + 4.0 * (cols == i), float(i))
    mat, rhs = sysm.finalize()
    arrs["rows_indptr"], arrs["rows_indices"], arrs["rows_data"], arrs["rows_rhs"] = (
        mat.indptr, mat.indices, mat.data, rhs)
    res = solve_sparse(mat, rhs)
    arrs["rows_u"] = res.u
    # errors
    msgs = {}
    def err(key, fn):
        try:
            fn()
            msgs[key] = ""
        except Exception as exc:  # noqa: BLE001
            msgs[key] = f"{type(exc).__name__}: {exc}"
    s2 = SparseSystem(4)
    s2.add_row(1, [1, 2], [1.0, 0.5], 0.0)
    err("double", lambda: s2.add_row(1, [1], [1.0], 0.0))
    err("range", lambda: s2.add_row(2, [2, 4], [1.0, 1.0], 0.0))
    err("dupcol", lambda: s2.add_row(2, [2, 2], [1.0, 1.0], 0.0))
    err("shape", lambda: s2.add_row(2, [2, 3], [1.0], 0.0))
    err("outside", lambda: s2.add_row(7, [1], [1.0], 0.0))
    err("missing", lambda: s2.finalize())
    pts, types, normals = jittered(20, 2, 960)
    nodes = find_closest_stencils(NodeSet(pts, types, normals), 12)
    store = compute_weights(nodes, RbfFd(Polyharmonic(3), degree=2, scale="support", solver="lu"),
                            ["laplacian", "gradient"])
    err("neu_interior", lambda: solve_poisson_implicit(nodes, store, terms="laplacian", rhs=1.0,
                                                       dirichlet={-1: 0.0, -2: 0.0}, neumann={1: 0.0}))
    err("no_tag", lambda: solve_poisson_implicit(nodes, store, terms="laplacian", rhs=1.0,
                                                 dirichlet={-1: 0.0, -7: 0.0}))
    err("uncovered", lambda: solve_poisson_implicit(nodes, store, terms="laplacian", rhs=1.0,
                                                    dirichlet={-1: 0.0}))
    err("double_bc", lambda: solve_poisson_implicit(nodes, store, terms="laplacian", rhs=1.0,
                                                    dirichlet={-1: 0.0, -2: 0.0}, neumann={-2: 0.0}))
    err("family", lambda: solve_poisson_implicit(nodes, store, terms="d2_0_0", rhs=1.0,
                                                 dirichlet={-1: 0.0, -2: 0.0}))
    err("config", lambda: solve_poisson_implicit(nodes, store, terms="laplacian", rhs=1.0,
                                                 dirichlet={-1: 0.0, -2: 0.0},
                                                 config=SolverConfig(preconditioner="jacobi")))
    err("maxiter", lambda: solve_poisson_implicit(nodes, store, terms="laplacian", rhs=1.0,
                                                  dirichlet={-1: 0.0, -2: 0.0}, config=SolverConfig(max_iter=1)))
    arrs["err_pts"], arrs["err_types"], arrs["err_normals"] = pts, types, normals
    arrs["err_keys"] = np.array(list(msgs))
    arrs["err_msgs"] = np.array([msgs[k] for k in msgs])
    for k, v in msgs.items():
        print(k, "->", v)
    save("implicit.npz", **arrs)


# -- node generation (fill_interior) ------------------------------------------------

def dump_fill():
    import time

    from meshfree.geometry import shapes as rshapes
    from meshfree.geometry import spacing as rspacing
    from meshfree.geometry.fill import fill_interior

    from gen_golden_specs import FILL_CASES, fill_seeds

    ns = {**vars(rshapes), **vars(rspacing)}
    arrs = {"names": np.array([c[0] for c in FILL_CASES])}
    for name, shape_expr, h_expr, seeds_kind, kw in FILL_CASES:
        shape = eval(shape_expr, ns)
        h = eval(h_expr, ns)
        seeds = fill_seeds(seeds_kind)
        d = shape.dim
        nodes = NodeSet(seeds, -np.ones(seeds.shape[0], dtype=np.int64)) if seeds is not None else \
            NodeSet(np.empty((0, d)), np.empty(0, dtype=np.int64))
        kw = dict(kw)
        seed = kw.pop("seed", 0)
        t = time.perf_counter()
        out = fill_interior(nodes, shape, h, seed, **kw)
        dt = time.perf_counter() - t
        arrs[f"{name}_positions"] = out.positions
        arrs[f"{name}_types"] = out.types
        arrs[f"{name}_time"] = np.array(dt)
        print(name, len(out), f"{dt:.2f}s")
    errs = {}
    disk = rshapes.Ball([0.0, 0.0], 1.0)
    empty = NodeSet(np.empty((0, 2)), np.empty(0, dtype=np.int64))
    for key, fn in [
        ("gamma", lambda: fill_interior(empty, disk, 0.1, start=[[0, 0]], gamma=1.6)),
        ("start_outside", lambda: fill_interior(empty, disk, 0.1, start=[[2.0, 0.0]])),
        ("no_seeds", lambda: fill_interior(empty, disk, 0.1)),
        ("max_nodes", lambda: fill_interior(empty, disk, 0.02, start=[[0, 0]], max_nodes=500)),
        ("dims", lambda: fill_interior(NodeSet(np.zeros((1, 3)), np.ones(1, dtype=np.int64)), disk, 0.1)),
    ]:
        try:
            fn()
            errs[key] = ""
        except Exception as exc:  # noqa: BLE001
            errs[key] = f"{type(exc).__name__}: {exc}"
        print(key, "->", errs[key])
    arrs["err_keys"] = np.array(list(errs))
    arrs["err_msgs"] = np.array([errs[k] for k in errs])
    save("fill.npz", **arrs)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    which = sys.argv[1:] or ["knn", "configs", "variants", "errors", "csr", "heat", "vector", "engines", "implicit", "fill"]
    if "knn" in which:
        dump_knn()
    if "variants" in which:
        dump_weight_variants()
    if "errors" in which:
        dump_weight_errors()
    if "csr" in which:
        dump_csr_apply()
    if "heat" in which:
        dump_heat()
    if "vector" in which:
        dump_vector_ops()
    if "engines" in which:
        dump_engines()
    if "implicit" in which:
        dump_implicit()
    if "fill" in which:
        dump_fill()
    if "configs" in which:
        dump_configs()
