"""Run-twice determinism of every GPU stage: the kernels use atomics
for fallback / re-solve lists, duplicate flags, peaks, grid scatters and
colouring, but none of them may change a result bit.  Each stage runs twice
on the same inputs (a mid-size 3D cloud with near-coincident nodes so the
HYBRID re-solve list is not empty) and the outputs are compared bitwise."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def run_once(pts, types, u):
    import paper_1912_13282_b200 as mf

    nodes = mf.find_closest_stencils(mf.NodeSet(pts, types), 35)
    eng = mf.RbfFd(mf.Polyharmonic(3), degree=2, scale="support", solver="lu")
    store = mf.compute_weights(nodes, eng, ["laplacian", "gradient"])
    mat = store.matrix("laplacian")
    y = store.apply_all("laplacian", u)
    grad = store.gradient(u)
    heat = mf.run_heat_explicit(nodes, store, dt=1e-13, steps=7, dirichlet={-1: 0.0}, initial=u)
    gen = mf.compute_weights(nodes, mf.RbfFd(mf.Polyharmonic(3), degree=2, scale="support", solver="qr"),
                             ["laplacian"])
    # implicit solve on a jittered grid (uniformly random clouds can stall BiCGStab)
    m = 16
    g = (np.arange(m) + 0.5) / m
    P = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    P = P + np.random.default_rng(5).uniform(-0.3 / m, 0.3 / m, P.shape)
    tp = np.where(np.min(np.minimum(P, 1 - P), axis=1) < 1.0 / m, -1, 1).astype(np.int64)
    gn = mf.find_closest_stencils(mf.NodeSet(P, tp), 35)
    gs = mf.compute_weights(gn, eng, ["laplacian"])
    res = mf.solve_poisson_implicit(gn, gs, terms=[(-1.0, "laplacian")], rhs=1.0, dirichlet={-1: 0.0})
    return {
        "stencils": nodes.stencil_matrix(),
        "w_lap": store.values["laplacian"], "w_d1_2": store.values["d1_2"],
        "indptr": mat.indptr, "indices": mat.indices, "data": mat.data,
        "apply": y, "grad": np.asarray(grad), "heat": heat, "qr": gen.values["laplacian"],
        "implicit_u": res.u, "implicit_iters": np.array(res.iterations),
        "fill": mf.fill_interior(mf.NodeSet(np.empty((0, 2)), np.empty(0, dtype=np.int64)),
                                 mf.Ball([0.0, 0.0], 1.0), 0.01, start=[[0.0, 0.0]]).positions,
    }


def test_every_stage_is_bitwise_reproducible():
    rng = np.random.default_rng(11)
    N = 60_000
    pts = rng.uniform(0, 1, (N, 3))
    pts[1:200:2] = pts[0:200:2] + 1e-5 * rng.standard_normal((100, 3))  # near-coincident pairs
    types = np.ones(N, dtype=np.int64)
    types[np.min(np.minimum(pts, 1 - pts), axis=1) < 0.04] = -1
    u = rng.standard_normal(N)
    a = run_once(pts, types, u)
    b = run_once(pts, types, u)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
