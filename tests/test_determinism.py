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


def test_wide_shape_solve_is_batch_size_independent():
    """The C5-shape pass pipelines consecutive stencils through one CTA (the next
    stencil's prologue runs beside the current one's multipliers): every row's weights
    must not depend on how many rows the call solves, nor on where the slice starts
    (1, 2, 3 rows; around the resident CTA count; several grid strides)."""
    import torch

    import paper_1912_13282_b200 as mf
    from paper_1912_13282_b200.stencils import knn_device
    from paper_1912_13282_b200.storage import expand_families, phs_weights_device

    rng = np.random.default_rng(3)
    p = rng.uniform(-1, 1, (60_000, 3))
    p = p[np.sum(p * p, axis=1) <= 1.0][:20_000]
    N = len(p)
    nodes = mf.NodeSet(p, np.ones(N, dtype=np.int64))
    pos_d = nodes.positions_device()
    idx_d = torch.arange(N, dtype=torch.int64, device="cuda")
    st, _ = knn_device(nodes, 70, idx_d, idx_d)
    eng = mf.RbfFd(mf.Polyharmonic(3), degree=4, scale="support", solver="lu")
    fams = expand_families(["laplacian", "gradient"], 3)
    full = phs_weights_device(pos_d, idx_d, st, eng, fams, 3)[0]
    for m in (1, 2, 3, 5, 147, 148, 149, 295, 296, 297, 593, 2367, 2368, 2369, 4737):
        for off in (0, 7777):
            out = phs_weights_device(pos_d, idx_d[off:off + m].contiguous(), st[off:off + m].contiguous(), eng,
                                     fams, 3)[0]
            assert torch.equal(out, full[off:off + m]), (m, off)
