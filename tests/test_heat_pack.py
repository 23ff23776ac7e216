"""The packed heat loop (mf_heat_pack + ell_heat_packed_k in csrc/sparse.cu)
against the oracle, bit for bit.  The node set is large enough that the
Morton-ordered plan has both tile kinds: 16-bit column offsets, and "wide"
tiles whose offsets leave int16 and read the 32-bit indices.  The oracle is
the C restatement of the run_heat_explicit loop (drivers.py:87-110).
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def test_packed_heat_bitwise_both_tile_kinds(monkeypatch):
    import paper_1912_13282_b200 as m
    from paper_1912_13282_b200 import drivers

    rng = np.random.default_rng(5)
    N = 120_000
    pts = rng.uniform(0, 1, (N, 2))
    h = 1 / np.sqrt(N)
    types = np.where(np.min(np.minimum(pts, 1 - pts), axis=1) < h, -1, 1).astype(np.int64)
    nodes = m.find_closest_stencils(m.NodeSet(pts, types), 15)
    store = m.compute_weights(nodes, m.RbfFd(m.Polyharmonic(3), degree=2, scale="support", solver="lu"),
                              ["laplacian"])
    lap = store.matrix("laplacian")
    plan = lap.plan(True)
    idx = plan.ell_idx.cpu().numpy().reshape(-1, plan.W, 32)
    ln = plan.ell_len.cpu().numpy()
    rows = np.arange(idx.shape[0] * 32).reshape(-1, 32)
    valid = np.arange(plan.W)[None, :, None] < np.pad(ln, (0, rows.size - N)).reshape(-1, 32)[:, None, :]
    off = np.abs(idx.astype(np.int64) - rows[:, None, :])
    wide = np.any(valid & (off > 32767), axis=(1, 2))
    assert 0 < wide.sum() < wide.size, f"{wide.sum()} wide tiles of {wide.size}"

    u0 = np.exp(-50 * ((pts[:, 0] - 0.5) ** 2 + (pts[:, 1] - 0.5) ** 2))
    dt = 1e-12
    steps = 12
    u_pack = m.run_heat_explicit(nodes, store, dt=dt, steps=steps, dirichlet={-1: 0.25}, initial=u0)
    monkeypatch.setattr(drivers, "PACK_OPERATOR", False)
    u_plain = m.run_heat_explicit(nodes, store, dt=dt, steps=steps, dirichlet={-1: 0.25}, initial=u0)
    assert np.array_equal(u_pack.view(np.int64), u_plain.view(np.int64))

    interior = (types > 0).astype(np.uint8)
    diri = (types == -1).astype(np.uint8)
    g = np.where(diri == 1, 0.25, 0.0)
    u_init = np.where(diri == 1, 0.25, u0)
    ref, bad, _ = oracle.heat_steps(lap.indptr, lap.indices, lap.data, interior, diri, g, u_init, dt=dt,
                                    steps=steps)
    assert bad == 0
    assert np.array_equal(u_pack.view(np.int64), ref.view(np.int64))


def test_packed_heat_time_dependent_matches_plain(monkeypatch):
    """Time-dependent Dirichlet data: one launch per step over the packed plan."""
    import paper_1912_13282_b200 as m
    from paper_1912_13282_b200 import drivers

    rng = np.random.default_rng(9)
    N = 3001  # not a multiple of 32: a partial last tile
    pts = rng.uniform(0, 1, (N, 2))
    types = np.where(np.min(np.minimum(pts, 1 - pts), axis=1) < 0.02, -1, 1).astype(np.int64)
    nodes = m.find_closest_stencils(m.NodeSet(pts, types), 9)
    store = m.compute_weights(nodes, m.RbfFd(m.Polyharmonic(3), degree=1, scale="support", solver="lu"),
                              ["laplacian"])
    fn = lambda p, t: t * p[:, 0] + 0.5  # noqa: E731
    args = dict(dt=1e-7, steps=11, dirichlet={-1: fn}, initial=np.cos(pts[:, 1]))
    u_pack = m.run_heat_explicit(nodes, store, **args)
    monkeypatch.setattr(drivers, "PACK_OPERATOR", False)
    u_plain = m.run_heat_explicit(nodes, store, **args)
    assert np.array_equal(u_pack.view(np.int64), u_plain.view(np.int64))
    idx = nodes.boundary_indices()
    assert np.array_equal(u_pack[idx], fn(pts[idx], 11 * 1e-7))
