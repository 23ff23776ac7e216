"""API edge cases of the drop-in layer: mixed-size host stencil
blocks, field validation before any kernel reads it, empty and duplicated row
selections, and the reference's dict behaviour of ``WeightStore.values``.
"""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def m():
    import paper_1912_13282_b200 as mod

    return mod


def small_set(N=400, seed=3):
    rng = np.random.default_rng(seed)
    pts = rng.uniform(0, 1, (N, 2))
    types = np.where(np.min(np.minimum(pts, 1 - pts), axis=1) < 0.03, -1, 1).astype(np.int64)
    return pts, types


def engine():
    return m().RbfFd(m().Polyharmonic(3), degree=2, scale="support", solver="lu")


def test_uniform_subset_of_mixed_host_stencils():
    """stencil_matrix_device uploads only the selected rows of a host-row block."""
    pts, types = small_set()
    ref_st, _ = oracle.knn(pts, 9)
    stencils = [list(r) for r in ref_st]
    stencils[5] = list(ref_st[5]) + [int(ref_st[5][-1] + 1) % len(pts)]  # one 10-node stencil
    nodes = m().NodeSet(pts, types, stencils=stencils)
    sel = np.array([0, 1, 2, 7, 11], dtype=np.int64)
    dev = nodes.stencil_matrix_device(sel).cpu().numpy()
    assert np.array_equal(dev, nodes.stencil_matrix(sel))
    store = m().compute_weights(nodes, engine(), ["laplacian"], for_which=sel)
    w, fail, _ = oracle.phs_weights(pts, sel, ref_st[sel], ["laplacian"])
    got = store.values["laplacian"].reshape(len(sel), 9)
    err = np.max(np.abs(got - w[:, 0, :]), 1) / np.max(np.abs(w[:, 0, :]), 1)
    assert not fail.any() and err.max() <= 1e-9
    with pytest.raises(m().StencilError, match="stencil sizes differ"):
        nodes.stencil_matrix_device(np.array([4, 5]))


def test_field_validation():
    pts, types = small_set()
    nodes = m().find_closest_stencils(m().NodeSet(pts, types), 9)
    store = m().compute_weights(nodes, engine(), ["laplacian"])
    N = len(pts)
    short = torch.zeros(N - 1, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="does not match"):
        store.apply_all("laplacian", short)
    with pytest.raises(ValueError, match="does not match"):
        store.matrix("laplacian") @ short
    with pytest.raises(ValueError, match="does not match"):
        store.apply_all("laplacian", np.zeros(N + 3))
    # broadcasting a scalar field is numpy's rule and stays allowed
    y = store.apply_all("laplacian", 1.0)
    assert y.shape == (N,) and np.max(np.abs(y)) < 1e-6


def test_empty_selection_gives_empty_store():
    # recycled allocator blocks full of garbage: the empty store's plan lengths
    # must be written, not left as whatever the block held
    junk = torch.full((1 << 20,), 0x7F7F7F7F, dtype=torch.int32, device="cuda")
    del junk
    pts, _ = small_set()
    types = np.ones(len(pts), dtype=np.int64)  # no boundary nodes
    nodes = m().find_closest_stencils(m().NodeSet(pts, types), 9)
    store = m().compute_weights(nodes, engine(), ["laplacian", "gradient"], for_which="boundary")
    assert store.rows.size == 0 and store.cols.size == 0
    assert store.values["laplacian"].size == 0
    y = store.apply_all("laplacian", np.ones(len(pts)))
    assert np.array_equal(y, np.zeros(len(pts)))
    mat = store.matrix("d1_0")
    assert mat.nnz == 0 and np.array_equal(mat.indptr, np.zeros(len(pts) + 1, dtype=np.int32))


def test_duplicate_rows_rejected_up_front():
    pts, types = small_set()
    nodes = m().find_closest_stencils(m().NodeSet(pts, types), 9)
    with pytest.raises(m().StorageError, match="distinct"):
        m().compute_weights(nodes, engine(), ["laplacian"], for_which=np.array([3, 4, 3]))


def test_values_behave_like_a_dict():
    pts, types = small_set()
    nodes = m().find_closest_stencils(m().NodeSet(pts, types), 9)
    store = m().compute_weights(nodes, engine(), ["laplacian", "gradient"])
    v = store.values
    assert v.get("laplacian") is v["laplacian"]
    assert v.get("nope") is None and "d1_1" in v and "nope" not in v
    cp = v.copy()
    assert set(cp) == {"laplacian", "d1_0", "d1_1"} and np.array_equal(cp["d1_0"], v["d1_0"])
    assert dict(v).keys() == cp.keys() and v == cp
    with pytest.raises(KeyError):
        v["nope"]
