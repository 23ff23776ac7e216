"""Canonical CSR for the C5 stencil size (n = 70: the 128-wide pruned sorting
network, keys column << 7 | slot) against the oracle's restatement of
WeightStore.matrix (storage.py:156-170), bit for bit, and the apply on it."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def test_csr_n70_bitwise():
    import paper_1912_13282_b200 as m

    rng = np.random.default_rng(21)
    N = 12_000
    pts = rng.uniform(-1, 1, (N, 3))
    nodes = m.find_closest_stencils(m.NodeSet(pts, np.ones(N, dtype=np.int64)), 70)
    store = m.compute_weights(nodes, m.RbfFd(m.Polyharmonic(3), degree=4, scale="support", solver="lu"),
                              ["laplacian"])
    mat = store.matrix("laplacian")
    st = np.stack([nodes.stencil(i) for i in range(N)])
    ip, ix, da = oracle.csr_canonical(np.arange(N), st, store.values["laplacian"].reshape(-1, 70), N)
    assert np.array_equal(mat.indptr, ip) and np.array_equal(mat.indices, ix)
    assert np.array_equal(mat.data, da)
    u = rng.standard_normal(N)
    assert np.array_equal(store.apply_all("laplacian", u), oracle.apply(ip, ix, da, u))
