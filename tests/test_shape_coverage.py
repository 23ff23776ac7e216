"""The nullspace first pass beyond the BASELINE shapes (phs_ns2_shapes.h): odd
and even stencil sizes, monomial degree 1..3 in 2D and 3D, family counts with
their own instantiation (1, d + 1) and counts run as chunks (gradient only,
hessian, laplacian + gradient + hessian), against the oracle at 1e-9 normwise
per stencil and family (the near-coincident-node allowance of
tests/test_full_configs.py applies)."""

import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1

CASES = [
    (2, 12, 2, ["laplacian"]), (2, 13, 2, ["laplacian", "gradient"]), (2, 20, 2, ["hessian"]),
    (2, 15, 2, ["laplacian", "gradient", "hessian"]), (2, 9, 1, ["laplacian", "gradient"]),
    (2, 24, 3, ["laplacian"]), (2, 16, 1, ["gradient"]), (2, 30, 2, ["laplacian", "gradient"]),
    (3, 30, 2, ["laplacian"]), (3, 35, 2, ["laplacian", "gradient"]), (3, 28, 2, ["gradient"]),
    (3, 40, 2, ["laplacian"]), (3, 16, 1, ["laplacian", "d1_2"]), (3, 45, 3, ["laplacian", "gradient"]),
    (3, 36, 2, ["hessian"]),
]


@pytest.mark.parametrize("case", CASES, ids=[f"d{c[0]}_n{c[1]}_deg{c[2]}_{'+'.join(c[3])}" for c in CASES])
def test_shape_against_oracle(case):
    import paper_1912_13282_b200 as mf
    from test_full_configs import check_bar, normwise

    d, n, deg, fams = case
    N = 20_000
    pts = np.random.default_rng(n * 10 + d).uniform(0, 1, (N, d))
    nodes = mf.find_closest_stencils(mf.NodeSet(pts, np.ones(N, dtype=np.int64)), n)
    st = nodes.stencil_matrix()
    eng = mf.RbfFd(mf.Polyharmonic(3), degree=deg, scale="support", solver="lu")
    store = mf.compute_weights(nodes, eng, fams)
    ref, fail, keys = oracle.phs_weights(pts, np.arange(N), st, fams, degree=deg, threads=THREADS)
    assert not fail.any()
    assert list(keys) == list(store.families)
    for f, key in enumerate(keys):
        err = normwise(store.values[key].reshape(N, n), ref[:, f, :])
        check_bar(pts, st, err, (case, key))
