"""Host-side logic of the §8(f) rows, on CPU (no device): shape membership and
spacing (geometry/shapes.py, spacing.py), the operator algebra and the
engine encoding for the general weight kernel (approx/operators.py,
engines.py), SparseSystem's per-row checks (assembly.py) and SolverConfig
validation (solve.py).  Messages are the reference's."""

import numpy as np
import pytest


def test_shapes_membership_and_boxes():
    from paper_1912_13282_b200 import Ball, Box
    from paper_1912_13282_b200.errors import GeometryError
    from paper_1912_13282_b200.geometry import IN, OUT, SURF

    disk = Ball([0.0, 0.0], 1.0)
    hole = Ball([0.5, 0.0], 0.25, tag=-2)
    shape = disk - hole
    pts = np.array([[0.0, 0.0], [0.5, 0.0], [1.0, 0.0], [0.75, 0.0], [2.0, 0.0], [0.0, 0.5]])
    assert shape.classify(pts).tolist() == [IN, OUT, SURF, SURF, OUT, IN]
    assert shape.interior_contains(pts).tolist() == [True, False, False, False, False, True]
    assert shape.contains(pts).tolist() == [True, False, True, True, False, True]
    u = Box([0, 0], [1, 1]) | Box([0.5, 0.5], [2, 2])
    lo, hi = u.bounding_box()
    assert lo.tolist() == [0, 0] and hi.tolist() == [2, 2]
    assert u.classify(np.array([[1.0, 1.0], [1.5, 0.2], [1.9, 1.9]])).tolist() == [IN, OUT, IN]
    with pytest.raises(GeometryError, match="boundary tags must be negative"):
        Ball([0, 0], 1.0, tag=1)
    with pytest.raises(GeometryError, match="box needs hi > lo"):
        Box([0, 0], [1, 0])
    with pytest.raises(GeometryError, match="points have dimension 3, shape has 2"):
        disk.contains(np.zeros((1, 3)))


def test_spacing():
    from paper_1912_13282_b200 import ConstantSpacing, LinearSpacing
    from paper_1912_13282_b200.errors import GeometryError
    from paper_1912_13282_b200.geometry import as_spacing

    assert as_spacing(0.1)(np.zeros((3, 2))).tolist() == [0.1, 0.1, 0.1]
    h = LinearSpacing(0.1, [0.5, 0.0])
    assert np.allclose(h(np.array([[0.0, 0.0], [1.0, 3.0]])), [0.1, 0.6])
    with pytest.raises(GeometryError, match="non-positive"):
        h(np.array([[-1.0, 0.0]]))
    with pytest.raises(GeometryError, match="spacing must be positive"):
        ConstantSpacing(0.0)


def test_operator_algebra_and_engine_encoding():
    import paper_1912_13282_b200 as mf
    from paper_1912_13282_b200 import _lib
    from paper_1912_13282_b200.storage import _batchable, encode_engine, expand_families

    op = 2 * mf.Laplacian() + mf.FirstDerivative(0) - 0.5 * mf.Identity()
    terms = op.terms()
    assert [(c, type(e).__name__) for c, e in terms] == [(2.0, "Laplacian"), (1.0, "FirstDerivative"),
                                                          (-0.5, "Identity")]
    assert op.order == 2
    # (L x^e)(0) through the algebra: laplacian of x^2 -> 2, d/dx of x -> 1, identity of 1 -> 1
    assert op.origin_monomial((2, 0)) == 4.0
    assert op.origin_monomial((1, 0)) == 1.0
    assert op.origin_monomial((0, 0)) == -0.5
    assert mf.Directional([0.6, 0.8]).origin_monomial((0, 1)) == 0.8
    fams = expand_families(["laplacian", ("mix", op), "gradient"], 2)
    assert list(fams) == ["laplacian", "mix", "d1_0", "d1_1"]
    rbf = mf.RbfFd(mf.Polyharmonic(3), degree=2)  # the reference default: qr
    assert not _batchable(rbf, fams)
    assert _batchable(mf.RbfFd(mf.Polyharmonic(3), degree=2, solver="lu"), expand_families(["laplacian"], 2))
    e = encode_engine(rbf, fams, 2, 15)
    assert (e.engine, e.rbf, e.k, e.solver, e.scale_code, e.l, e.nf) == (
        _lib.MF_ENGINE_RBFFD, _lib.MF_RBF_PHS, 3, _lib.MF_SOLVER_QR, 1, 6, 4)
    assert list(e.term0[:5]) == [0, 1, 4, 5, 6]
    assert list(e.term_kind[:6]) == [_lib.MF_TERM_LAPLACIAN, _lib.MF_TERM_LAPLACIAN, _lib.MF_TERM_D1,
                                     _lib.MF_TERM_IDENTITY, _lib.MF_TERM_D1, _lib.MF_TERM_D1]
    assert list(e.term_coeff[:4]) == [1.0, 2.0, 1.0, -0.5]
    w = encode_engine(mf.WeightedLeastSquares(2, weight=mf.GaussianWeight(0.5), scale="support", solver="svd"),
                      {"laplacian": mf.Laplacian()}, 3, 20)
    assert (w.engine, w.weight, w.weight_sigma, w.l, w.solver) == (_lib.MF_ENGINE_WLS, _lib.MF_WEIGHT_GAUSSIAN,
                                                                    0.5, 10, _lib.MF_SOLVER_SVD)


def test_sparse_system_row_checks_and_solver_config():
    import paper_1912_13282_b200 as mf

    s = mf.SparseSystem(4)
    s.add_row(1, [1, 2], [1.0, 0.5], 3.0)
    assert s.nnz == 2 and s.rhs[1] == 3.0
    assert repr(s) == "SparseSystem(n=4, committed=1, nnz=2)"
    for args, msg in [((1, [1], [1.0], 0.0), "row 1 is already committed"),
                      ((2, [2, 4], [1.0, 1.0], 0.0), "row 2: column index out of range"),
                      ((2, [2, 2], [1.0, 1.0], 0.0), "row 2: duplicate columns in one equation"),
                      ((2, [2, 3], [1.0], 0.0), "cols and vals must be matching 1-d arrays"),
                      ((7, [1], [1.0], 0.0), "row 7 outside system of size 4")]:
        with pytest.raises(mf.StorageError, match=msg):
            s.add_row(*args)
    with pytest.raises(mf.StorageError, match=r"3 rows never committed \(first: node 0\)"):
        s.finalize()
    mf.SolverConfig().validate()
    mf.SolverConfig(preconditioner="ilu0").validate()
    for bad, msg in [(dict(method="gmres"), "unknown solver method"), (dict(preconditioner="jacobi"),
                     "unknown preconditioner"), (dict(tol=0.0), "out of range"), (dict(fill_factor=0.5),
                     "out of range"), (dict(max_iter=-1), "out of range")]:
        with pytest.raises(mf.ConfigError, match=msg):
            mf.SolverConfig(**bad).validate()
