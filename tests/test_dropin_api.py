"""The reference's object-level API on the path,
as a caller who swaps the import would use it: module paths through
``compat.install()``, host evaluation of kernels / operators / bases
(approx/basis.py:67-82, 101-228; operators.py:28-37), the per-stencil
``engine.weights(points, center, op)`` entry (engines.py:115-138, 160-209;
computed by the device kernels), and the scipy vocabulary of ``matrix()``.
"""

import sys

import numpy as np
import pytest

import paper_1912_13282_b200 as mf


def test_compat_aliases_resolve_to_this_package():
    import paper_1912_13282_b200.compat as compat

    root = compat.install()
    try:
        import meshfree
        from meshfree.approx.basis import MonomialBasis, graded_lex_exponents
        from meshfree.approx.engines import RbfFd, WeightedLeastSquares
        from meshfree.drivers import run_heat_explicit, solve_poisson_implicit
        from meshfree.geometry.nodeset import NodeSet
        from meshfree.geometry.spacing import ConstantSpacing, as_spacing
        from meshfree.storage import expand_families

        assert meshfree is root and compat.install() is root
        assert NodeSet is mf.NodeSet and RbfFd is mf.RbfFd and WeightedLeastSquares is mf.WeightedLeastSquares
        assert MonomialBasis is mf.MonomialBasis and graded_lex_exponents is mf.graded_lex_exponents
        assert run_heat_explicit is mf.run_heat_explicit and solve_poisson_implicit is mf.solve_poisson_implicit
        assert expand_families is mf.expand_families and ConstantSpacing is mf.ConstantSpacing and callable(as_spacing)
        assert meshfree.backend_name() == "cuda-sm_100a"
        for name in ("NodeSet", "find_closest_stencils", "compute_weights", "WeightStore", "SparseSystem",
                     "solve_sparse", "SolverConfig", "fill_interior", "Ball", "Box", "Laplacian", "Polyharmonic"):
            assert hasattr(meshfree, name), name
        # out-of-scope names import, and say so when called
        from meshfree import discretize_boundary

        with pytest.raises(mf.ConfigError, match="outside the B200 hot path"):
            discretize_boundary(mf.Ball([0.0, 0.0], 1.0), 0.1)
    finally:
        compat.uninstall()
    assert "meshfree" not in sys.modules and "meshfree.geometry" not in sys.modules


def test_compat_refuses_to_shadow_another_meshfree():
    import types

    import paper_1912_13282_b200.compat as compat

    sys.modules["meshfree"] = types.ModuleType("meshfree")
    try:
        with pytest.raises(mf.ConfigError, match="already imported"):
            compat.install()
    finally:
        del sys.modules["meshfree"]


REFERENCE_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not __import__("os").path.isdir(REFERENCE_SRC), reason="the reference exists only in the build container")
def test_compat_routes_boundary_discretisation_to_a_supplied_reference():
    """compat.install(reference=...): host boundary geometry from the CPU package, this
    package's NodeSet out; nothing else is routed."""
    import importlib

    import paper_1912_13282_b200.compat as compat

    sys.path.insert(0, REFERENCE_SRC)
    try:
        reference = importlib.import_module("meshfree")
        root = compat.install(force=True, reference=reference)
        import meshfree

        assert meshfree is root and meshfree.NodeSet is mf.NodeSet and meshfree.compute_weights is mf.compute_weights
        shape = mf.Ball([0.0, 0.0], 1.0) - mf.Ball([0.3, 0.0], 0.2, tag=-2)
        nodes = meshfree.discretize_boundary(shape, 0.1, seed=1)
        assert isinstance(nodes, mf.NodeSet) and set(np.unique(nodes.types)) == {-2, -1}
        ref_nodes = reference.discretize_boundary(
            reference.Ball([0.0, 0.0], 1.0) - reference.Ball([0.3, 0.0], 0.2, tag=-2), 0.1, seed=1)
        assert np.array_equal(nodes.positions, ref_nodes.positions) and np.array_equal(nodes.normals, ref_nodes.normals)
        grid = meshfree.grid_nodes([0.0, 0.0], [1.0, 1.0], 0.25)
        assert isinstance(grid, mf.NodeSet) and len(grid) == 25 and int(np.sum(grid.types < 0)) == 16
        ghosts, ghost_of = meshfree.add_ghost_nodes(nodes, 0.1)
        assert isinstance(ghosts, mf.NodeSet) and len(ghosts) == 2 * len(nodes) and ghost_of[0] == len(nodes)
    finally:
        compat.uninstall()
        for key in [k for k in sys.modules if k == "meshfree" or k.startswith("meshfree.")]:
            del sys.modules[key]
        sys.path.remove(REFERENCE_SRC)


def test_monomial_basis_eval_and_apply():
    b = mf.MonomialBasis(2, 2)  # 1, x, y, x^2, xy, y^2 in graded-lex order
    pts = np.array([[2.0, 3.0], [-1.0, 0.5]])
    x, y = pts[:, 0], pts[:, 1]
    table = {(0, 0): np.ones(2), (1, 0): x, (0, 1): y, (2, 0): x * x, (1, 1): x * y, (0, 2): y * y}
    assert np.array_equal(b.eval(pts), np.stack([table[e] for e in b.exponents], axis=1))
    lap = {(2, 0): 2.0, (0, 2): 2.0}
    assert np.array_equal(b.apply(mf.Laplacian(), pts),
                          np.stack([np.full(2, lap.get(e, 0.0)) for e in b.exponents], axis=1))
    dx = {(1, 0): np.ones(2), (2, 0): 2 * x, (1, 1): y}
    assert np.array_equal(b.apply(mf.FirstDerivative(0), pts),
                          np.stack([dx.get(e, np.zeros(2)) for e in b.exponents], axis=1))
    mix = 3.0 * mf.SecondDerivative(0, 1) - mf.Directional([0.0, 2.0])
    got = b.apply(mix, pts)
    want = 3.0 * b.apply(mf.SecondDerivative(1, 0), pts) - 2.0 * b.apply(mf.FirstDerivative(1), pts)
    assert np.allclose(got, want, rtol=0, atol=1e-15)
    # origin rows used by the device encoding agree with the pointwise evaluation
    for op in (mf.Identity(), mf.FirstDerivative(1), mf.SecondDerivative(0, 0), mf.Laplacian(), mix):
        assert np.array_equal(b.origin_row(op), b.apply(op, np.zeros((1, 2)))[0])
    cubic = mf.MonomialBasis.from_exponents(3, [(0, 0, 3), (1, 1, 1)])
    p3 = np.array([[0.5, -2.0, 1.5]])
    assert np.allclose(cubic.apply(mf.SecondDerivative(2, 2), p3), [[6 * 1.5, 0.0]])
    assert np.allclose(cubic.apply(mf.SecondDerivative(0, 2), p3), [[0.0, -2.0]])


@pytest.mark.parametrize("rbf", [mf.Gaussian(1.3), mf.Multiquadric(0.9), mf.InverseMultiquadric(1.1),
                                 mf.Polyharmonic(3), mf.Polyharmonic(4), mf.Polyharmonic(5)], ids=repr)
def test_radial_profiles_match_finite_differences(rbf):
    r = np.linspace(0.2, 2.5, 12)
    h = 1e-5
    d1 = (rbf.value(r + h) - rbf.value(r - h)) / (2 * h)
    d2 = (rbf.value(r + h) - 2 * rbf.value(r) + rbf.value(r - h)) / h**2
    assert np.allclose(rbf.d1_over_r(r) * r, d1, rtol=1e-7, atol=1e-8)
    assert np.allclose(rbf.d2(r), d2, rtol=2e-4, atol=2e-5)


def test_operators_on_a_radial_kernel_match_finite_differences():
    rbf = mf.Polyharmonic(3)
    rng = np.random.default_rng(5)
    diff = rng.uniform(-1, 1, (20, 3))
    phi = lambda p: rbf.value(np.linalg.norm(p, axis=1))  # noqa: E731
    h = 1e-4
    e = np.eye(3)
    fd1 = [(phi(diff + h * e[a]) - phi(diff - h * e[a])) / (2 * h) for a in range(3)]
    fd2 = [(phi(diff + h * e[a]) - 2 * phi(diff) + phi(diff - h * e[a])) / h**2 for a in range(3)]
    for a in range(3):
        assert np.allclose(mf.FirstDerivative(a).apply_rbf(rbf, diff), fd1[a], atol=1e-6)
        assert np.allclose(mf.SecondDerivative(a, a).apply_rbf(rbf, diff), fd2[a], atol=1e-5)
    assert np.allclose(mf.Laplacian().apply_rbf(rbf, diff), sum(fd2), atol=1e-5)
    assert np.allclose(mf.Directional([1.0, -2.0, 0.5]).apply_rbf(rbf, diff), fd1[0] - 2 * fd1[1] + 0.5 * fd1[2],
                       atol=1e-6)
    assert np.allclose((2.0 * mf.Laplacian() + mf.Identity()).apply_rbf(rbf, diff), 2 * sum(fd2) + phi(diff),
                       atol=1e-5)
    # at the centre: gradient zero, r^3 Laplacian zero; r^2-type kernels refuse derivatives there
    zero = np.zeros((1, 3))
    assert mf.FirstDerivative(0).apply_rbf(rbf, zero)[0] == 0.0 and mf.Laplacian().apply_rbf(rbf, zero)[0] == 0.0
    with pytest.raises(mf.NumericalError, match="singular at the stencil center"):
        mf.Laplacian().apply_rbf(mf.Polyharmonic(2), zero)
    assert mf.Polyharmonic(2).value(np.array([0.0]))[0] == 0.0


def test_shape_diameter_and_rigid_transforms():
    """shapes.py:64-70, 243-290 (membership side; boundary sampling is out of scope)."""
    assert mf.Ball([0.0, 0.0, 0.0], 1.0).diameter() == pytest.approx(2.0 * np.sqrt(3.0))
    assert mf.Box([0.0, 1.0], [3.0, 5.0]).diameter() == pytest.approx(5.0)
    moved = mf.Ball([0.0, 0.0], 1.0).translate([5.0, 0.0])
    assert moved.contains([[5.5, 0.0], [4.1, 0.0]]).all() and not moved.contains([[0.0, 0.0], [6.1, 0.0]]).any()
    lo, hi = moved.bounding_box()
    assert np.array_equal(lo, [4.0, -1.0]) and np.array_equal(hi, [6.0, 1.0])
    th = 0.3
    rot = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    box = mf.Box([0.0, 0.0], [2.0, 1.0]).rotate(rot)
    assert box.contains([rot @ np.array([1.0, 0.5]), rot @ np.array([1.9, 0.9])]).all()
    assert not box.contains([rot @ np.array([2.5, 0.5]), rot @ np.array([1.0, -0.2])]).any()
    lo, hi = box.bounding_box()
    assert lo[0] == pytest.approx(-np.sin(th)) and hi[1] == pytest.approx(2 * np.sin(th) + np.cos(th))
    both = (box | moved) - mf.Ball([5.0, 0.0], 0.5)
    assert both.interior_contains([[5.8, 0.0]]).all() and not both.contains([[5.1, 0.0]]).any()
    with pytest.raises(mf.GeometryError, match="orthogonal"):
        mf.Box([0.0, 0.0], [1.0, 1.0]).rotate([[1.0, 0.2], [0.0, 1.0]])
    with pytest.raises(mf.GeometryError, match="offset dimension"):
        mf.Ball([0.0, 0.0], 1.0).translate([1.0, 2.0, 3.0])


def test_weight_functions_are_callable():
    off = np.array([[0.3, 0.4], [0.0, 0.0]])
    assert np.array_equal(mf.ConstantWeight()(off), np.ones(2))
    assert np.allclose(mf.GaussianWeight(0.5)(off), [np.exp(-1.0), 1.0])


CROSS = np.array([[0.0, 0.0], [1.0, 0.0], [-1.0, 0.0], [0.0, 1.0], [0.0, -1.0]])


@pytest.mark.gpu
def test_engine_weights_single_stencil_closed_forms():
    h = 0.25
    w = mf.WeightedLeastSquares(mf.MonomialBasis.from_exponents(2, [(0, 0), (1, 0), (0, 1), (2, 0), (0, 2)])) \
        .weights(h * CROSS, np.zeros(2), mf.Laplacian())
    assert np.allclose(w, np.array([-4.0, 1.0, 1.0, 1.0, 1.0]) / h**2, rtol=1e-10)
    line = np.array([[-h], [0.0], [h]])
    assert np.allclose(mf.WeightedLeastSquares(2).weights(line, np.zeros(1), mf.FirstDerivative(0)),
                       [-0.5 / h, 0.0, 0.5 / h], atol=1e-10 / h)
    assert np.allclose(mf.WeightedLeastSquares(2).weights(line, np.zeros(1), mf.SecondDerivative(0, 0)),
                       np.array([1.0, -2.0, 1.0]) / h**2, rtol=1e-10)
    # the centre need not be a support node; weights move with it
    rng = np.random.default_rng(2)
    pts = rng.uniform(-1, 1, (12, 2))
    c = np.array([0.1, -0.2])
    for eng in (mf.RbfFd(mf.Polyharmonic(3), degree=2), mf.RbfFd(mf.Polyharmonic(3), degree=2, solver="lu"),
                mf.WeightedLeastSquares(2), mf.RbfFd(mf.Gaussian(1.0), degree=1, scale="support")):
        wl = eng.weights(pts, c, mf.Laplacian())
        wx = eng.weights(pts, c, mf.FirstDerivative(0))
        assert wl.shape == (12,) and wx.shape == (12,)
        # exact on the augmentation / fit space: u = 1 + x - y (+ x^2 - 3xy for degree 2)
        x, y = pts[:, 0], pts[:, 1]
        lin = 1 + x - y
        assert abs(wx @ lin - 1.0) < 1e-8 and abs(wl @ lin) < 1e-7
        if "Gaussian" not in repr(eng):
            quad = lin + x * x - 3 * x * y
            assert abs(wl @ quad - 2.0) < 1e-7 and abs(wx @ quad - (1 + 2 * c[0] - 3 * c[1])) < 1e-8
        shifted = eng.weights(pts + 5.0, c + 5.0, mf.Laplacian())
        assert np.allclose(shifted, wl, rtol=1e-6, atol=1e-8 * np.max(np.abs(wl)))


@pytest.mark.gpu
def test_engine_weights_error_classes():
    rng = np.random.default_rng(3)
    pts = rng.uniform(-1, 1, (9, 2))
    with pytest.raises(mf.ConfigError, match="unknown dense solver"):
        mf.RbfFd(mf.Polyharmonic(3), degree=1, solver="bogus").weights(pts, np.zeros(2), mf.Laplacian())
    with pytest.raises(mf.ConfigError, match="unknown scale rule"):
        mf.WeightedLeastSquares(2, scale="bogus").weights(pts, np.zeros(2), mf.Laplacian())
    with pytest.raises(mf.NumericalError, match="needs at least 10"):
        mf.RbfFd(mf.Polyharmonic(3), degree=3).weights(pts, np.zeros(2), mf.Laplacian())
    with pytest.raises(mf.NumericalError, match="lu needs a square local system"):
        mf.WeightedLeastSquares(2, solver="lu").weights(pts, np.zeros(2), mf.Laplacian())
    try:
        mf.RbfFd(mf.Polyharmonic(3), degree=3).weights(pts, np.zeros(2), mf.Laplacian())
    except mf.NumericalError as exc:
        assert not isinstance(exc, mf.WeightError) and not str(exc).startswith("node ")


@pytest.mark.gpu
def test_matrix_speaks_scipy():
    rng = np.random.default_rng(4)
    pts = rng.uniform(0, 1, (400, 2))
    nodes = mf.find_closest_stencils(mf.NodeSet(pts, np.ones(400, dtype=np.int64)), 9)
    store = mf.compute_weights(nodes, mf.RbfFd(mf.Polyharmonic(3), degree=2, solver="lu"), ["laplacian", "d1_0"])
    A, B = store.matrix("laplacian"), store.matrix("d1_0")
    S = A.to_scipy()
    assert np.array_equal(np.asarray(abs(A).sum(axis=1)).ravel(), np.asarray(abs(S).sum(axis=1)).ravel())
    assert np.array_equal(A.diagonal(), S.diagonal()) and np.array_equal(A.toarray(), S.toarray())
    assert np.array_equal(A[3].toarray(), S[3].toarray()) and A.T.shape == (400, 400)
    assert np.array_equal((A + B).toarray(), (S + B.to_scipy()).toarray())
    assert np.array_equal((2.0 * A).toarray(), (2.0 * S).toarray()) and np.array_equal((-A).toarray(), -S.toarray())
    u = rng.standard_normal(400)
    assert np.array_equal(A @ u, S @ u)  # the product itself stays on the device, bitwise scipy's
    import torch

    u_d = torch.as_tensor(u).cuda()
    for prod in (A * u_d, A.dot(u_d)):  # scipy's other spellings of the product: the device too
        assert isinstance(prod, torch.Tensor) and prod.is_cuda and np.array_equal(prod.cpu().numpy(), S @ u)
    assert np.array_equal(A * u, S @ u) and np.array_equal(A.dot(u), S @ u)
    with pytest.raises(AttributeError):
        A.no_such_attribute
