"""Specs of the general-engine golden cases (TEST INFRASTRUCTURE), shared by
oracle/gen_golden.py (which evaluates them against the reference) and
tests/test_engines.py (against paper_1912_13282_b200)."""

# name, d, N, n, engine expression, family expressions (strings are family names,
# "name=expr" a custom (name, operator) family); evaluated against the reference
# module here and against paper_1912_13282_b200 in tests/test_engines.py
ENGINE_VARIANTS = [
    ("rbf_qr_default_2d", 2, 300, 15, "RbfFd(Polyharmonic(3), degree=2)", ["laplacian", "gradient"]),
    ("rbf_svd_k3_2d", 2, 300, 15, "RbfFd(Polyharmonic(3), degree=2, scale='support', solver='svd')",
     ["laplacian", "d1_1"]),
    ("rbf_qr_k3_3d_n35", 3, 400, 35, "RbfFd(Polyharmonic(3), degree=2, scale='support', solver='qr')",
     ["laplacian", "gradient"]),
    ("rbf_qr_k5_deg3_3d", 3, 400, 30, "RbfFd(Polyharmonic(5), degree=3, scale='support', solver='qr')",
     ["hessian"]),
    ("rbf_lu_k2_grad_2d", 2, 300, 12, "RbfFd(Polyharmonic(2), degree=1, scale='support', solver='lu')",
     ["gradient", "identity"]),
    ("rbf_qr_k4_even_2d", 2, 300, 12, "RbfFd(Polyharmonic(4), degree=1, scale='support', solver='qr')",
     ["laplacian", "d2_0_1"]),
    ("gauss_lu_deg1_2d", 2, 300, 12, "RbfFd(Gaussian(1.0), degree=1, scale='support', solver='lu')",
     ["laplacian", "d1_0"]),
    ("gauss_qr_nodeg_2d", 2, 300, 9, "RbfFd(Gaussian(0.8), degree=-1, scale='support', solver='qr')",
     ["laplacian", "identity"]),
    ("mq_qr_deg1_2d", 2, 300, 12, "RbfFd(Multiquadric(1.0), degree=1, scale='support', solver='qr')",
     ["laplacian", "gradient"]),
    ("imq_svd_deg1_3d", 3, 300, 20, "RbfFd(InverseMultiquadric(1.5), degree=1, scale='support', solver='svd')",
     ["laplacian", "d1_2"]),
    ("wls_qr_2d", 2, 300, 12, "WeightedLeastSquares(2)", ["laplacian", "gradient"]),
    ("wls_gw_svd_2d", 2, 300, 12,
     "WeightedLeastSquares(2, weight=GaussianWeight(1.0), scale='support', solver='svd')", ["laplacian", "d1_0"]),
    ("wls_lu_square_2d", 2, 300, 6, "WeightedLeastSquares(2, scale='support', solver='lu')", ["laplacian"]),
    ("wls_qr_3d", 3, 300, 20, "WeightedLeastSquares(2, scale='support')", ["laplacian", "gradient"]),
    ("wls_tall_qr_2d", 2, 300, 5, "WeightedLeastSquares(2, scale='support')", ["d1_0"]),
    ("wls_expos_qr_2d", 2, 300, 8,
     "WeightedLeastSquares(MonomialBasis.from_exponents(2, [(0, 0), (1, 0), (0, 1), (2, 0), (0, 2)]), "
     "scale='support')", ["laplacian"]),
    ("custom_ops_lu_2d", 2, 300, 15, "RbfFd(Polyharmonic(3), degree=2, scale='support', solver='lu')",
     ["laplacian", "mix=2 * Laplacian() + FirstDerivative(0)", "dirv=Directional([0.6, 0.8])",
      "neg=-SecondDerivative(0, 1) - 0.5 * Identity()"]),
]

# name, d, N, n, engine, families, mutate (expression on pts), for_which
ENGINE_ERRORS = [
    ("phs2_laplacian", 2, 60, 9, "RbfFd(Polyharmonic(2), degree=1, solver='lu')", ["gradient", "laplacian"],
     None),
    ("coincident_qr", 2, 60, 6, "RbfFd(Polyharmonic(3), degree=1, solver='qr')", ["laplacian"], "coincide"),
    ("wls_lu_nonsquare", 2, 60, 9, "WeightedLeastSquares(2, solver='lu')", ["laplacian"], None),
    ("aug_too_large_qr", 2, 60, 5, "RbfFd(Polyharmonic(3), degree=2, solver='qr')", ["laplacian"], None),
    ("wls_weight_zero", 2, 60, 9, "WeightedLeastSquares(1, weight=GaussianWeight(0.01), scale='support')",
     ["laplacian"], None),
    ("unknown_solver", 2, 60, 9, "RbfFd(Polyharmonic(3), degree=1, solver='cholesky')", ["laplacian"], None),
]


def family_specs(mod, fams):
    ns = vars(mod)
    out = []
    for f in fams:
        if "=" in f:
            name, expr = f.split("=", 1)
            out.append((name, eval(expr, ns)))
        else:
            out.append(f)
    return out


# fill_interior cases: name, shape expression (Ball / Box / differences, evaluated
# against the reference's geometry.shapes here and paper_1912_13282_b200 in the
# tests), spacing expression, seed-node generator, keyword arguments
FILL_CASES = [
    ("disk_hole_2d", "Ball([0.0, 0.0], 1.0) - Ball([0.3, 0.1], 0.25, tag=-2)", "0.02", "circles", {}),
    ("box_linear_2d", "Box([0.0, 0.0], [1.0, 0.5])", "LinearSpacing(0.01, [0.02, 0.0])", "box_edges", {}),
    ("ball_start_3d", "Ball([0.0, 0.0, 0.0], 1.0)", "0.07", "none", {"start": [[0.1, 0.0, 0.0]]}),
    ("interval_1d", "Ball([0.0], 1.0)", "0.01", "none", {"start": [[0.05]], "gamma": 0.6}),
    ("box3d_gamma", "Box([0.0, 0.0, 0.0], [1.0, 1.0, 0.6])", "0.06", "none",
     {"start": [[0.5, 0.5, 0.3], [0.2, 0.2, 0.2]], "gamma": 0.9, "n_candidates": 10, "seed": 7}),
]


def fill_seeds(kind):
    """Seed node positions for FILL_CASES (analytic boundary samples)."""
    import numpy as np

    if kind == "circles":
        t = np.arange(0, 2 * np.pi, 0.02)
        outer = np.stack([np.cos(t), np.sin(t)], 1)
        t2 = np.arange(0, 2 * np.pi, 0.02 / 0.25)
        inner = np.stack([0.3 + 0.25 * np.cos(t2), 0.1 + 0.25 * np.sin(t2)], 1)
        return np.concatenate([outer, inner])
    if kind == "box_edges":
        x = np.linspace(0, 1, 61)
        y = np.linspace(0, 0.5, 31)[1:-1]
        return np.concatenate([np.stack([x, 0 * x], 1), np.stack([x, 0 * x + 0.5], 1),
                               np.stack([0 * y, y], 1), np.stack([0 * y + 1, y], 1)])
    return None
