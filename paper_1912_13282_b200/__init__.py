"""meshfree-b200: the RBF-FD hot path of the reference ``meshfree`` package on B200.

Public API mirrors the reference:

    NodeSet, find_closest_stencils          stencil selection  (csrc/knn.cu)
    RbfFd, Polyharmonic, compute_weights    batched shape solve (csrc/phs*.cu)
    WeightedLeastSquares, Gaussian, ...      general engines, batched (csrc/engines.cu)
    WeightStore.matrix / apply / apply_all  canonical CSR + explicit apply (csrc/sparse.cu)
    run_heat_explicit                       fused forward-Euler stepping (csrc/sparse.cu)
    fill_interior                           node generation, GPU acceptance pass (csrc/fill.cu)
    SparseSystem, solve_sparse,             implicit assembly + multicolour ILU(0) BiCGStab
    solve_poisson_implicit                  (csrc/solve.cu)

All compute runs in hand-written sm_100a kernels behind the C ABI declared in
include/meshfree_b200.h; there is no CPU fallback.
"""

from .approx import (
    ConstantWeight,
    Directional,
    FirstDerivative,
    Gaussian,
    GaussianWeight,
    Identity,
    InverseMultiquadric,
    Laplacian,
    MonomialBasis,
    Multiquadric,
    Operator,
    OperatorSum,
    Polyharmonic,
    RbfFd,
    ScaledOperator,
    SecondDerivative,
    WeightedLeastSquares,
    graded_lex_exponents,
    monomial_count,
)
from .assembly import SparseSystem
from .drivers import run_heat_explicit, solve_poisson_implicit
from .errors import (
    ConfigError,
    GeometryError,
    InstabilityError,
    MeshfreeError,
    NumericalError,
    StencilError,
    StorageError,
    WeightError,
)
from .geometry import Ball, Box, ConstantSpacing, LinearSpacing, Shape, fill_interior
from .nodeset import NodeSet
from .solve import SolverConfig, SolveResult, SystemMatrix, make_preconditioner, solve_sparse
from .stencils import find_closest_stencils
from .storage import DeviceCSR, WeightStore, compute_weights, expand_families

__all__ = [
    "Ball",
    "Box",
    "ConstantSpacing",
    "LinearSpacing",
    "Shape",
    "fill_interior",
    "ConfigError",
    "ConstantWeight",
    "Directional",
    "Gaussian",
    "GaussianWeight",
    "InverseMultiquadric",
    "Multiquadric",
    "OperatorSum",
    "ScaledOperator",
    "WeightedLeastSquares",
    "DeviceCSR",
    "FirstDerivative",
    "GeometryError",
    "Identity",
    "InstabilityError",
    "Laplacian",
    "MeshfreeError",
    "MonomialBasis",
    "NodeSet",
    "NumericalError",
    "Operator",
    "Polyharmonic",
    "RbfFd",
    "SecondDerivative",
    "StencilError",
    "StorageError",
    "WeightError",
    "WeightStore",
    "compute_weights",
    "make_preconditioner",
    "solve_poisson_implicit",
    "solve_sparse",
    "SolveResult",
    "SolverConfig",
    "SparseSystem",
    "SystemMatrix",
    "expand_families",
    "find_closest_stencils",
    "graded_lex_exponents",
    "monomial_count",
    "run_heat_explicit",
]

__version__ = "0.1.0"
