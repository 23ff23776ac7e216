"""Approximation primitives needed by the batched shape path (host side).

Restates the pieces of the reference's approx package that feed the batched
kernel: graded-lex exponents (approx/basis.py:25-33),
monomial counts (basis.py:88-90), the polyharmonic kernel (basis.py:172-228),
the elementary operators and their derivative orders (operators.py:80-155),
and the RbfFd engine descriptor (engines.py:147-158).  The per-point operator
algebra of the reference (apply_rbf/apply_monomial on arbitrary points) is not
needed on the GPU path; only the constraint right-hand side at the origin is.
"""

from __future__ import annotations

import math
from itertools import product

import numpy as np

from .errors import ConfigError


def graded_lex_exponents(dim: int, degree: int):
    """All exponent tuples with total degree <= degree, graded-lex order.

    Within one total degree, earlier axes carry higher exponents first:
    in 2D degree 2 the order is 1, x, y, x^2, xy, y^2.
    """
    expos = [e for e in product(range(degree + 1), repeat=dim) if sum(e) <= degree]
    expos.sort(key=lambda e: (sum(e), tuple(-x for x in e)))
    return expos


def monomial_count(degree: int, dim: int) -> int:
    return math.comb(degree + dim, dim)


class Operator:
    """Elementary linear differential operator evaluated at a point."""

    order: int = 0

    def terms(self):
        return [(1.0, self)]

    def origin_monomial(self, expo) -> float:
        """(L x^expo)(0)."""
        raise NotImplementedError


class Identity(Operator):
    order = 0

    def origin_monomial(self, expo):
        return 1.0 if sum(expo) == 0 else 0.0

    def __repr__(self):
        return "Identity()"


class FirstDerivative(Operator):
    order = 1

    def __init__(self, axis: int):
        self.axis = int(axis)

    def origin_monomial(self, expo):
        return 1.0 if (sum(expo) == 1 and expo[self.axis] == 1) else 0.0

    def __repr__(self):
        return f"FirstDerivative({self.axis})"


class SecondDerivative(Operator):
    order = 2

    def __init__(self, a: int, b: int):
        self.a, self.b = sorted((int(a), int(b)))

    def origin_monomial(self, expo):
        if sum(expo) != 2:
            return 0.0
        if self.a == self.b:
            return 2.0 if expo[self.a] == 2 else 0.0
        return 1.0 if (expo[self.a] == 1 and expo[self.b] == 1) else 0.0

    def __repr__(self):
        return f"SecondDerivative({self.a}, {self.b})"


class Laplacian(Operator):
    order = 2

    def origin_monomial(self, expo):
        return 2.0 if (sum(expo) == 2 and max(expo) == 2) else 0.0

    def __repr__(self):
        return "Laplacian()"


class Polyharmonic:
    """phi(r) = r^k for odd k, r^k log(r) for even k, with phi(0) = 0."""

    def __init__(self, exponent: int):
        self.exponent = int(exponent)
        if self.exponent < 1:
            raise ConfigError("polyharmonic exponent must be a positive integer")
        self.even = self.exponent % 2 == 0

    def __repr__(self):
        return f"Polyharmonic({self.exponent})"


class MonomialBasis:
    """Full monomial basis up to ``degree`` (basis.py:36-85, subset)."""

    def __init__(self, dim: int, degree: int):
        if degree < 0:
            raise ConfigError("monomial degree must be non-negative")
        self.dim = int(dim)
        self.degree = int(degree)
        self.exponents = graded_lex_exponents(self.dim, self.degree)

    @property
    def size(self) -> int:
        return len(self.exponents)

    def origin_row(self, op: Operator):
        """(L b_j)(0) for each basis monomial (basis.apply(op, origin)[0])."""
        return np.array([op.origin_monomial(e) for e in self.exponents], dtype=float)

    def __repr__(self):
        return f"MonomialBasis(dim={self.dim}, size={self.size})"


class RbfFd:
    """RBF collocation with optional monomial augmentation (engines.py:147-158).

    The GPU path implements the reference's batched configuration: a
    Polyharmonic kernel with exponent >= 3, ``solver="lu"``, scale rule
    ``none``/``nearest``/``support``.  ``mode`` selects the shape-solve variant
    (``"hybrid"``: FMA solve, conditioning-flagged stencils re-solved in the
    reference's op order; ``"replay"``: reference op order everywhere;
    ``"fast"``: FMA only).
    """

    def __init__(self, rbf, degree: int = 2, scale="nearest", solver="qr", mode="hybrid"):
        self.rbf = rbf
        self.degree = int(degree)
        self.scale = scale
        self.solver = solver
        self.mode = mode

    def __repr__(self):
        return (
            f"RbfFd({self.rbf!r}, degree={self.degree}, "
            f"scale={self.scale!r}, solver={self.solver!r})"
        )
