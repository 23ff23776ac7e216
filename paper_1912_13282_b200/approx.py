"""Approximation primitives of the shape path (host side).

Restates the pieces of the reference's approx package that parameterise the
GPU weight kernels: graded-lex exponents
(approx/basis.py:25-33), monomial counts (basis.py:88-90), the radial kernels
(basis.py:93-228: polyharmonic, Gaussian, multiquadric, inverse
multiquadric), the elementary operators, their derivative orders and the
operator algebra (operators.py:18-244), the least-squares weight functions
(approx/weights.py) and the engine descriptors RbfFd / WeightedLeastSquares
(engines.py:102-209).  The per-point evaluation itself (apply_rbf /
apply_monomial) runs inside the kernels; only the constraint right-hand side at
the origin is evaluated here.
"""

from __future__ import annotations

import math
from itertools import product

import numpy as np

from .errors import ConfigError, NumericalError


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


def _monomial_derivative(expo, orders, points):
    """d^orders (x^expo) at `points` (M, d): every axis contributes the falling
    factorial e (e-1) .. (e-o+1) and the power x^(e-o); zero once o > e."""
    pts = np.atleast_2d(np.asarray(points, dtype=float))
    coeff = 1.0
    out = np.ones(pts.shape[0])
    for ax, (e, o) in enumerate(zip(expo, orders)):
        if o > e:
            return np.zeros(pts.shape[0])
        for t in range(o):
            coeff *= e - t
        if e - o:
            out = out * pts[:, ax] ** (e - o)
    return coeff * out


def _unit(dim, *axes):
    o = [0] * dim
    for a in axes:
        o[a] += 1
    return o


def _radius(diff):
    return np.sqrt(np.sum(np.asarray(diff, dtype=float) ** 2, axis=1))


class Operator:
    """Linear differential operator evaluated at a point (operators.py:18-52).

    Host evaluation (the reference's per-operator contract, used by
    MonomialBasis.apply and by callers that inspect operators):
    ``apply_monomial(expo, points)`` = (L x^expo)(points) and
    ``apply_rbf(rbf, diff)`` = (L phi(|x - c|)) at diff = x - c.

    ``terms()`` flattens sums and scalar multiples into (coefficient,
    elementary) pairs; ``2 * Laplacian() + FirstDerivative(0)`` builds an
    OperatorSum.  User subclasses with their own point evaluation cannot run
    on the GPU (ConfigError at compute_weights).
    """

    order: int = 0

    def terms(self):
        return [(1.0, self)]

    def origin_monomial(self, expo) -> float:
        """(L x^expo)(0)."""
        raise NotImplementedError

    def apply_monomial(self, expo, points):
        raise NotImplementedError

    def apply_rbf(self, rbf, diff):
        raise NotImplementedError

    def __mul__(self, c):
        return ScaledOperator(float(c), self)

    __rmul__ = __mul__

    def __neg__(self):
        return ScaledOperator(-1.0, self)

    def __add__(self, other):
        return OperatorSum([self, other])

    def __sub__(self, other):
        return OperatorSum([self, ScaledOperator(-1.0, other)])


class Identity(Operator):
    order = 0

    def origin_monomial(self, expo):
        return 1.0 if sum(expo) == 0 else 0.0

    def apply_monomial(self, expo, points):
        return _monomial_derivative(expo, [0] * len(expo), points)

    def apply_rbf(self, rbf, diff):
        return rbf.value(_radius(diff))

    def __repr__(self):
        return "Identity()"


class FirstDerivative(Operator):
    order = 1

    def __init__(self, axis: int):
        self.axis = int(axis)

    def origin_monomial(self, expo):
        return 1.0 if (sum(expo) == 1 and expo[self.axis] == 1) else 0.0

    def apply_monomial(self, expo, points):
        return _monomial_derivative(expo, _unit(len(expo), self.axis), points)

    def apply_rbf(self, rbf, diff):
        # phi'(r) x_a / r; zero at the centre (the kernel is only asked where r > 0)
        diff = np.atleast_2d(np.asarray(diff, dtype=float))
        r = _radius(diff)
        away = r > 0
        out = np.zeros(r.shape[0])
        out[away] = diff[away, self.axis] * rbf.d1_over_r(r[away])
        return out

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

    def apply_monomial(self, expo, points):
        return _monomial_derivative(expo, _unit(len(expo), self.a, self.b), points)

    def apply_rbf(self, rbf, diff):
        # phi'' e_a e_b + (phi'/r) (delta_ab - e_a e_b), e = diff / r (e e^T -> 0 at the centre)
        diff = np.atleast_2d(np.asarray(diff, dtype=float))
        r = _radius(diff)
        rr = np.where(r > 0, r * r, 1.0)
        ee = np.where(r > 0, diff[:, self.a] * diff[:, self.b] / rr, 0.0)
        delta = 1.0 if self.a == self.b else 0.0
        return rbf.d2(r) * ee + rbf.d1_over_r(r) * (delta - ee)

    def __repr__(self):
        return f"SecondDerivative({self.a}, {self.b})"


class Laplacian(Operator):
    order = 2

    def origin_monomial(self, expo):
        return 2.0 if (sum(expo) == 2 and max(expo) == 2) else 0.0

    def apply_monomial(self, expo, points):
        total = np.zeros(np.atleast_2d(points).shape[0])
        for ax in range(len(expo)):
            total += _monomial_derivative(expo, _unit(len(expo), ax, ax), points)
        return total

    def apply_rbf(self, rbf, diff):
        diff = np.atleast_2d(np.asarray(diff, dtype=float))
        r = _radius(diff)
        return rbf.d2(r) + (diff.shape[1] - 1) * rbf.d1_over_r(r)

    def __repr__(self):
        return "Laplacian()"


class Directional(Operator):
    """First derivative along a fixed vector, (v . grad) (operators.py:178-202)."""

    order = 1

    def __init__(self, vector):
        self.vector = np.atleast_1d(np.asarray(vector, dtype=float))

    def origin_monomial(self, expo):
        if sum(expo) != 1:
            return 0.0
        a = list(expo).index(1)
        return float(self.vector[a]) if a < self.vector.shape[0] else 0.0

    def apply_monomial(self, expo, points):
        total = np.zeros(np.atleast_2d(points).shape[0])
        for ax, v in enumerate(self.vector):
            if v != 0.0:
                total += v * _monomial_derivative(expo, _unit(len(expo), ax), points)
        return total

    def apply_rbf(self, rbf, diff):
        total = np.zeros(np.atleast_2d(diff).shape[0])
        for ax, v in enumerate(self.vector):
            if v != 0.0:
                total += v * FirstDerivative(ax).apply_rbf(rbf, diff)
        return total

    def __repr__(self):
        return f"Directional({self.vector.tolist()})"


class ScaledOperator(Operator):
    def __init__(self, coeff: float, inner: Operator):
        self.coeff = float(coeff)
        self.inner = inner

    @property
    def order(self):
        return self.inner.order

    def terms(self):
        return [(self.coeff * c, op) for c, op in self.inner.terms()]

    def origin_monomial(self, expo):
        return self.coeff * self.inner.origin_monomial(expo)

    def apply_monomial(self, expo, points):
        return self.coeff * self.inner.apply_monomial(expo, points)

    def apply_rbf(self, rbf, diff):
        return self.coeff * self.inner.apply_rbf(rbf, diff)

    def __mul__(self, c):
        return ScaledOperator(self.coeff * float(c), self.inner)

    __rmul__ = __mul__

    def __repr__(self):
        return f"{self.coeff} * {self.inner!r}"


class OperatorSum(Operator):
    def __init__(self, parts):
        flat = []
        for p in parts:
            if isinstance(p, OperatorSum):
                flat.extend(p.parts)
            else:
                flat.append(p)
        self.parts = flat

    @property
    def order(self):
        return max(p.order for p in self.parts)

    def terms(self):
        out = []
        for p in self.parts:
            out.extend(p.terms())
        return out

    def origin_monomial(self, expo):
        acc = self.parts[0].origin_monomial(expo)
        for p in self.parts[1:]:
            acc = acc + p.origin_monomial(expo)
        return acc

    def apply_monomial(self, expo, points):
        return sum(p.apply_monomial(expo, points) for p in self.parts)

    def apply_rbf(self, rbf, diff):
        return sum(p.apply_rbf(rbf, diff) for p in self.parts)

    def __repr__(self):
        return " + ".join(repr(p) for p in self.parts)


class Gaussian:
    """phi(r) = exp(-(r / sigma)^2) (basis.py:93-113)."""

    def __init__(self, sigma: float):
        self.sigma = float(sigma)
        if self.sigma <= 0:
            raise ConfigError("gaussian shape parameter must be positive")

    # radial profile on the host: value, phi'(r) / r and phi''(r) (basis.py:101-112)
    def value(self, r):
        return np.exp(-(np.asarray(r, dtype=float) / self.sigma) ** 2)

    def d1_over_r(self, r):
        return self.value(r) * (-2.0 / self.sigma**2)

    def d2(self, r):
        q = (np.asarray(r, dtype=float) / self.sigma) ** 2
        return self.value(r) * (4.0 * q - 2.0) / self.sigma**2

    def __repr__(self):
        return f"Gaussian({self.sigma})"


class Multiquadric:
    """phi(r) = sqrt(1 + (r / sigma)^2) (basis.py:116-140)."""

    def __init__(self, sigma: float):
        self.sigma = float(sigma)
        if self.sigma <= 0:
            raise ConfigError("multiquadric shape parameter must be positive")

    def value(self, r):
        return np.sqrt(1.0 + (np.asarray(r, dtype=float) / self.sigma) ** 2)

    def d1_over_r(self, r):
        return 1.0 / (self.sigma**2 * self.value(r))

    def d2(self, r):
        return 1.0 / (self.sigma**2 * self.value(r) ** 3)

    def __repr__(self):
        return f"Multiquadric({self.sigma})"


class InverseMultiquadric:
    """phi(r) = 1 / sqrt(1 + (r / sigma)^2) (basis.py:143-167)."""

    def __init__(self, sigma: float):
        self.sigma = float(sigma)
        if self.sigma <= 0:
            raise ConfigError("inverse multiquadric shape parameter must be positive")

    def value(self, r):
        return 1.0 / np.sqrt(1.0 + (np.asarray(r, dtype=float) / self.sigma) ** 2)

    def d1_over_r(self, r):
        return -self.value(r) ** 3 / self.sigma**2

    def d2(self, r):
        g = self.value(r)
        q = (np.asarray(r, dtype=float) / self.sigma) ** 2
        return g**3 * (3.0 * q * g * g - 1.0) / self.sigma**2

    def __repr__(self):
        return f"InverseMultiquadric({self.sigma})"


class ConstantWeight:
    """w(x) = 1 (approx/weights.py:15-20)."""

    def __call__(self, offsets):
        return np.ones(np.atleast_2d(offsets).shape[0])

    def __repr__(self):
        return "ConstantWeight()"


class GaussianWeight:
    """w(x) = exp(-(|x| / sigma)^2) (approx/weights.py:23-37)."""

    def __init__(self, sigma: float):
        self.sigma = float(sigma)
        if self.sigma <= 0:
            raise ConfigError("weight shape parameter must be positive")

    def __call__(self, offsets):
        off = np.atleast_2d(np.asarray(offsets, dtype=float))
        return np.exp(-np.sum(off * off, axis=1) / self.sigma**2)

    def __repr__(self):
        return f"GaussianWeight({self.sigma})"


class Polyharmonic:
    """phi(r) = r^k for odd k, r^k log(r) for even k, with phi(0) = 0."""

    def __init__(self, exponent: int):
        self.exponent = int(exponent)
        if self.exponent < 1:
            raise ConfigError("polyharmonic exponent must be a positive integer")
        self.even = self.exponent % 2 == 0

    # radial profile on the host (basis.py:186-228): r^k, or r^k log r for even k
    # with phi(0) = 0; derivatives at r = 0 need k >= 3
    def _derivative_radius(self, r):
        r = np.asarray(r, dtype=float)
        if self.exponent <= 2 and np.any(r == 0):
            raise NumericalError(
                f"derivatives of polyharmonic r^{self.exponent} are singular "
                "at the stencil center; use an exponent of 3 or more"
            )
        return r

    def value(self, r):
        r = np.asarray(r, dtype=float)
        if not self.even:
            return r**self.exponent
        pos = r > 0
        safe = np.where(pos, r, 1.0)
        return np.where(pos, safe**self.exponent * np.log(safe), 0.0)

    def d1_over_r(self, r):
        k, r = self.exponent, self._derivative_radius(r)
        with np.errstate(divide="ignore", invalid="ignore"):
            if not self.even:
                return k * r ** (k - 2.0)
            pos = r > 0
            safe = np.where(pos, r, 1.0)
            return np.where(pos, safe ** (k - 2) * (1.0 + k * np.log(safe)), 0.0)

    def d2(self, r):
        k, r = self.exponent, self._derivative_radius(r)
        with np.errstate(divide="ignore", invalid="ignore"):
            if not self.even:
                return (k * (k - 1.0)) * r ** (k - 2.0)
            pos = r > 0
            safe = np.where(pos, r, 1.0)
            return np.where(pos, safe ** (k - 2) * (k * (k - 1) * np.log(safe) + (2.0 * k - 1.0)), 0.0)

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

    @classmethod
    def from_exponents(cls, dim: int, exponents):
        """Explicit exponent list (basis.py:50-62)."""
        self = cls.__new__(cls)
        self.dim = int(dim)
        self.exponents = [tuple(int(x) for x in e) for e in exponents]
        if not self.exponents:
            raise ConfigError("empty monomial basis")
        for e in self.exponents:
            if len(e) != dim or any(x < 0 for x in e):
                raise ConfigError(f"bad exponent tuple {e} for dimension {dim}")
        self.degree = max(sum(e) for e in self.exponents)
        return self

    @property
    def size(self) -> int:
        return len(self.exponents)

    def eval(self, points):
        """B[i, j] = b_j(points[i]) (basis.py:67-71)."""
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        zero = [0] * self.dim
        return np.stack([_monomial_derivative(e, zero, pts) for e in self.exponents], axis=1)

    def apply(self, op, points):
        """(L b_j)(points[i]), one column per basis function (basis.py:73-82)."""
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        cols = []
        for e in self.exponents:
            col = np.zeros(pts.shape[0])
            for coeff, elem in op.terms():
                col += coeff * elem.apply_monomial(e, pts)
            cols.append(col)
        return np.stack(cols, axis=1)

    def origin_row(self, op: Operator):
        """(L b_j)(0) for each basis monomial (basis.apply(op, origin)[0])."""
        return np.array([op.origin_monomial(e) for e in self.exponents], dtype=float)

    def __repr__(self):
        return f"MonomialBasis(dim={self.dim}, size={self.size})"


def _single_stencil_weights(engine, points, center, op):
    """engine.weights(points, center, op): the reference's per-stencil entry point.

    One target whose support is `points` and whose centre is `center` (which
    need not be a support node) goes through compute_weights, i.e. through
    the same device kernels as a whole node set; a failure surfaces as the
    engine's NumericalError (the reference raises it from the engine and
    wraps it per node only in compute_weights)."""
    from .errors import WeightError
    from .nodeset import NodeSet
    from .storage import compute_weights

    pts = np.atleast_2d(np.asarray(points, dtype=float))
    ctr = np.asarray(center, dtype=float).reshape(-1)
    n, dim = pts.shape
    if ctr.shape[0] != dim:
        raise ConfigError(f"center of dimension {ctr.shape[0]} for points of dimension {dim}")
    pos = np.concatenate([pts, ctr[None, :]], axis=0)  # node n is the centre
    nodes = NodeSet(pos, np.ones(n + 1, dtype=np.int64), stencils=[None] * n + [np.arange(n, dtype=np.int64)])
    try:
        store = compute_weights(nodes, engine, [("w", op)], for_which=np.array([n]))
    except WeightError as exc:
        text = str(exc)
        for prefix in (f"node {n}: ", "family 'w': "):
            if text.startswith(prefix):
                text = text[len(prefix):]
        raise (ConfigError if getattr(exc, "config", False) else NumericalError)(text) from None
    return np.array(store.weights("w", n), dtype=float)


class WeightedLeastSquares:
    """Weighted least squares fit over a monomial basis (engines.py:102-145).

    ``basis`` is a MonomialBasis or an int degree (the full basis of that
    degree once the dimension is known).  Runs in the general engine kernel
    (csrc/engines.cu): minimum-norm (qr / svd) or square (lu) solves of
    (W B)^T y = L b(0), w = W y.
    """

    def __init__(self, basis, weight=None, scale="nearest", solver="qr"):
        self.basis = basis
        self.weight = weight if weight is not None else ConstantWeight()
        self.scale = scale
        self.solver = solver

    def _resolve_basis(self, dim):
        if isinstance(self.basis, int):
            self.basis = MonomialBasis(dim, self.basis)
        if self.basis.dim != dim:
            raise ConfigError(
                f"basis dimension {self.basis.dim} does not match points ({dim})"
            )
        return self.basis

    def weights(self, points, center, op):
        """Weights of one stencil (engines.py:115-138), computed on the device."""
        return _single_stencil_weights(self, points, center, op)

    def __repr__(self):
        return (
            f"WeightedLeastSquares({self.basis!r}, weight={self.weight!r}, "
            f"scale={self.scale!r}, solver={self.solver!r})"
        )


class RbfFd:
    """RBF collocation with optional monomial augmentation (engines.py:147-209).

    The reference's batched configuration (Polyharmonic exponent >= 3,
    ``solver="lu"``, uniform stencils) runs in the hot shape kernels, where
    ``mode`` selects the variant (``"hybrid"``: FMA solve, conditioning-flagged
    stencils re-solved in the reference's op order; ``"replay"``: reference op
    order everywhere; ``"fast"``: FMA only).  Every other configuration (qr /
    svd solvers, Gaussian / multiquadric / inverse multiquadric kernels, r^k
    with k <= 2, composite operators) runs in the general engine kernel.
    """

    def __init__(self, rbf, degree: int = 2, scale="nearest", solver="qr", mode="hybrid"):
        self.rbf = rbf
        self.degree = int(degree)
        self.scale = scale
        self.solver = solver
        self.mode = mode

    def weights(self, points, center, op):
        """Weights of one stencil (engines.py:160-209), computed on the device."""
        return _single_stencil_weights(self, points, center, op)

    def __repr__(self):
        return (
            f"RbfFd({self.rbf!r}, degree={self.degree}, "
            f"scale={self.scale!r}, solver={self.solver!r})"
        )
