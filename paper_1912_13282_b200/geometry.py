"""Node generation: fill_interior with its acceptance pass on the GPU.

Restates the membership part of the reference's geometry package that
``fill_interior`` needs (geometry/shapes.py:28-242: Ball, Box, union,
difference; closed / open membership; bounding boxes) and its spacing
functions (geometry/spacing.py), and runs ``fill_interior``
(geometry/fill.py:204-298) with the same queue semantics: generation by
generation, candidates drawn from numpy's generator in the reference's order
and shape / spacing evaluated on the host exactly as the reference does, the
order-dependent acceptance pass (fill.py:38-117, the hot spot) on the device
(``mf_fill_accept``).  The accepted node set is the reference's, bitwise:
same candidates, same distance arithmetic, same greedy order.

Any object with ``dim``, ``classify`` / ``contains`` / ``interior_contains``
and ``bounding_box`` works as a shape (the reference's own shape objects
included).  Boundary discretisation (``discretize_boundary``) is not part of
this package; seed nodes come from ``nodes`` or ``start``.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import GeometryError

IN = 1
SURF = 0
OUT = -1


class Shape:
    """Base class: membership classification and bounding box (shapes.py:28-95)."""

    dim: int
    tag: int = -1

    def classify(self, points, tol: float = 0.0):
        raise NotImplementedError

    def contains(self, points):
        """Closed membership test."""
        return self.classify(self._batch(points)) != OUT

    def interior_contains(self, points):
        """Open membership test (strict interior)."""
        return self.classify(self._batch(points)) == IN

    def _batch(self, points):
        points = np.asarray(points, dtype=float)
        if points.ndim == 1:
            points = points[None, :]
        if points.shape[1] != self.dim:
            raise GeometryError(f"points have dimension {points.shape[1]}, shape has {self.dim}")
        return points

    def bounding_box(self):
        raise NotImplementedError

    def diameter(self) -> float:
        """Diagonal of the bounding box (shapes.py:68-70)."""
        lo, hi = self.bounding_box()
        return float(np.sqrt(np.sum((np.asarray(hi) - np.asarray(lo)) ** 2)))

    def __or__(self, other):
        return ShapeUnion(self, other)

    def __sub__(self, other):
        return ShapeDifference(self, other)

    def translate(self, offset):
        return Translated(self, offset)

    def rotate(self, matrix):
        return Rotated(self, matrix)


class Ball(Shape):
    """Closed ball (shapes.py:98-137)."""

    def __init__(self, center, radius: float, tag: int = -1):
        self.center = np.atleast_1d(np.asarray(center, dtype=float))
        self.radius = float(radius)
        if self.radius <= 0:
            raise GeometryError(f"ball radius must be positive, got {radius}")
        if tag >= 0:
            raise GeometryError("boundary tags must be negative")
        self.tag = tag
        self.dim = self.center.shape[0]

    def classify(self, points, tol=0.0):
        t = np.linalg.norm(points - self.center, axis=1) - self.radius
        return np.where(t > tol, OUT, np.where(t < -tol, IN, SURF)).astype(np.int8)

    def bounding_box(self):
        return self.center - self.radius, self.center + self.radius

    def __repr__(self):
        return f"Ball({self.center.tolist()}, {self.radius}, tag={self.tag})"


class Box(Shape):
    """Closed axis-aligned box (shapes.py:140-179)."""

    def __init__(self, lo, hi, tag: int = -1):
        self.lo = np.atleast_1d(np.asarray(lo, dtype=float))
        self.hi = np.atleast_1d(np.asarray(hi, dtype=float))
        if self.lo.shape != self.hi.shape:
            raise GeometryError("box corners must have equal dimension")
        if np.any(self.hi <= self.lo):
            raise GeometryError("box needs hi > lo in every axis")
        if tag >= 0:
            raise GeometryError("boundary tags must be negative")
        self.tag = tag
        self.dim = self.lo.shape[0]

    def classify(self, points, tol=0.0):
        m = np.minimum((points - self.lo).min(axis=1), (self.hi - points).min(axis=1))
        return np.where(m < -tol, OUT, np.where(m > tol, IN, SURF)).astype(np.int8)

    def bounding_box(self):
        return self.lo.copy(), self.hi.copy()

    def __repr__(self):
        return f"Box({self.lo.tolist()}, {self.hi.tolist()}, tag={self.tag})"


class ShapeUnion(Shape):
    def __init__(self, a, b):
        if a.dim != b.dim:
            raise GeometryError("cannot combine shapes of different dimension")
        self.a, self.b = a, b
        self.dim = a.dim

    def classify(self, points, tol=0.0):
        ca = self.a.classify(points, tol)
        cb = self.b.classify(points, tol)
        out = np.full(points.shape[0], SURF, dtype=np.int8)
        out[(ca == IN) | (cb == IN)] = IN
        out[(ca == OUT) & (cb == OUT)] = OUT
        return out

    def bounding_box(self):
        alo, ahi = self.a.bounding_box()
        blo, bhi = self.b.bounding_box()
        return np.minimum(alo, blo), np.maximum(ahi, bhi)

    def __repr__(self):
        return f"({self.a!r} | {self.b!r})"


class ShapeDifference(Shape):
    """Points of ``a`` not in the open interior of ``b`` (shapes.py:211-241)."""

    def __init__(self, a, b):
        if a.dim != b.dim:
            raise GeometryError("cannot combine shapes of different dimension")
        self.a, self.b = a, b
        self.dim = a.dim

    def classify(self, points, tol=0.0):
        ca = self.a.classify(points, tol)
        cb = self.b.classify(points, tol)
        out = np.full(points.shape[0], SURF, dtype=np.int8)
        out[(ca == IN) & (cb == OUT)] = IN
        out[(ca == OUT) | (cb == IN)] = OUT
        return out

    def bounding_box(self):
        return self.a.bounding_box()

    def __repr__(self):
        return f"({self.a!r} - {self.b!r})"


# -- spacing (geometry/spacing.py) ------------------------------------------------

class Translated(Shape):
    """Membership of a shape moved by `offset` (shapes.py:243-257): x is classified as x - offset."""

    def __init__(self, inner, offset):
        self.inner = inner
        self.offset = np.atleast_1d(np.asarray(offset, dtype=float))
        if self.offset.shape[0] != inner.dim:
            raise GeometryError("offset dimension does not match shape")
        self.dim = inner.dim
        self.tag = getattr(inner, "tag", -1)

    def classify(self, points, tol: float = 0.0):
        return self.inner.classify(np.asarray(points, dtype=float) - self.offset, tol)

    def bounding_box(self):
        lo, hi = self.inner.bounding_box()
        return lo + self.offset, hi + self.offset

    def __repr__(self):
        return f"{self.inner!r}.translate({self.offset.tolist()})"


class Rotated(Shape):
    """Membership of a shape rotated about the origin by an orthogonal matrix R
    (shapes.py:270-290): x = R y lies in the rotated shape iff y = R^T x lies in the original."""

    def __init__(self, inner, matrix):
        self.inner = inner
        self.matrix = np.asarray(matrix, dtype=float)
        d = inner.dim
        if self.matrix.shape != (d, d):
            raise GeometryError(f"rotation matrix must be {d}x{d}")
        if not np.allclose(self.matrix @ self.matrix.T, np.eye(d), atol=1e-12):
            raise GeometryError("rotation matrix must be orthogonal")
        self.dim = d
        self.tag = getattr(inner, "tag", -1)

    def classify(self, points, tol: float = 0.0):
        return self.inner.classify(np.asarray(points, dtype=float) @ self.matrix, tol)

    def bounding_box(self):
        lo, hi = self.inner.bounding_box()
        corners = np.stack(np.meshgrid(*[(a, b) for a, b in zip(lo, hi)], indexing="ij"), axis=-1).reshape(-1, self.dim)
        turned = corners @ self.matrix.T
        return turned.min(axis=0), turned.max(axis=0)

    def __repr__(self):
        return f"{self.inner!r}.rotate(...)"


class ConstantSpacing:
    def __init__(self, value: float):
        self.value = float(value)
        if not self.value > 0:
            raise GeometryError(f"spacing must be positive, got {value}")

    def __call__(self, points):
        points = np.atleast_2d(np.asarray(points, dtype=float))
        return np.full(points.shape[0], self.value)

    def __repr__(self):
        return f"ConstantSpacing({self.value})"


class LinearSpacing:
    """Affine spacing h(p) = base + gradient . p."""

    def __init__(self, base: float, gradient):
        self.base = float(base)
        self.gradient = np.asarray(gradient, dtype=float)

    def __call__(self, points):
        points = np.atleast_2d(np.asarray(points, dtype=float))
        h = self.base + points @ self.gradient
        if np.any(h <= 0):
            raise GeometryError("spacing function is non-positive inside the domain")
        return h

    def __repr__(self):
        return f"LinearSpacing({self.base}, {self.gradient.tolist()})"


def as_spacing(h):
    """Coerce a float or callable into a spacing function."""
    if callable(h):
        return h
    return ConstantSpacing(h)


# -- fill ------------------------------------------------------------------------

def _estimate_h_range(shape, h, seeds):
    lo, hi = shape.bounding_box()
    d = lo.shape[0]
    axes = [np.linspace(lo[a], hi[a], 9) for a in range(d)]
    mesh = np.meshgrid(*axes, indexing="ij")
    probes = np.stack([m.ravel() for m in mesh], axis=1)
    inside = shape.contains(probes)
    pts = probes[inside]
    if seeds.shape[0]:
        pts = np.concatenate([pts, seeds], axis=0) if pts.shape[0] else seeds
    if pts.shape[0] == 0:
        pts = 0.5 * (lo + hi)[None, :]
    vals = h(pts)
    return float(np.min(vals)), float(np.max(vals))


def _candidate_directions(rng, m, k, d):
    """(m, k, d) unit vectors, uniform on the sphere (fill.py:175-186)."""
    if d == 1:
        return np.where(rng.random((m, k, 1)) < 0.5, -1.0, 1.0)
    if d == 2:
        theta = 2.0 * np.pi * rng.random((m, k))
        return np.stack([np.cos(theta), np.sin(theta)], axis=2)
    g = rng.standard_normal((m, k, d))
    norms = np.linalg.norm(g, axis=2, keepdims=True)
    norms[norms == 0] = 1.0
    return g / norms


MAX_GRID_CELLS = 1 << 26


class _DeviceFill:
    """Device node arrays + cell grid of one fill, grown on demand."""

    def __init__(self, seeds, hv_seeds, lo, hi, cell, cap):
        self.d = seeds.shape[1]
        dev = _lib.device()
        self.grid = _lib.FillGridT()
        dims = []
        for a in range(3):
            if a < self.d:
                span = float(hi[a] - lo[a])
                n = int(np.ceil(span / cell)) + 3
                self.grid.lo[a] = float(lo[a]) - cell
                dims.append(n)
            else:
                self.grid.lo[a] = 0.0
                dims.append(1)
        ncell = int(np.prod(dims))
        if ncell > MAX_GRID_CELLS:
            raise GeometryError(f"fill grid of {ncell} cells is too fine for the device (cell {cell:g})")
        for a in range(3):
            self.grid.dims[a] = dims[a]
        self.grid.cell = float(cell)
        self.grid.d = self.d
        self.head = torch.full((ncell,), -1, dtype=torch.int32, device=dev)
        self.head2 = torch.full((ncell,), -1, dtype=torch.int32, device=dev)
        self.cap = int(cap)
        self.pos = torch.empty((self.cap, self.d), dtype=torch.float64, device=dev)
        self.hv = torch.empty(self.cap, dtype=torch.float64, device=dev)
        self.nxt = torch.empty(self.cap, dtype=torch.int32, device=dev)
        n = seeds.shape[0]
        self.pos[:n] = _lib.to_device(seeds, torch.float64)
        self.hv[:n] = _lib.to_device(hv_seeds, torch.float64)
        _lib.check(_lib.load().mf_fill_insert(self.pos.data_ptr(), 0, n, ctypes.byref(self.grid),
                                              self.head.data_ptr(), self.nxt.data_ptr(), _lib.stream_ptr()),
                   "mf_fill_insert")
        self.rounds = []

    def grow(self, need):
        new_cap = max(need, 2 * self.cap)
        for name in ("pos", "hv", "nxt"):
            old = getattr(self, name)
            t = torch.empty((new_cap,) + tuple(old.shape[1:]), dtype=old.dtype, device=old.device)
            t[: self.cap] = old
            setattr(self, name, t)
        self.cap = new_cap

    def accept(self, count, cand, hc, gamma):
        """Accepted candidate indices (in order); they are appended at count.."""
        lib = _lib.load()
        M = cand.shape[0]
        if count + M > self.cap:
            self.grow(count + M)
        cand_d = _lib.to_device(cand, torch.float64)
        hc_d = _lib.to_device(hc, torch.float64)
        acc = torch.empty(max(M, 1), dtype=torch.int32, device=cand_d.device)
        size = ctypes.c_size_t(0)
        _lib.check(lib.mf_fill_workspace_size(M, ctypes.byref(size)), "mf_fill_workspace_size")
        ws = _lib.workspace(size.value)
        na = ctypes.c_int64(0)
        rounds = ctypes.c_int32(0)
        _lib.check(lib.mf_fill_accept(self.pos.data_ptr(), self.hv.data_ptr(), self.nxt.data_ptr(), count, self.cap,
                                      ctypes.byref(self.grid), self.head.data_ptr(), self.head2.data_ptr(),
                                      cand_d.data_ptr(), hc_d.data_ptr(), M, float(gamma), acc.data_ptr(),
                                      ctypes.byref(na), ctypes.byref(rounds), ws.data_ptr(), size.value,
                                      _lib.stream_ptr()), "mf_fill_accept")
        self.rounds.append(int(rounds.value))
        return acc[: na.value].cpu().numpy()


@_lib.traced("meshfree.fill_interior")
def fill_interior(nodes, shape, h, seed: int = 0, *, interior_tag: int = 1, gamma: float = 0.75,
                  n_candidates: int = 15, start=None, max_nodes: int = 4_000_000):
    """Fill the interior of ``shape`` with nodes spaced by ``h`` (fill.py:204-298).

    All nodes already in ``nodes`` act as queue seeds and as blockers for the
    minimum-distance test; ``start`` supplies interior seed points when
    ``nodes`` is empty.  Returns a new NodeSet with the accepted interior
    nodes appended, tagged ``interior_tag`` -- the reference's nodes, bitwise.
    """
    h = as_spacing(h)
    d = shape.dim
    if len(nodes) and nodes.dim != d:
        raise GeometryError("node set and shape dimensions differ")
    if gamma <= 0 or gamma >= 1.5:
        raise GeometryError(f"gamma out of range: {gamma}")

    seeds = nodes.positions
    extra = 0
    if start is not None:
        start = np.atleast_2d(np.asarray(start, dtype=float))
        if not np.all(shape.interior_contains(start)):
            raise GeometryError("start points must lie strictly inside the shape")
        seeds = np.concatenate([seeds, start], axis=0) if seeds.size else start
        extra = start.shape[0]
    n_seed = seeds.shape[0]
    if n_seed == 0:
        raise GeometryError("fill needs seed nodes: a boundary discretization or start points")

    h_min, h_max = _estimate_h_range(shape, h, seeds)
    cell = gamma * h_max * 1.0001
    lo, hi = shape.bounding_box()
    lo = np.minimum(lo, seeds.min(axis=0))
    hi = np.maximum(hi, seeds.max(axis=0))
    vol = float(np.prod(hi - lo))
    est = int(vol / max(h_min, 1e-300) ** d * 3.0) + n_seed + 1024
    cap = min(max(n_seed + 1024, est), max_nodes + 1024)

    hv_seeds = np.asarray(h(seeds), dtype=float)
    pos = np.empty((cap, d))
    hv = np.empty(cap)
    pos[:n_seed] = seeds
    hv[:n_seed] = hv_seeds
    dev = _DeviceFill(seeds, hv_seeds, lo, hi, cell, cap)
    count = n_seed
    rng = np.random.default_rng(seed)
    proc = 0
    while proc < count:
        m = count - proc
        parents = pos[proc:count]
        radii = hv[proc:count]
        dirs = _candidate_directions(rng, m, n_candidates, d)
        cand = (parents[:, None, :] + radii[:, None, None] * dirs).reshape(-1, d)
        inside = shape.interior_contains(cand)
        cand = np.ascontiguousarray(cand[inside])
        proc = count
        if cand.shape[0] == 0:
            continue
        hc = np.ascontiguousarray(h(cand), dtype=float)
        acc = dev.accept(count, cand, hc, gamma)
        k = acc.shape[0]
        limit = max_nodes - count
        if k >= limit:
            # the reference fails once its count reaches max_nodes with candidates
            # of the generation still unprocessed (fill.py:281-285)
            if limit <= 0 or k > limit or acc[limit - 1] < cand.shape[0] - 1:
                raise GeometryError(f"fill exceeded max_nodes={max_nodes}; spacing too small for the shape")
        if count + k > pos.shape[0]:
            grow = max(count + k, 2 * pos.shape[0])
            pos = np.concatenate([pos, np.empty((grow - pos.shape[0], d))], axis=0)
            hv = np.concatenate([hv, np.empty(grow - hv.shape[0])])
        pos[count:count + k] = cand[acc]
        hv[count:count + k] = hc[acc]
        count += k
    new_pts = pos[n_seed:count]
    if extra:
        new_pts = np.concatenate([seeds[n_seed - extra:], new_pts], axis=0)
    out = nodes.append(new_pts, interior_tag) if new_pts.shape[0] else nodes
    out.fill_rounds = dev.rounds  # diagnostics: resolution rounds per generation
    return out
