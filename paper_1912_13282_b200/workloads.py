"""Seeded synthetic node sets for the five BASELINE.json configurations.

The reference ships no data files and no public dataset exists for this
path, so these generators stand in for the benchmark inputs (SURVEY.md
§8(d)).  They are host-side numpy and are used by ``bench.py``, the tests
and ``oracle/gen_golden.py``; nothing here runs on the hot path.

C1  2D unit square, N=10,000 uniform, n=15, laplacian, u = sin(pi x) sin(pi y)
C2  unit disk minus 3 seeded holes, ~200k jittered grid, n=25, d1_0 d1_1 laplacian
C3  3D unit cube, N=1,000,000 uniform, n=35, laplacian (the metric config)
C4  2D unit square, N=1,000,000 uniform, n=15, heat stepping, Dirichlet band
C5  3D unit ball, N=4,000,000 uniform, n=70, degree 4, laplacian + gradient
"""

from __future__ import annotations

import math
import dataclasses
from dataclasses import dataclass

import numpy as np


@dataclass
class Workload:
    name: str
    positions: np.ndarray
    types: np.ndarray
    n: int
    degree: int
    families: list
    field: np.ndarray | None = None
    extra: dict = dataclasses.field(default_factory=dict)

    @property
    def N(self) -> int:
        return self.positions.shape[0]

    @property
    def dim(self) -> int:
        return self.positions.shape[1]


def _norm_rows(x):
    # np.linalg.norm(x, axis=1) as the reference's Ball.classify evaluates it
    return np.sqrt(np.add.reduce(x * x, axis=1))


def c1(N: int = 10_000) -> Workload:
    rng = np.random.default_rng(0)
    pts = rng.uniform(0.0, 1.0, (N, 2))
    u = np.sin(np.pi * pts[:, 0]) * np.sin(np.pi * pts[:, 1])
    return Workload("C1", pts, np.ones(N, dtype=np.int64), 15, 2, ["laplacian"], u)


def c2_holes(rng):
    centres, radii = [], []
    while len(centres) < 3:
        c = rng.uniform(-0.6, 0.6, 2)
        r = rng.uniform(0.1, 0.2)
        if np.linalg.norm(c) + r >= 0.9:
            continue
        if any(np.linalg.norm(c - cj) <= r + rj + 0.05 for cj, rj in zip(centres, radii)):
            continue
        centres.append(c)
        radii.append(r)
    return np.array(centres), np.array(radii)


def c2_inside(P, centres, radii):
    """Open interior of Ball([0,0],1) minus the holes (shapes.py:115-117, 224-230)."""
    keep = (_norm_rows(P) - 1.0) < 0.0
    for c, r in zip(centres, radii):
        keep &= (_norm_rows(P - c) - r) > 0.0
    return keep


def c2(target: int = 200_000) -> Workload:
    rng = np.random.default_rng(0)
    centres, radii = c2_holes(rng)
    area = math.pi * (1.0 - float(np.sum(radii**2)))
    h = math.sqrt(area / target)
    g = np.arange(-1.0 + h / 2.0, 1.0, h)
    X, Y = np.meshgrid(g, g, indexing="ij")
    P = np.stack([X.ravel(), Y.ravel()], axis=1)
    P = P + rng.uniform(-0.3 * h, 0.3 * h, P.shape)
    P = P[c2_inside(P, centres, radii)]
    u = np.random.default_rng(1).standard_normal(P.shape[0])
    return Workload("C2", np.ascontiguousarray(P), np.ones(P.shape[0], dtype=np.int64), 25, 2,
                    ["d1_0", "d1_1", "laplacian"], u,
                    {"centres": centres, "radii": radii, "h": h})


def c3(N: int = 1_000_000) -> Workload:
    rng = np.random.default_rng(0)
    pts = rng.uniform(0.0, 1.0, (N, 3))
    u = np.random.default_rng(1).standard_normal(N)
    return Workload("C3", pts, np.ones(N, dtype=np.int64), 35, 2, ["laplacian"], u)


def c4(N: int = 1_000_000, seed: int = 0) -> Workload:
    rng = np.random.default_rng(seed)
    pts = rng.uniform(0.0, 1.0, (N, 2))
    h = 1.0 / math.sqrt(N)
    edge = np.minimum(np.minimum(pts[:, 0], pts[:, 1]), np.minimum(1.0 - pts[:, 0], 1.0 - pts[:, 1]))
    types = np.where(edge < h, -1, 1).astype(np.int64)
    d = pts - 0.5
    u0 = np.exp(-50.0 * (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]))
    return Workload("C4", pts, types, 15, 2, ["laplacian"], u0,
                    {"h": h, "dt_literal": 0.1 * h * h, "steps": 1000})


def c5(N: int = 4_000_000) -> Workload:
    rng = np.random.default_rng(0)
    chunks, have = [], 0
    while have < N:
        b = rng.uniform(-1.0, 1.0, (N, 3))
        b = b[np.einsum("ij,ij->i", b, b) <= 1.0]
        chunks.append(b)
        have += b.shape[0]
    pts = np.ascontiguousarray(np.concatenate(chunks)[:N])
    u = np.random.default_rng(1).standard_normal(N)
    return Workload("C5", pts, np.ones(N, dtype=np.int64), 70, 4, ["laplacian", "gradient"], u)


CONFIGS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}


def make(name: str, **kw) -> Workload:
    return CONFIGS[name](**kw)
