"""The kNN fast passes (knn_fast in csrc/knn.cu) against the oracle, bit for bit,
on inputs built to exercise their hand-back paths: clustered node sets (the
cube proof fails near density jumps, so rows go to the wider second pass and
to the general kernel), exact ties on lattices (equal d2 high words collide in
the 32-bit ranks and are re-counted on the full key), coincident nodes, and
target / pool subsets.  The oracle is the C restatement of
find_closest_stencils (stencils.py:19-93), pinned to the reference's goldens
in test_oracle_pins.py.
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def mf():
    import paper_1912_13282_b200 as m

    return m


def clustered(N, d, seed):
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.2, 0.8, (6, d))
    widths = rng.uniform(0.01, 0.08, 6)
    k = rng.integers(0, 6, N)
    pts = centres[k] + widths[k, None] * rng.standard_normal((N, d))
    bg = rng.uniform(0, 1, (N // 5, d))  # sparse background between the clusters
    return np.concatenate([pts, bg])


def check(pts, n, for_which=None, search_among=None):
    m = mf()
    N = pts.shape[0]
    nodes = m.NodeSet(pts, np.ones(N, dtype=np.int64))
    out = m.find_closest_stencils(nodes, n, for_which=for_which, search_among=search_among)
    targets = np.arange(N) if for_which is None else np.asarray(for_which)
    got = np.stack([out.stencil(int(t)) for t in targets])
    ref, _ = oracle.knn(pts, n, targets=targets, pool=search_among)
    bad = np.flatnonzero(np.any(got != ref, axis=1))
    assert bad.size == 0, f"{bad.size} rows differ, first target {targets[bad[0]]}"


@pytest.mark.parametrize("d,n", [(3, 35), (2, 15), (2, 25), (3, 20), (3, 70)])
def test_clustered_bitwise(d, n):
    check(clustered(40_000, d, seed=d * 100 + n), n)


@pytest.mark.parametrize("d,n", [(3, 35), (2, 15)])
def test_lattice_ties_bitwise(d, n):
    g = np.arange(14 if d == 3 else 60, dtype=np.float64)
    pts = np.stack(np.meshgrid(*([g] * d), indexing="ij"), -1).reshape(-1, d)
    check(pts, n)


def test_coincident_nodes_bitwise():
    rng = np.random.default_rng(7)
    base = rng.uniform(0, 1, (6000, 3))
    pts = np.concatenate([base, base[:1500], base[:300]])  # double and triple points
    check(pts, 35)


def test_target_and_pool_subsets_bitwise():
    rng = np.random.default_rng(11)
    pts = rng.uniform(0, 1, (30_000, 3))
    targets = rng.choice(30_000, 5000, replace=False)
    pool = np.sort(rng.choice(30_000, 20_000, replace=False))
    check(pts, 35, for_which=targets, search_among=pool)


def test_wide_k_uniform_and_subsets_bitwise():
    """K = n + 8 = 78 (C5's stencil size): the wide fast passes (coarser grid,
    128 ranked survivors) on a box-filling cloud."""
    rng = np.random.default_rng(13)
    pts = rng.uniform(-1, 1, (40_000, 3))
    check(pts, 70)
    targets = rng.choice(40_000, 3000, replace=False)
    pool = np.sort(rng.choice(40_000, 30_000, replace=False))
    check(pts, 70, for_which=targets, search_among=pool)


@pytest.mark.parametrize("n", [49, 70, 104, 105])
def test_wide_k_ball_clustered_and_ties_bitwise(n):
    """Wide stencils (56 < K <= 112 take the wide fast passes, K = 113 the general
    kernel) on clouds that do not fill their bounding box (the grid is refit to
    the occupied cells), on a clustered cloud and on lattice ties."""
    rng = np.random.default_rng(17 + n)
    p = rng.uniform(-1, 1, (90_000, 3))
    ball = p[np.sum(p * p, axis=1) <= 1.0][:40_000]
    check(ball, n)
    check(clustered(30_000, 3, seed=n), n)
    g = np.arange(16, dtype=np.float64)
    check(np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3), n)


@pytest.mark.parametrize("N,n", [(80, 70), (75, 70), (71, 70), (200, 104), (5000, 57)])
def test_wide_k_small_pools_bitwise(N, n):
    """Wide stencils on pools barely larger than the stencil (K = min(n + 8, P): the
    candidate cube is the whole grid) and at the K = 57 switch-over."""
    rng = np.random.default_rng(N + n)
    check(rng.uniform(0, 1, (N, 3)), n)
    check(rng.standard_normal((N, 3)) * np.array([1.0, 0.01, 5.0]), n)  # anisotropic cloud
