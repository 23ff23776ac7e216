"""SURVEY §8f.4, node generation: fill_interior with the acceptance pass on the
GPU, against the LIVE reference (tests/golden/fill.npz, oracle/gen_golden.py
dump_fill): 1D / 2D / 3D shapes (ball, box, ball minus ball), constant and
linear spacing, boundary seeds and start points, gamma / n_candidates / seed
variations.  The accepted node set is compared BITWISE (positions and
types, in the reference's order); errors by class and text.
"""

import os
import sys

import numpy as np
import pytest

from conftest import REPO, golden

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(REPO, "oracle"))
from gen_golden_specs import FILL_CASES, fill_seeds  # noqa: E402


def m():
    import paper_1912_13282_b200 as mod

    return mod


@pytest.fixture(scope="module")
def g():
    return golden("fill.npz")


@pytest.mark.parametrize("case", FILL_CASES, ids=[c[0] for c in FILL_CASES])
def test_fill_matches_reference_bitwise(g, case):
    from paper_1912_13282_b200 import geometry

    name, shape_expr, h_expr, seeds_kind, kw = case
    mod = m()
    ns = vars(geometry)
    shape = eval(shape_expr, ns)
    h = eval(h_expr, ns)
    seeds = fill_seeds(seeds_kind)
    d = shape.dim
    nodes = mod.NodeSet(seeds, -np.ones(seeds.shape[0], dtype=np.int64)) if seeds is not None else \
        mod.NodeSet(np.empty((0, d)), np.empty(0, dtype=np.int64))
    kw = dict(kw)
    seed = kw.pop("seed", 0)
    out = mod.fill_interior(nodes, shape, h, seed, **kw)
    ref = g[f"{name}_positions"]
    assert out.positions.shape == ref.shape, (out.positions.shape, ref.shape)
    assert np.array_equal(out.positions, ref)
    assert np.array_equal(out.types, g[f"{name}_types"])


def test_fill_errors_match_reference(g):
    mod = m()
    disk = mod.Ball([0.0, 0.0], 1.0)
    empty = mod.NodeSet(np.empty((0, 2)), np.empty(0, dtype=np.int64))
    cases = {
        "gamma": lambda: mod.fill_interior(empty, disk, 0.1, start=[[0, 0]], gamma=1.6),
        "start_outside": lambda: mod.fill_interior(empty, disk, 0.1, start=[[2.0, 0.0]]),
        "no_seeds": lambda: mod.fill_interior(empty, disk, 0.1),
        "max_nodes": lambda: mod.fill_interior(empty, disk, 0.02, start=[[0, 0]], max_nodes=500),
        "dims": lambda: mod.fill_interior(mod.NodeSet(np.zeros((1, 3)), np.ones(1, dtype=np.int64)), disk, 0.1),
    }
    want = dict(zip([str(k) for k in g["err_keys"]], [str(v) for v in g["err_msgs"]]))
    for key, fn in cases.items():
        try:
            fn()
            got = ""
        except Exception as exc:  # noqa: BLE001
            got = f"{type(exc).__name__}: {exc}"
        assert got == want[key], (key, got, want[key])
