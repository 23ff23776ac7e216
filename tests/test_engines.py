"""the engines the reference runs through its per-node loop
(storage.py:325-339) -- qr / svd solvers (qr is the reference's default),
Gaussian / multiquadric / inverse multiquadric / r^k (k <= 2) kernels,
WeightedLeastSquares (constant and Gaussian weights, explicit exponent
lists, square / wide / tall systems), composite operators -- against the LIVE
reference (tests/golden/engines.npz, oracle/gen_golden.py dump_engines).

Weights: per stencil and family max_j |w - w_ref| / max_j |w_ref| <= 1e-9 (the
reference's own solvers differ from each other by rounding; the GPU solves the
same system with its own factorisation).  Errors: the same WeightError text
(lowest failing node, first failing family, the engine's message).
"""

import json
import os

import numpy as np
import pytest

from conftest import REPO, golden

pytestmark = pytest.mark.gpu

import sys  # noqa: E402

sys.path.insert(0, os.path.join(REPO, "oracle"))
from gen_golden_specs import ENGINE_ERRORS, ENGINE_VARIANTS, family_specs  # noqa: E402

TOL = 1e-9


def m():
    import paper_1912_13282_b200 as mod

    return mod


@pytest.fixture(scope="module")
def g():
    return golden("engines.npz")


RESULTS = {}


@pytest.mark.parametrize("variant", ENGINE_VARIANTS, ids=[v[0] for v in ENGINE_VARIANTS])
def test_engine_weights_match_reference(g, variant):
    name, d, N, n, eng_expr, fams = variant
    mod = m()
    pts = g[f"{name}_pts"]
    nodes = mod.find_closest_stencils(mod.NodeSet(pts, np.ones(N, dtype=np.int64)), n)
    assert np.array_equal(nodes.stencil_matrix(), g[f"{name}_stencils"])
    eng = eval(eng_expr, vars(mod))
    store = mod.compute_weights(nodes, eng, family_specs(mod, fams))
    assert list(store.families) == list(g[f"{name}_keys"])
    worst = {}
    for k in store.families:
        ref = g[f"{name}_w_{k}"]
        w = store.values[k].reshape(ref.shape)
        err = np.max(np.abs(w - ref), 1) / np.max(np.abs(ref), 1)
        worst[k] = float(err.max())
    RESULTS[name] = worst
    assert max(worst.values()) <= TOL, worst


@pytest.mark.parametrize("case", ENGINE_ERRORS, ids=[v[0] for v in ENGINE_ERRORS])
def test_engine_errors_match_reference(g, case):
    name, d, N, n, eng_expr, fams, mutate = case
    mod = m()
    pts = g[f"err_{name}_pts"]
    nodes = mod.find_closest_stencils(mod.NodeSet(pts, np.ones(N, dtype=np.int64)), n)
    with pytest.raises(mod.WeightError) as exc:
        mod.compute_weights(nodes, eval(eng_expr, vars(mod)), family_specs(mod, fams))
    assert str(exc.value) == str(g[f"err_{name}_msg"])


def test_engine_records():
    """Write the per-variant worst errors (run after the parity cases)."""
    if RESULTS:
        out = os.path.join(REPO, "gpurun_out")
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "engines_parity.json"), "w") as fh:
            json.dump(RESULTS, fh, indent=1, sort_keys=True)


def test_python_defined_pieces_raise_config_error():
    """A user kernel / weight / operator class has no GPU implementation."""
    mod = m()
    pts = np.random.default_rng(3).uniform(0, 1, (100, 2))
    nodes = mod.find_closest_stencils(mod.NodeSet(pts, np.ones(100, dtype=np.int64)), 9)

    class MyKernel:
        pass

    class MyOp(mod.Operator):
        order = 1

    with pytest.raises(mod.ConfigError):
        mod.compute_weights(nodes, mod.RbfFd(MyKernel(), degree=1), ["laplacian"])
    with pytest.raises(mod.ConfigError):
        mod.compute_weights(nodes, mod.RbfFd(mod.Polyharmonic(3), degree=1), [("mine", MyOp())])
    with pytest.raises(mod.ConfigError):
        mod.compute_weights(nodes, mod.WeightedLeastSquares(1, weight=lambda x: 1.0), ["laplacian"])
