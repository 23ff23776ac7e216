"""SURVEY §8f.1 against the LIVE reference (tests/golden/vector_ops.npz, made by
oracle/gen_golden.py dump_vector_ops): per-node apply / gradient / divergence /
vector_laplacian / grad_div, the explicit Neumann closure (neumann_value,
normal_combination) and run_heat_explicit with Neumann nodes
(storage.py:174-250, drivers.py:87-110), plus the whole-field and multi-family
forms (one launch over the shared stencil structure).

With the reference's own weights injected, every result is compared BITWISE
(same addend order); with the weights this package computes, within the 1e-9
normwise weight tolerance.
"""

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu

FAMS = ["laplacian", "d1_0", "d1_1", "d2_0_0", "d2_0_1", "d2_1_1"]


def m():
    import paper_1912_13282_b200 as mod

    return mod


@pytest.fixture(scope="module")
def g():
    return golden("vector_ops.npz")


def golden_store(g):
    from paper_1912_13282_b200 import _lib
    from paper_1912_13282_b200.storage import WeightStore

    N = g["pts"].shape[0]
    st_d = _lib.to_device(g["stencils"], torch.int32)
    vals = {k: _lib.to_device(g[f"w_{k}"], torch.float64) for k in FAMS}
    nodes = m().NodeSet(g["pts"], g["types"], g["normals"], stencils=list(g["stencils"]))
    return nodes, WeightStore(N, np.arange(N), st_d, vals, 15, positions_d=nodes.positions_device())


def test_weights_match_reference(g):
    nodes = m().find_closest_stencils(m().NodeSet(g["pts"], g["types"], g["normals"]), 15)
    assert np.array_equal(nodes.stencil_matrix(), g["stencils"])
    eng = m().RbfFd(m().Polyharmonic(3), degree=2, scale="support", solver="lu")
    store = m().compute_weights(nodes, eng, ["laplacian", "gradient", "hessian"])
    for k in FAMS:
        w, ref = store.values[k].reshape(ref_shape := g[f"w_{k}"].shape), g[f"w_{k}"]
        err = np.max(np.abs(w - ref), 1) / np.max(np.abs(ref), 1)
        assert err.max() <= 1e-9, (k, float(err.max()))
        y = store.apply_all(k, g["u"])
        assert np.max(np.abs(y - g[f"y_{k}"])) <= 1e-9 * np.max(np.abs(g[f"y_{k}"])), k
        assert ref_shape == (g["pts"].shape[0], 15)


def test_per_node_vector_ops_bitwise(g):
    _, store = golden_store(g)
    s = g["sample"]
    assert np.array_equal(np.array([store.apply("laplacian", g["u"], int(i)) for i in s[:20]]), g["apply_lap"][:20])
    assert np.array_equal(store.apply("laplacian", g["u"], s), g["apply_lap"])
    for k, i in enumerate(s[:25]):
        i = int(i)
        assert np.array_equal(store.gradient(g["u"], i), g["gradient"][k])
        assert store.divergence(g["vec"], i) == g["divergence"][k]
        assert np.array_equal(store.vector_laplacian(g["vec"], i), g["vector_laplacian"][k])
        assert np.array_equal(store.grad_div(g["vec"], i), g["grad_div"][k])
    # index arrays: all sampled nodes from one launch each
    assert np.array_equal(store.gradient(g["u"], s), g["gradient"])
    assert np.array_equal(store.divergence(g["vec"], s), g["divergence"])
    assert np.array_equal(store.vector_laplacian(g["vec"], s), g["vector_laplacian"])
    assert np.array_equal(store.grad_div(g["vec"], s), g["grad_div"])


def test_whole_field_forms_bitwise(g):
    _, store = golden_store(g)
    s = g["sample"]
    grad = store.gradient(g["u"])
    assert grad.shape == (g["pts"].shape[0], 2)
    assert np.array_equal(grad[s], g["gradient"])
    assert np.array_equal(store.divergence(g["vec"])[s], g["divergence"])
    assert np.array_equal(store.vector_laplacian(g["vec"])[s], g["vector_laplacian"])
    assert np.array_equal(store.grad_div(g["vec"])[s], g["grad_div"])
    many = store.apply_families(FAMS, g["u"])
    for k in FAMS:
        assert np.array_equal(many[k], g[f"y_{k}"]), k
    # device fields in, device tensors out
    u_d = torch.from_numpy(g["u"]).cuda()
    vec_d = torch.from_numpy(np.ascontiguousarray(g["vec"])).cuda()
    assert torch.equal(store.gradient(u_d).cpu(), torch.from_numpy(grad))
    assert np.array_equal(store.divergence(vec_d).cpu().numpy()[s], g["divergence"])


def test_neumann_closure_bitwise(g):
    _, store = golden_store(g)
    bnd, gn = g["neumann_nodes"], g["neumann_gn"]
    normals = g["normals"]
    for k in range(40):
        i = int(bnd[k])
        assert np.array_equal(store.normal_combination(i, normals[i]), g["normal_comb"][k])
        assert store.neumann_value(g["u"], i, normals[i], float(gn[k])) == g["neumann_values"][k]


def test_heat_with_neumann_bitwise(g):
    nodes, store = golden_store(g)
    dt = float(g["heat_dt"])
    u = m().run_heat_explicit(nodes, store, dt=dt, steps=30, dirichlet={-1: 0.0}, neumann={-2: 0.3},
                              initial=g["heat_u0"])
    assert np.array_equal(u, g["heat_neumann"])
    u2 = m().run_heat_explicit(nodes, store, dt=dt, steps=20, diffusivity=0.5,
                               dirichlet={-1: lambda p, t: p[:, 0] * (1.0 + t)},
                               neumann={-2: lambda p, t: p[:, 1] + t}, initial=g["heat_u0"])
    assert np.array_equal(u2, g["heat_neumann_fn"])


def test_vector_ops_errors(g):
    _, store = golden_store(g)
    lap_only = store.__class__(store.n_nodes, store.rows, store.stencils_device,
                               {"laplacian": store.values_device("laplacian")}, 15)
    with pytest.raises(m().StorageError, match="first-derivative"):
        lap_only.gradient(g["u"], 3)
    with pytest.raises(m().StorageError, match="not stored"):
        lap_only.apply("d1_0", g["u"], 3)
