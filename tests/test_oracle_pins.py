"""Pin the C oracle to golden vectors produced by the live reference.

The fixtures under tests/golden/ come from oracle/gen_golden.py calling the
reference package's public API.  The oracle must reproduce every one of them
bit-for-bit before it is trusted as the checker for the CUDA path.
"""

import numpy as np
import pytest

import oracle
from conftest import golden


def test_knn_small_cases_bitwise():
    g = golden("knn_small.npz")
    for i in range(int(g["count"])):
        pts, n = g[f"c{i}_pts"], int(g[f"c{i}_n"])
        out, _ = oracle.knn(pts, n, g[f"c{i}_targets"], g[f"c{i}_pool"])
        assert np.array_equal(out, g[f"c{i}_stencils"]), str(g[f"c{i}_name"])


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4"])
def test_config_subsets_knn_and_weights_bitwise(cfg):
    from paper_1912_13282_b200 import workloads

    g = golden(f"config_{cfg}.npz")
    w = workloads.make(cfg)
    st, _ = oracle.knn(w.positions, w.n, g["targets"])
    assert np.array_equal(st, g["stencils"])
    out, fail, keys = oracle.phs_weights(w.positions, g["targets"], st, list(w.families),
                                         degree=w.degree)
    assert not fail.any()
    assert list(keys) == list(g["families"])
    for f, key in enumerate(keys):
        assert np.array_equal(out[:, f, :], g[f"w_{key}"]), key


def test_weight_variants_bitwise():
    g = golden("weight_variants.npz")
    for name in g["names"]:
        name = str(name)
        d, N, n, k, deg = (int(x) for x in g[f"{name}_params"])
        pts = g[f"{name}_pts"]
        st, _ = oracle.knn(pts, n)
        assert np.array_equal(st, g[f"{name}_stencils"]), name
        out, fail, keys = oracle.phs_weights(pts, np.arange(N), st, list(g[f"{name}_families"]),
                                             k=k, degree=deg, scale=str(g[f"{name}_scale"]))
        assert not fail.any(), name
        assert list(keys) == [str(x) for x in g[f"{name}_keys"]]
        for f, key in enumerate(keys):
            assert np.array_equal(out[:, f, :], g[f"{name}_w_{key}"]), (name, key)


def test_weight_failures_match_reference_node():
    g = golden("weight_errors.npz")
    pts = g["scale_pts"]
    rows = np.arange(13, 50)
    st, _ = oracle.knn(pts, 5, rows)
    _, fail, _ = oracle.phs_weights(pts, rows, st, ["laplacian"], degree=1)
    bad = np.flatnonzero(fail)
    msg = str(g["scale_msg"])
    assert msg == f"node {rows[bad[0]]}: all stencil nodes coincide with the center"
    assert fail[bad[0]] == 2
    pts = g["singular_pts"]
    rows = np.arange(8)
    st, _ = oracle.knn(pts, 4, rows)
    _, fail, _ = oracle.phs_weights(pts, rows, st, ["laplacian"], degree=1)
    bad = np.flatnonzero(fail)
    msg = str(g["singular_msg"])
    assert msg == f"node {rows[bad[0]]}: singular local collocation system; try a larger stencil"
    assert fail[bad[0]] == 1


def test_csr_and_apply_bitwise():
    g = golden("csr_apply.npz")
    N = g["pts"].shape[0]
    for key in ("laplacian", "d1_0", "d1_1"):
        ip, ix, da = oracle.csr_canonical(g["rows"], g["stencils"], g[f"{key}_w"].reshape(-1, 12), N)
        assert np.array_equal(ip, g[f"{key}_indptr"])
        assert np.array_equal(ix, g[f"{key}_indices"])
        assert np.array_equal(da, g[f"{key}_data"])
        y = oracle.apply(ip, ix, da, g["u"])
        assert np.array_equal(y, g[f"{key}_y"])


def test_heat_steps_bitwise_and_instability():
    g = golden("heat.npz")
    N = g["pts"].shape[0]
    ip, ix, da = oracle.csr_canonical(np.arange(N), g["stencils"], g["w"], N)
    interior = g["types"] > 0
    diri = g["types"] == -1
    u, bad, _ = oracle.heat_steps(ip, ix, da, interior, diri, np.zeros(N), g["u0"],
                                  dt=float(g["dt"]), steps=int(g["steps"]))
    assert bad == 0
    assert np.array_equal(u, g["u_final"])
    u, bad, _ = oracle.heat_steps(ip, ix, da, interior, diri, np.full(N, 0.25), g["u0"],
                                  dt=float(g["dt"]), steps=25, diffusivity=0.7,
                                  source=np.full(N, 2.0))
    assert np.array_equal(u, g["u_final_src"])
    msg = str(g["unstable2_msg"])
    u, bad, peak = oracle.heat_steps(ip, ix, da, interior, diri, np.zeros(N), g["u0"],
                                     dt=0.5, steps=50)
    assert msg.startswith(f"step {bad}: field peak {peak:.2e} exceeds")
