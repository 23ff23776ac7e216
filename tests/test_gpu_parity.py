"""CUDA path vs the golden vectors of the live reference and vs the pinned oracle.

Bars (BASELINE.json north star): neighbour indices and CSR structure bitwise;
weights and operator outputs within 1e-9 normwise (per stencil and family:
max_j |w - w_ref| / max_j |w_ref|); apply and heat stepping bitwise given the
same weights.
"""

import numpy as np
import pytest

import oracle
from conftest import golden

pytestmark = pytest.mark.gpu

WEIGHT_TOL = 1e-9


def mf():
    import paper_1912_13282_b200 as m

    return m


def normwise(w, ref):
    w = w.reshape(ref.shape[0], -1)
    ref = ref.reshape(ref.shape[0], -1)
    den = np.max(np.abs(ref), axis=1)
    return np.max(np.abs(w - ref), axis=1) / np.where(den > 0, den, 1.0)


# ---------------------------------------------------------------------------
# stencils
# ---------------------------------------------------------------------------

def test_knn_small_goldens_bitwise():
    m = mf()
    g = golden("knn_small.npz")
    for i in range(int(g["count"])):
        nodes = m.NodeSet(g[f"c{i}_pts"], g[f"c{i}_types"])
        tg, pool = g[f"c{i}_targets"], g[f"c{i}_pool"]
        out = m.find_closest_stencils(nodes, int(g[f"c{i}_n"]), for_which=tg, search_among=pool)
        got = np.stack([out.stencil(int(t)) for t in tg])
        assert np.array_equal(got, g[f"c{i}_stencils"]), str(g[f"c{i}_name"])


def test_knn_reference_test_cases():
    """Assertions of the reference's tests/test_stencils.py on the GPU path."""
    m = mf()
    g = np.stack(np.meshgrid(np.arange(5.0), np.arange(5.0), indexing="ij"), axis=-1)
    nodes = m.NodeSet(g.reshape(-1, 2), np.ones(25, dtype=np.int64))
    out = m.find_closest_stencils(nodes, 4)
    assert out.stencil(12).tolist() == [12, 7, 11, 13]
    rng = np.random.default_rng(3)
    nodes = m.NodeSet(rng.uniform(-1, 1, (40, 3)), np.ones(40, dtype=np.int64))
    out = m.find_closest_stencils(nodes, 5)
    assert all(out.stencil(i)[0] == i for i in range(40))
    types = np.ones(30, dtype=np.int64)
    types[:6] = -1
    nodes = m.NodeSet(np.random.default_rng(1).uniform(-1, 1, (30, 2)), types)
    out = m.find_closest_stencils(nodes, 4, for_which="interior")
    assert all(out.has_stencil(i) for i in range(6, 30))
    assert not any(out.has_stencil(i) for i in range(6))
    with pytest.raises(m.StencilError):
        m.find_closest_stencils(nodes, 31)
    with pytest.raises(m.StencilError):
        m.find_closest_stencils(nodes, 0)


@pytest.mark.parametrize("seed", range(12))
def test_knn_property_vs_oracle(seed):
    m = mf()
    rng = np.random.default_rng(seed)
    d = 1 + seed % 3
    N = int(rng.integers(20, 400))
    n = int(rng.integers(1, min(N, 40)))
    if seed % 4 == 0:
        pts = np.round(rng.uniform(0, 6, (N, d)))  # heavy exact ties
    else:
        pts = rng.uniform(-1, 1, (N, d))
    nodes = m.find_closest_stencils(m.NodeSet(pts, np.ones(N, dtype=np.int64)), n)
    ref, _ = oracle.knn(pts, n)
    assert np.array_equal(nodes.stencil_matrix(), ref)


# ---------------------------------------------------------------------------
# weights
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4", "C5"])
@pytest.mark.parametrize("mode", ["replay", "hybrid"])
def test_config_subset_knn_and_weights(cfg, mode):
    m = mf()
    from paper_1912_13282_b200 import workloads

    g = golden(f"config_{cfg}.npz")
    w = workloads.make(cfg)
    nodes = m.NodeSet(w.positions, w.types)
    nodes = m.find_closest_stencils(nodes, w.n, for_which=g["targets"])
    st = np.stack([nodes.stencil(int(t)) for t in g["targets"]])
    assert np.array_equal(st, g["stencils"])
    eng = m.RbfFd(m.Polyharmonic(3), degree=w.degree, scale="support", solver="lu", mode=mode)
    store = m.compute_weights(nodes, eng, w.families, for_which=g["targets"])
    assert store.families == [str(f) for f in g["families"]]
    for key in store.families:
        err = normwise(store.values[key], g[f"w_{key}"])
        assert err.max() <= WEIGHT_TOL, (cfg, key, float(err.max()))
        if mode == "replay":
            # correctly rounded r^3 vs glibc pow differ in ~0.1% of entries
            assert err.max() <= 1e-11, (cfg, key, float(err.max()))


@pytest.mark.parametrize("mode", ["replay", "hybrid", "fast"])
def test_weight_variants(mode):
    m = mf()
    g = golden("weight_variants.npz")
    for name in g["names"]:
        name = str(name)
        d, N, n, k, deg = (int(x) for x in g[f"{name}_params"])
        pts = g[f"{name}_pts"]
        nodes = m.find_closest_stencils(m.NodeSet(pts, np.ones(N, dtype=np.int64)), n)
        assert np.array_equal(nodes.stencil_matrix(), g[f"{name}_stencils"]), name
        eng = m.RbfFd(m.Polyharmonic(k), degree=deg, scale=str(g[f"{name}_scale"]), solver="lu", mode=mode)
        store = m.compute_weights(nodes, eng, [str(f) for f in g[f"{name}_families"]])
        for key in store.families:
            err = normwise(store.values[key], g[f"{name}_w_{key}"])
            tol = WEIGHT_TOL if mode != "fast" else 1e-7
            assert err.max() <= tol, (name, key, float(err.max()))


def test_weight_error_messages():
    m = mf()
    g = golden("weight_errors.npz")
    eng = m.RbfFd(m.Polyharmonic(3), degree=1, scale="support", solver="lu")
    pts = g["scale_pts"]
    rows = np.arange(13, 50)
    nodes = m.find_closest_stencils(m.NodeSet(pts, np.ones(50, dtype=np.int64)), 5, for_which=rows)
    with pytest.raises(m.WeightError) as exc:
        m.compute_weights(nodes, eng, ["laplacian"], for_which=rows)
    assert str(exc.value) == str(g["scale_msg"])
    pts = g["singular_pts"]
    rows = np.arange(8)
    nodes = m.find_closest_stencils(m.NodeSet(pts, np.ones(40, dtype=np.int64)), 4, for_which=rows)
    with pytest.raises(m.WeightError) as exc:
        m.compute_weights(nodes, eng, ["laplacian"], for_which=rows)
    assert str(exc.value) == str(g["singular_msg"])


def test_unsupported_engine_raises_config_error():
    m = mf()
    nodes = m.find_closest_stencils(m.NodeSet(np.random.default_rng(0).uniform(0, 1, (50, 2)),
                                              np.ones(50, dtype=np.int64)), 9)
    # the reference default (solver qr) runs in the general engine kernel
    store = m.compute_weights(nodes, m.RbfFd(m.Polyharmonic(3), degree=1), ["laplacian"])
    assert np.all(np.isfinite(store.values["laplacian"]))
    with pytest.raises(m.ConfigError):  # a kernel class without a GPU implementation
        m.compute_weights(nodes, m.RbfFd(object(), degree=1), ["laplacian"])
    with pytest.raises(m.WeightError, match="augmentation of degree 3"):
        m.compute_weights(nodes, m.RbfFd(m.Polyharmonic(3), degree=3, solver="lu"), ["laplacian"])


# ---------------------------------------------------------------------------
# CSR, apply, heat
# ---------------------------------------------------------------------------

def _store_from(m, N, rows, stencils, weights: dict, n):
    import torch

    from paper_1912_13282_b200 import _lib
    from paper_1912_13282_b200.storage import WeightStore

    st_d = _lib.to_device(np.asarray(stencils, dtype=np.int32), torch.int32)
    vals = {k: _lib.to_device(np.asarray(v, dtype=float).reshape(-1, n), torch.float64) for k, v in weights.items()}
    return WeightStore(N, rows, st_d, vals, n)


def test_csr_and_apply_bitwise_vs_reference():
    m = mf()
    g = golden("csr_apply.npz")
    N = g["pts"].shape[0]
    keys = ["laplacian", "d1_0", "d1_1"]
    store = _store_from(m, N, g["rows"], g["stencils"], {k: g[f"{k}_w"] for k in keys}, 12)
    for key in keys:
        mat = store.matrix(key)
        assert mat.indptr.dtype == np.int32 and mat.indices.dtype == np.int32
        assert np.array_equal(mat.indptr, g[f"{key}_indptr"])
        assert np.array_equal(mat.indices, g[f"{key}_indices"])
        assert np.array_equal(mat.data, g[f"{key}_data"])
        y = store.apply_all(key, g["u"])
        assert np.array_equal(y, g[f"{key}_y"]), key
        import torch

        u_d = torch.from_numpy(g["u"]).cuda()
        assert np.array_equal(mat.apply_csr_device(u_d).cpu().numpy(), g[f"{key}_y"])
        for i in (int(g["rows"][0]), int(g["rows"][-1])):
            assert store.apply(key, g["u"], i) == g[f"{key}_y"][i]
    # boundary rows were not stored: empty rows, zero output, StorageError on access
    b = int(np.flatnonzero(g["types"] < 0)[0])
    assert store.apply_all("laplacian", g["u"])[b] == 0.0
    with pytest.raises(m.StorageError):
        store.weights("laplacian", b)


def test_csr_from_gpu_weights_matches_oracle_layout():
    m = mf()
    g = golden("csr_apply.npz")
    nodes = m.find_closest_stencils(m.NodeSet(g["pts"], g["types"]), 12)
    store = m.compute_weights(nodes, m.RbfFd(m.Polyharmonic(3), 2, "support", "lu"),
                              ["laplacian", "gradient"], for_which="interior")
    N = g["pts"].shape[0]
    for key in ("laplacian", "d1_0", "d1_1"):
        mat = store.matrix(key)
        assert np.array_equal(mat.indptr, g[f"{key}_indptr"])
        assert np.array_equal(mat.indices, g[f"{key}_indices"])
        ip, ix, da = oracle.csr_canonical(store.rows, store.cols.reshape(-1, 12),
                                          store.values[key].reshape(-1, 12), N)
        assert np.array_equal(mat.data, da)
        assert np.array_equal(store.apply_all(key, g["u"]), oracle.apply(ip, ix, da, g["u"]))


def test_heat_bitwise_and_instability():
    m = mf()
    g = golden("heat.npz")
    N = g["pts"].shape[0]
    nodes = m.NodeSet(g["pts"], g["types"])
    nodes = m.find_closest_stencils(nodes, 15)
    assert np.array_equal(nodes.stencil_matrix(), g["stencils"])
    store = _store_from(m, N, np.arange(N), g["stencils"], {"laplacian": g["w"]}, 15)
    u = m.run_heat_explicit(nodes, store, dt=float(g["dt"]), steps=int(g["steps"]),
                            dirichlet={-1: 0.0}, initial=g["u0"])
    assert np.array_equal(u, g["u_final"])
    u = m.run_heat_explicit(nodes, store, dt=float(g["dt"]), steps=25, diffusivity=0.7,
                            source=lambda p, t: 2.0, dirichlet={-1: 0.25}, initial=g["u0"])
    assert np.array_equal(u, g["u_final_src"])
    with pytest.raises(m.InstabilityError) as exc:
        m.run_heat_explicit(nodes, store, dt=float(g["dt_literal"]), steps=400, dirichlet={-1: 0.0},
                            initial=g["u0"])
    assert str(exc.value) == str(g["unstable_msg"])
    with pytest.raises(m.InstabilityError) as exc:
        m.run_heat_explicit(nodes, store, dt=0.5, steps=50, dirichlet={-1: 0.0}, initial=g["u0"])
    assert str(exc.value) == str(g["unstable2_msg"])
    u0 = m.run_heat_explicit(nodes, store, dt=0.1, steps=0, initial=g["u0"])
    assert np.array_equal(u0, g["u0"])


def test_heat_time_dependent_dirichlet_assigned_exactly():
    m = mf()
    g = golden("heat.npz")
    N = g["pts"].shape[0]
    nodes = m.find_closest_stencils(m.NodeSet(g["pts"], g["types"]), 15)
    store = _store_from(m, N, np.arange(N), g["stencils"], {"laplacian": g["w"]}, 15)
    fn = lambda pts, t: t * pts[:, 0]
    dt, steps = float(g["dt"]), 7
    u = m.run_heat_explicit(nodes, store, dt=dt, steps=steps, dirichlet={-1: fn}, initial=0.0)
    idx = nodes.boundary_indices()
    assert np.array_equal(u[idx], fn(nodes.positions[idx], steps * dt))
    with pytest.raises(m.ConfigError):
        m.run_heat_explicit(nodes, store, dt=0.0, steps=5)
    with pytest.raises(m.ConfigError, match="no node"):
        m.run_heat_explicit(nodes, store, dt=1e-4, steps=1, dirichlet={-9: 0.0})
