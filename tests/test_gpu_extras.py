"""GPU coverage beyond the core parity suite: the Neumann closure and the heat
loop with Neumann nodes, vector helpers, the opt-in shape
kernels, REPLAY-mode agreement statistics, and the C-ABI error paths.

The Neumann reference here is a numpy restatement of storage.py:226-250 /
drivers.py:99-102 applied to the same stored weights (test infrastructure).
"""

import os
import sys

import numpy as np
import pytest

import oracle
from conftest import REPO, golden

pytestmark = pytest.mark.gpu


def mf():
    import paper_1912_13282_b200 as m

    return m


def annulus(N=3000, seed=0):
    """Unit disk minus a hole: interior nodes +1, outer boundary -1, hole -2 with normals."""
    rng = np.random.default_rng(seed)
    r = np.sqrt(rng.uniform(0.16, 1.0, N))
    t = rng.uniform(0, 2 * np.pi, N)
    pts = np.stack([r * np.cos(t), r * np.sin(t)], 1)
    nb = 200
    tb = np.linspace(0, 2 * np.pi, nb, endpoint=False)
    outer = np.stack([np.cos(tb), np.sin(tb)], 1)
    inner = 0.4 * np.stack([np.cos(tb + 0.01), np.sin(tb + 0.01)], 1)
    P = np.concatenate([pts, outer, inner])
    types = np.concatenate([np.ones(N, np.int64), -np.ones(nb, np.int64), -2 * np.ones(nb, np.int64)])
    normals = np.full(P.shape, np.nan)
    normals[N:N + nb] = outer
    normals[N + nb:] = -inner / 0.4
    return P, types, normals


def neumann_ref(store, u, i, normal, gn):
    """storage.py:236-250 on host arrays (c = sum_a n_a w_d1_a; pivot guard; value)."""
    c = None
    for a, na in enumerate(np.asarray(normal, float)):
        part = na * store.weights(f"d1_{a}", i)
        c = part if c is None else c + part
    st = store.stencil(i)
    acc = float(gn)
    for j in range(1, st.shape[0]):
        acc -= c[j] * u[st[j]]
    return acc / c[0]


def test_neumann_value_and_heat_with_neumann():
    m = mf()
    P, types, normals = annulus()
    nodes = m.NodeSet(P, types, normals)
    nodes = m.find_closest_stencils(nodes, 12)
    eng = m.RbfFd(m.Polyharmonic(3), degree=2, scale="support", solver="lu")
    store = m.compute_weights(nodes, eng, ["laplacian", "gradient"])
    u = np.sin(P[:, 0]) + P[:, 1] ** 2
    for i in nodes.select(-2)[:20]:
        i = int(i)
        got = store.neumann_value(u, i, nodes.normal(i), 0.3)
        ref = neumann_ref(store, u, i, nodes.normal(i), 0.3)
        assert abs(got - ref) <= 1e-12 * max(1.0, abs(ref))
        c = store.normal_combination(i, nodes.normal(i))
        u2 = u.copy()
        u2[i] = got
        assert abs(c @ u2[store.stencil(i)] - 0.3) <= 1e-9 * np.abs(c).sum()
    # heat with Dirichlet on the outer circle and Neumann on the hole; 10 steps
    # run the packed operator (mf_heat_pack) on the node-ordered plan
    dt = 1e-6
    for steps in (4, 10):
        out = m.run_heat_explicit(nodes, store, dt=dt, steps=steps, dirichlet={-1: 0.0}, neumann={-2: 0.0},
                                  initial=u)
        lap = store.matrix("laplacian")
        cur = u.copy()
        cur[nodes.select(-1)] = 0.0
        for _ in range(steps):
            lap_u = oracle.apply(lap.indptr, lap.indices, lap.data, cur)
            new = cur.copy()
            it = nodes.interior_indices()
            new[it] = cur[it] + dt * (1.0 * lap_u[it] + 0.0)
            new[nodes.select(-1)] = 0.0
            for i in nodes.select(-2):
                new[int(i)] = neumann_ref(store, cur, int(i), nodes.normal(int(i)), 0.0)
            cur = new
        assert np.max(np.abs(out - cur)) <= 1e-12 * np.max(np.abs(cur))


def test_vector_helpers_exact_on_linear_fields():
    m = mf()
    rng = np.random.default_rng(2)
    P = rng.uniform(-1, 1, (800, 2))
    nodes = m.find_closest_stencils(m.NodeSet(P, np.ones(800, dtype=np.int64)), 12)
    store = m.compute_weights(nodes, m.RbfFd(m.Polyharmonic(3), 2, "support", "lu"),
                              ["laplacian", "gradient", "hessian"])
    u = 2.0 * P[:, 0] - 3.0 * P[:, 1] + 0.5
    vec = np.stack([4.0 * P[:, 0], P[:, 1]], axis=1)
    i = 5
    assert np.allclose(store.gradient(u, i), [2.0, -3.0], atol=1e-8)
    assert store.divergence(vec, i) == pytest.approx(5.0, abs=1e-8)
    assert np.allclose(store.vector_laplacian(vec, i), [0.0, 0.0], atol=1e-6)
    assert np.allclose(store.grad_div(vec, i), [0.0, 0.0], atol=1e-6)


def test_replay_mode_agreement_statistics():
    """REPLAY follows the reference op order; only glibc pow vs correctly rounded r^3 differs."""
    m = mf()
    from paper_1912_13282_b200 import workloads

    g = golden("config_C4.npz")
    w = workloads.make("C4")
    nodes = m.find_closest_stencils(m.NodeSet(w.positions, w.types), w.n, for_which=g["targets"])
    store = m.compute_weights(nodes, m.RbfFd(m.Polyharmonic(3), 2, "support", "lu", mode="replay"),
                              ["laplacian"], for_which=g["targets"])
    got = store.values["laplacian"].reshape(g["w_laplacian"].shape)
    bitwise = np.mean(np.all(got == g["w_laplacian"], axis=1))
    err = np.max(np.abs(got - g["w_laplacian"]), 1) / np.max(np.abs(g["w_laplacian"]), 1)
    print(f"C4 replay: {bitwise:.3f} of rows bitwise, max normwise {err.max():.2e}")
    assert bitwise >= 0.5 and err.max() <= 1e-11


def test_c_abi_rejects_bad_arguments():
    import ctypes

    import torch

    from paper_1912_13282_b200 import _lib

    lib = _lib.load()
    size = ctypes.c_size_t(0)
    assert lib.mf_knn_workspace_size(10, 4, 5, 10, 3, ctypes.byref(size)) != 0  # d = 4
    assert b"bad arguments" in lib.mf_last_error()
    dummy = torch.zeros(16, dtype=torch.float64, device="cuda")
    rc = lib.mf_knn(dummy.data_ptr(), 2, 2, dummy.data_ptr(), 1, dummy.data_ptr(), 2, 3, dummy.data_ptr(), None,
                    dummy.data_ptr(), 128, _lib.stream_ptr())
    assert rc != 0 and b"stencil size" in lib.mf_last_error()
    assert lib.mf_apply(None, None, None, None, None, -1, None) != 0
