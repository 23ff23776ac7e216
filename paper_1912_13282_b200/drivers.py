"""Explicit forward-Euler heat stepping and the implicit steady solve on the GPU.

Drop-in for the reference's run_heat_explicit (drivers.py:48-111): same
arguments, checks, boundary handling order (interior Euler update, Dirichlet
assignment at t_new, Neumann closure from the previous field) and the same
InstabilityError at the first step whose max|u| exceeds 1e12 or is not
finite.  Step-invariant data (constant Dirichlet/Neumann values and source)
runs as one ``mf_heat_steps`` call over the ELL-32 plan of the laplacian;
time-dependent callables are evaluated on the host at the reference's times
and the device steps one at a time.

``solve_poisson_implicit`` (drivers.py:114-157) assembles the whole
collocation system in one device pass over the weight store's canonical
structure (``mf_assemble_*``: the same canonical CSR the reference's row loop
and ``SparseSystem.finalize`` produce, bitwise) and solves it with the GPU
BiCGStab of solve.py.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, GeometryError, InstabilityError, NumericalError, StorageError
from .solve import SolverConfig, SystemMatrix, solve_sparse
from .storage import _to_host

BLOWUP_LIMIT = 1e12
# the loop runs over the packed operator (16-bit column offsets) when rows fit it;
# tests switch it off to compare against the unpacked plan (the sums are identical)
PACK_OPERATOR = True


def _bc_values(value, points, t):
    if callable(value):
        out = value(points, t)
        return np.broadcast_to(np.asarray(out, dtype=float), (points.shape[0],))
    return np.full(points.shape[0], float(value))


def _tag_indices(nodes, bc_dict):
    out = {}
    for tag, value in (bc_dict or {}).items():
        idx = nodes.select(int(tag))
        if idx.size == 0:
            raise ConfigError(f"boundary condition for tag {tag} matches no node")
        out[int(tag)] = (idx, value)
    return out


def _instability(step, peak):
    return InstabilityError(
        step,
        f"field peak {peak:.2e} exceeds {BLOWUP_LIMIT:.0e}; forward Euler "
        "needs roughly dt <= h_min^2 / (2 d D)",
    )


@_lib.traced("meshfree.run_heat_explicit")
def run_heat_explicit(
    nodes,
    store,
    *,
    dt: float,
    steps: int,
    diffusivity: float = 1.0,
    source=None,
    dirichlet=None,
    neumann=None,
    initial=0.0,
    return_device: bool = False,
):
    """Forward-Euler march of du/dt = D lap(u) + f (drivers.py:48-111).

    Returns the field after ``steps`` steps as a host array (or the device
    tensor with ``return_device=True``).
    """
    if dt <= 0 or steps < 0:
        raise ConfigError("need dt > 0 and steps >= 0")
    lib = _lib.load()
    n = len(nodes)
    pts = nodes.positions
    u = np.empty(n)
    if callable(initial):
        u[:] = np.asarray(initial(pts), dtype=float)
    else:
        u[:] = np.asarray(initial, dtype=float)

    diri = _tag_indices(nodes, dirichlet)
    neum = _tag_indices(nodes, neumann)
    for idx, value in diri.values():
        u[idx] = _bc_values(value, pts[idx], 0.0)

    dev = _lib.device()
    u_d = _lib.to_device(u, torch.float64)
    if steps == 0:
        return u_d if return_device else u

    lap = store.matrix("laplacian")
    # Morton-ordered plan unless a Neumann closure needs node-ordered fields
    plan = lap.plan(ordered=not neum)
    perm = plan.order.long() if plan.ordered else None

    def to_plan(arr, dtype):
        t = _lib.to_device(arr, dtype)
        return t.index_select(0, perm) if perm is not None else t

    interior = np.zeros(n, dtype=np.uint8)
    interior[nodes.interior_indices()] = 1
    interior_d = to_plan(interior, torch.uint8)
    dmask = np.zeros(n, dtype=np.uint8)
    for idx, _ in diri.values():
        dmask[idx] = 1
    dmask_d = to_plan(dmask, torch.uint8)

    time_dep = callable(source) or any(callable(v) for _, v in diri.values()) or any(
        callable(v) for _, v in neum.values())

    def dirichlet_vals(t):
        g = np.zeros(n)
        for idx, value in diri.values():
            g[idx] = _bc_values(value, pts[idx], t)
        return g

    # Neumann closure: nodes in tag order, normals, stencil weights (drivers.py:99-102)
    nm = None
    if neum:
        nm_nodes = np.concatenate([idx for idx, _ in neum.values()]).astype(np.int64)
        for i in nm_nodes:
            store._row(int(i))
        normals = np.stack([nodes.normal(int(i)) for i in nm_nodes])
        plane = store.neumann_plane(nodes.dim)
        normals_d = _lib.to_device(normals, torch.float64)
        _, bad = store.neumann_values_device(nm_nodes, normals, np.zeros(nm_nodes.shape[0]), u_d,
                                             plane=plane, normals_d=normals_d)
        if bad is not None:
            raise NumericalError(
                f"node {int(nm_nodes[bad])}: negligible self-weight in the normal derivative; "
                "the stencil cannot enforce a Neumann condition explicitly"
            )
        nm_mask = np.zeros(n, dtype=np.uint8)
        nm_mask[nm_nodes] = 1
        nm_keep = dict(nodes=_lib.to_device(nm_nodes, torch.int64), plane=plane, normals=normals_d,
                       mask=_lib.to_device(nm_mask, torch.uint8), node_row=store.node_row_device())

        def neumann_vals(t):
            return np.concatenate([_bc_values(v, pts[idx], t) for idx, v in neum.values()])

        def make_nm(g_d):
            return _lib.NeumannT(store.stencils_device.data_ptr(), store.n, plane.data_ptr(), plane.shape[1],
                                 nodes.dim, normals_d.data_ptr(), nm_keep["nodes"].data_ptr(),
                                 nm_keep["node_row"].data_ptr(), g_d.data_ptr(), nm_nodes.shape[0],
                                 nm_keep["mask"].data_ptr())

    scratch = torch.empty(n, dtype=torch.float64, device=dev)
    peaks = torch.empty(steps, dtype=torch.int64, device=dev)
    u_node = u_d
    if perm is not None:
        u_d = torch.empty_like(u_node)
        _lib.check(lib.mf_permute(u_node.data_ptr(), plan.order.data_ptr(), n, 0, u_d.data_ptr(),
                                  _lib.stream_ptr()), "mf_permute")

    # packed operator (16-bit column offsets, one meta byte per row) for the
    # loop when the rows fit it; the sums are unchanged
    pack = None
    if steps >= 8 and 0 < plan.W <= 16 and PACK_OPERATOR:
        d16 = torch.empty(max(plan.ell_idx.numel(), 1), dtype=torch.int16, device=dev)
        meta = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        wide = torch.empty(max((n + 31) // 32, 1), dtype=torch.uint8, device=dev)
        _lib.check(lib.mf_heat_pack(plan.ell_len.data_ptr(), plan.ell_idx.data_ptr(), interior_d.data_ptr(),
                                    dmask_d.data_ptr(), n, plan.W, d16.data_ptr(), meta.data_ptr(),
                                    wide.data_ptr(), _lib.stream_ptr()), "mf_heat_pack")
        pack = (_lib.HeatPackT(d16.data_ptr(), meta.data_ptr(), wide.data_ptr()), d16, meta, wide)

    def launch(k_steps, g_d, src_d, nm_struct, peak_view):
        _lib.check(lib.mf_heat_steps(
            plan.ell_len.data_ptr(), plan.ell_idx.data_ptr(), plan.ell_val.data_ptr(), n, plan.W,
            interior_d.data_ptr(), dmask_d.data_ptr(), g_d.data_ptr(), _lib.ptr(src_d), float(dt),
            float(diffusivity), None if nm_struct is None else ctypes.byref(nm_struct), k_steps,
            u_d.data_ptr(), scratch.data_ptr(), peak_view.data_ptr(),
            None if pack is None else ctypes.byref(pack[0]), _lib.stream_ptr()), "mf_heat_steps")

    if not time_dep:
        g_d = to_plan(dirichlet_vals(dt), torch.float64)
        src_d = None if source is None else to_plan(_bc_values(source, pts, 0.0), torch.float64)
        nm_struct = None
        if neum:
            gn_d = _lib.to_device(neumann_vals(dt), torch.float64)
            nm_struct = make_nm(gn_d)
        launch(steps, g_d, src_d, nm_struct, peaks)
    else:
        for step in range(steps):
            t_new = (step + 1) * dt
            g_d = to_plan(dirichlet_vals(t_new), torch.float64)
            src_d = None if source is None else to_plan(_bc_values(source, pts, step * dt), torch.float64)
            nm_struct = None
            if neum:
                gn_d = _lib.to_device(neumann_vals(t_new), torch.float64)
                nm_struct = make_nm(gn_d)
            launch(1, g_d, src_d, nm_struct, peaks[step:step + 1])
            if (step + 1) % 64 == 0 or step + 1 == steps:
                if _first_bad(peaks[: step + 1]) is not None:
                    break

    bad = _first_bad(peaks)
    if bad is not None:
        step, peak = bad
        raise _instability(step, peak)
    if perm is not None:
        _lib.check(lib.mf_permute(u_d.data_ptr(), plan.order.data_ptr(), n, 1, u_node.data_ptr(),
                                  _lib.stream_ptr()), "mf_permute")
        u_d = u_node
    return u_d if return_device else _to_host(u_d)


def _first_bad(peaks: torch.Tensor):
    """(1-based step, peak) of the first step with max|u| > 1e12 or non-finite, else None."""
    limit_bits = int(np.float64(BLOWUP_LIMIT).view(np.int64))
    bad = torch.nonzero(peaks > limit_bits)
    if bad.numel() == 0:
        return None
    s = int(bad[0, 0].item())
    peak = float(np.int64(peaks[s].item()).view(np.float64))
    if math.isnan(peak):
        peak = float("nan")
    return s + 1, peak


def _steady_values(value, points):
    if callable(value):
        out = value(points)
        return np.broadcast_to(np.asarray(out, dtype=float), (points.shape[0],))
    arr = np.asarray(value, dtype=float)
    if arr.ndim == 0:
        return np.full(points.shape[0], float(arr))
    return np.broadcast_to(arr, (points.shape[0],))


def assemble_poisson_system(nodes, store, *, terms, rhs, dirichlet=None, neumann=None):
    """The assembly half of solve_poisson_implicit (drivers.py:135-154): the
    canonical system matrix (SystemMatrix) and right-hand side.  Errors are the
    reference's, raised for the node its row loop would reach first."""
    lib = _lib.load()
    n = len(nodes)
    pts = nodes.positions
    kind = np.zeros(n, dtype=np.int8)
    rhs_vec = np.zeros(n)
    node_row = store.node_row

    interior = nodes.interior_indices()
    f = _steady_values(rhs, pts[interior])
    if isinstance(terms, str):
        terms = [(1.0, terms)]
    if interior.size:
        lacking = interior[node_row[interior] < 0]
        if lacking.size:
            raise StorageError(f"no weights stored for node {int(lacking[0])}")
        for _, key in terms:
            store._family(key)
    kind[interior] = 1
    rhs_vec[interior] = f

    def claim(idx):
        taken = kind[idx] != 0
        if taken.any():
            raise StorageError(f"row {int(idx[np.argmax(taken)])} is already committed")

    for idx, value in _tag_indices(nodes, dirichlet).values():
        g = _steady_values(value, pts[idx])
        claim(idx)
        kind[idx] = 2
        rhs_vec[idx] = g
    neu_nodes, neu_normals = [], []
    for idx, value in _tag_indices(nodes, neumann).values():
        g = _steady_values(value, pts[idx])
        # per row, in order: nodes.normal(i), store.stencil(i), the d1 families of
        # normal_combination, then the claim (drivers.py:149-152, assembly.py:85-88)
        e_geom = nodes.types[idx] >= 0
        e_store = node_row[idx] < 0
        fam_missing = any(f"d1_{a}" not in store.families for a in range(nodes.dim))
        e_claim = kind[idx] != 0
        bad = e_geom | e_store | e_claim | fam_missing
        if bad.any():
            j = int(np.argmax(bad))
            i = int(idx[j])
            if e_geom[j]:
                raise GeometryError(f"node {i} is not a boundary node")
            if e_store[j]:
                raise StorageError(f"no weights stored for node {i}")
            for a in range(nodes.dim):
                store._family(f"d1_{a}")
            raise StorageError(f"row {i} is already committed")
        kind[idx] = 3
        rhs_vec[idx] = g
        neu_nodes.append(idx)
        neu_normals.append(nodes.normals[idx])
    missing = np.flatnonzero(kind == 0)
    if missing.size:
        raise StorageError(f"{missing.size} rows never committed (first: node {missing[0]})")

    # values: interior term combination over every stored row (storage order of
    # the reference's `acc`), Neumann normal combinations for the Neumann rows
    dev = _lib.device()
    v_int = None
    for coeff, key in terms:
        part = float(coeff) * store._family(key).reshape(-1)
        v_int = part if v_int is None else v_int + part
    if v_int is None:
        v_int = torch.zeros(1, dtype=torch.float64, device=dev)
    v_neu = torch.zeros(1, dtype=torch.float64, device=dev)
    neu_row = torch.zeros(1, dtype=torch.int64, device=dev)
    if neu_nodes:
        nn = np.concatenate(neu_nodes)
        nrm = np.concatenate(neu_normals, axis=0)
        rows_n = _lib.to_device(node_row[nn], torch.int64)
        nrm_d = _lib.to_device(nrm, torch.float64)
        acc = None
        for a in range(nrm.shape[1]):
            part = nrm_d[:, a:a + 1] * store._family(f"d1_{a}")[rows_n]
            acc = part if acc is None else acc + part
        v_neu = acc.contiguous()
        nr = np.zeros(n, dtype=np.int64)
        nr[nn] = np.arange(nn.size)
        neu_row = _lib.to_device(nr, torch.int64)
    s = store.structure()
    kind_d = _lib.to_device(kind, torch.int8)
    indptr = torch.empty(n + 1, dtype=torch.int32, device=dev)
    miss = torch.empty(1, dtype=torch.int64, device=dev)
    size = ctypes.c_size_t(0)
    _lib.check(lib.mf_assemble_workspace_size(n, ctypes.byref(size)), "mf_assemble_workspace_size")
    ws = _lib.workspace(size.value)
    nnz = ctypes.c_int64(0)
    _lib.check(lib.mf_assemble_rows(s.indptr.data_ptr(), kind_d.data_ptr(), n, indptr.data_ptr(), miss.data_ptr(),
                                    ctypes.byref(nnz), ws.data_ptr(), size.value, _lib.stream_ptr()),
               "mf_assemble_rows")
    bad = int(miss.item())
    if bad != _lib.SENTINEL_OK:  # pre-checked above; kept as a device-side guard
        raise StorageError(f"no weights stored for node {bad}")
    indices = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)
    data = torch.empty(max(nnz.value, 1), dtype=torch.float64, device=dev)
    _lib.check(lib.mf_assemble_fill(s.indptr.data_ptr(), s.indices.data_ptr(), s.perm.data_ptr(), store.n,
                                    v_int.data_ptr(), v_neu.data_ptr(), neu_row.data_ptr(), kind_d.data_ptr(), n,
                                    indptr.data_ptr(), indices.data_ptr(), data.data_ptr(), _lib.stream_ptr()),
               "mf_assemble_fill")
    return SystemMatrix(indptr, indices[: nnz.value], data[: nnz.value], n), rhs_vec


@_lib.traced("meshfree.solve_poisson_implicit")
def solve_poisson_implicit(
    nodes,
    store,
    *,
    terms,
    rhs,
    dirichlet=None,
    neumann=None,
    config: SolverConfig | None = None,
    system_out: list | None = None,
):
    """Assemble and solve a steady collocation problem (drivers.py:114-157).

    ``terms`` is a family name or ``(coeff, family)`` list and ``rhs`` a
    constant or callable ``f(points)`` for the interior rows.  Every node must
    end up covered: interior by the PDE, boundary by exactly one of the
    condition dictionaries.  ``system_out``, when given, receives the
    assembled ``(matrix, rhs)`` (a device SystemMatrix; ``.to_scipy()`` gives
    the reference's scipy CSR).
    """
    matrix, rhs_vec = assemble_poisson_system(nodes, store, terms=terms, rhs=rhs, dirichlet=dirichlet,
                                              neumann=neumann)
    if system_out is not None:
        system_out.append((matrix, rhs_vec))
    return solve_sparse(matrix, rhs_vec, config)
