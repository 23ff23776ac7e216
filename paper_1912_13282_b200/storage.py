"""Weight tables on the GPU: compute once, apply many times.

Drop-in for the reference's storage module (storage.py:1-409).
``compute_weights`` runs the batched polyharmonic RBF-FD kernel
(``mf_phs_weights``) over the stencils of the chosen nodes for a list of
operator families and returns a :class:`WeightStore` whose weights stay on
the device.  The reference's public fields (``rows``, ``offsets``, ``cols``,
``values``, ``node_row``) are available as host arrays, materialised lazily.

``WeightStore.matrix(key)`` returns a :class:`DeviceCSR` with the reference's
canonical layout (rows ascending, columns ascending, int32 indices, rows only
for stored nodes -- storage.py:156-170); ``@`` and ``apply_all`` run on the GPU
and are bitwise equal to scipy's ``csr_matvec`` on the same matrix.

The reference's batched configuration (storage.py:310-322: RbfFd +
Polyharmonic(k >= 3), ``solver="lu"``, scale none/nearest/support,
elementary operator families) runs in the hot shape kernels
(``mf_phs_weights``); every other engine configuration the reference sends
through its per-node loop (storage.py:325-339) -- qr / svd solvers,
Gaussian / multiquadric / inverse multiquadric kernels, r^k with k <= 2,
WeightedLeastSquares, composite operators -- runs batched in the general
engine kernel (``mf_engine_weights``).  Stencils must have one size (the
device store is dense); user-defined operator or weight classes, whose point
evaluation is Python code, raise ConfigError: there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
from collections.abc import Mapping

import numpy as np
import torch

from . import _lib
from .approx import (
    ConstantWeight,
    Directional,
    FirstDerivative,
    Gaussian,
    GaussianWeight,
    Identity,
    InverseMultiquadric,
    Laplacian,
    MonomialBasis,
    Multiquadric,
    Operator,
    OperatorSum,
    Polyharmonic,
    RbfFd,
    ScaledOperator,
    SecondDerivative,
    WeightedLeastSquares,
    graded_lex_exponents,
    monomial_count,
)
from .errors import ConfigError, NumericalError, StencilError, StorageError, WeightError

# first-slot pivot guard for the explicit Neumann solve (storage.py:41-42)
NEUMANN_PIVOT_RTOL = 1e-12

KIND_IDENTITY, KIND_D1, KIND_D2, KIND_LAPLACIAN = 0, 1, 2, 3
SCALE_CODES = {"none": 0, "nearest": 1, "support": 2}
MODES = {"replay": _lib.PHS_REPLAY, "fast": _lib.PHS_FAST, "hybrid": _lib.PHS_HYBRID}


def _canonical_key(op) -> str:
    if isinstance(op, Identity):
        return "identity"
    if isinstance(op, FirstDerivative):
        return f"d1_{op.axis}"
    if isinstance(op, SecondDerivative):
        return f"d2_{op.a}_{op.b}"
    if isinstance(op, Laplacian):
        return "laplacian"
    raise StorageError(
        f"{op!r} has no canonical family name; store it as (name, operator)"
    )


def _key_to_operator(key: str, dim: int) -> Operator:
    if key == "identity":
        return Identity()
    if key == "laplacian":
        return Laplacian()
    if key.startswith("d1_"):
        axis = int(key[3:])
        if not 0 <= axis < dim:
            raise StorageError(f"axis out of range in family {key!r}")
        return FirstDerivative(axis)
    if key.startswith("d2_"):
        a, b = (int(x) for x in key[3:].split("_"))
        if not 0 <= a <= b < dim:
            raise StorageError(f"axes out of range in family {key!r}")
        return SecondDerivative(a, b)
    raise StorageError(f"unknown family {key!r}")


def expand_families(families, dim: int):
    """Normalize a family spec list into an ordered {name: operator} dict (storage.py:77-108)."""
    out: dict[str, Operator] = {}

    def put(key, op):
        if key in out:
            raise StorageError(f"family {key!r} requested twice")
        out[key] = op

    for spec in families:
        if isinstance(spec, str):
            if spec == "gradient":
                for a in range(dim):
                    put(f"d1_{a}", FirstDerivative(a))
            elif spec == "hessian":
                for a in range(dim):
                    for b in range(a, dim):
                        put(f"d2_{a}_{b}", SecondDerivative(a, b))
            else:
                put(spec, _key_to_operator(spec, dim))
        elif isinstance(spec, Operator):
            put(_canonical_key(spec), spec)
        elif isinstance(spec, tuple) and len(spec) == 2 and isinstance(spec[1], Operator):
            name = str(spec[0])
            if "," in name or not name:
                raise StorageError(f"bad custom family name {name!r}")
            put(name, spec[1])
        else:
            raise StorageError(f"cannot interpret family spec {spec!r}")
    if not out:
        raise StorageError("no operator families requested")
    return out


# ---------------------------------------------------------------------------
# device CSR
# ---------------------------------------------------------------------------

def _to_host(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> numpy array backed by pinned memory (fast D2H; torch caches pinned blocks)."""
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


def _result_to_host(y: torch.Tensor, structure) -> np.ndarray:
    """The applied field to the host with the structure's deferred duplicate-row
    check riding on the same synchronisation (one host wait instead of two)."""
    h = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
    h.copy_(y, non_blocking=True)
    flag = None
    if not structure._checked:
        flag = torch.empty(1, dtype=structure._dup.dtype, pin_memory=True)
        flag.copy_(structure._dup, non_blocking=True)
    torch.cuda.current_stream(y.device).synchronize()
    if flag is not None:
        if int(flag[0]) != 0:
            raise StorageError("stored rows must be distinct node indices")
        structure._checked = True
    return h.numpy()


def _to_field(field, N):
    """Field argument -> (device f64 tensor, was_numpy).

    The kernels index the field by node number without bounds checks, so a
    device field must be a length-N vector on the current device (a shorter
    one would be read out of bounds); host fields broadcast like numpy.
    """
    if isinstance(field, torch.Tensor) and field.is_cuda:
        if field.ndim != 1 or field.shape[0] != N:
            raise ValueError(f"field of shape {tuple(field.shape)} does not match the {N} nodes")
        if field.device != _lib.device():
            raise ValueError(f"field on {field.device}, weights on {_lib.device()}")
        return field.to(torch.float64).contiguous(), False
    arr = np.asarray(field, dtype=float)
    if arr.shape != (N,):
        try:
            arr = np.broadcast_to(arr, (N,))
        except ValueError:
            raise ValueError(f"field of shape {arr.shape} does not match the {N} nodes") from None
    return _lib.to_device(arr, torch.float64), True


class _CsrStructure:
    """indptr / indices / stencil-slot permutation shared by every family of a store."""

    def __init__(self, n_nodes, rows_d, stencils_d, n, positions_d=None):
        lib = _lib.load()
        dev = _lib.device()
        m = int(stencils_d.shape[0])
        self.N = int(n_nodes)
        self.n = int(n)
        self.nnz = m * self.n
        self.positions_d = positions_d
        self.indptr = torch.empty(self.N + 1, dtype=torch.int32, device=dev)
        self.indices = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev)
        self.perm = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev)
        self._dup = torch.zeros(1, dtype=torch.int32, device=dev)
        size = ctypes.c_size_t(0)
        _lib.check(lib.mf_csr_workspace_size(self.N, ctypes.byref(size)), "mf_csr_workspace_size")
        ws = _lib.workspace(size.value)
        _lib.check(lib.mf_csr_build(rows_d.data_ptr(), stencils_d.data_ptr(), m, self.n, self.N,
                                    self.indptr.data_ptr(), self.indices.data_ptr(), self.perm.data_ptr(),
                                    self._dup.data_ptr(), ws.data_ptr(), size.value, _lib.stream_ptr()),
                   "mf_csr_build")
        # checked lazily (no host sync on the build path): see check()
        self._checked = False
        self._plans = {}

    def check(self):
        if not self._checked:
            if int(self._dup.item()) != 0:
                raise StorageError("stored rows must be distinct node indices")
            self._checked = True

    def _order(self, ordered: bool):
        """(order, inv) of the Morton renumbering, or (None, None)."""
        if not ordered:
            return None, None
        if getattr(self, "_morton", None) is None:
            lib = _lib.load()
            dev = self.indptr.device
            order = torch.empty(self.N, dtype=torch.int32, device=dev)
            inv = torch.empty(self.N, dtype=torch.int32, device=dev)
            size = ctypes.c_size_t(0)
            _lib.check(lib.mf_order_workspace_size(self.N, ctypes.byref(size)), "mf_order_workspace_size")
            ws = _lib.workspace(size.value)
            pos = self.positions_d
            _lib.check(lib.mf_locality_order(pos.data_ptr(), self.N, int(pos.shape[1]), order.data_ptr(),
                                             inv.data_ptr(), ws.data_ptr(), size.value, _lib.stream_ptr()),
                       "mf_locality_order")
            self._morton = (order, inv)
        return self._morton

    def plan(self, ordered: bool):
        """Apply-plan structure: (order, inv, ell_idx, ell_len); order/inv None when unordered."""
        ordered = ordered and self.positions_d is not None
        if ordered not in self._plans:
            lib = _lib.load()
            dev = self.indptr.device
            order, inv = self._order(ordered)
            total = ((self.N + 31) // 32) * 32 * self.n
            ell_idx = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
            ell_len = torch.empty(max(self.N, 1), dtype=torch.int32, device=dev)
            _lib.check(lib.mf_plan_build(self.indptr.data_ptr(), self.indices.data_ptr(), None, self.N, self.n,
                                         _lib.ptr(order), _lib.ptr(inv), ell_idx.data_ptr(), None,
                                         ell_len.data_ptr(), _lib.stream_ptr()), "mf_plan_build")
            self._plans[ordered] = (order, inv, ell_idx, ell_len)
        return self._plans[ordered]

    def plan_direct(self, data):
        """(order, ell_idx, ell_val, ell_len) of a Morton-row plan whose columns stay
        in node numbering (mf_plan_apply_direct: one launch, no permutes).  Values
        are those of `data`; the index arrays are built once."""
        if self.positions_d is None:  # no positions: no locality order (node-ordered plan instead)
            return None
        total = ((self.N + 31) // 32) * 32 * self.n
        order, _ = self._order(True)
        val = torch.empty(max(total, 1), dtype=torch.float64, device=data.device)
        fresh = getattr(self, "_direct", None) is None
        if fresh:
            idx = torch.empty(max(total, 1), dtype=torch.int32, device=data.device)
            ln = torch.empty(max(self.N, 1), dtype=torch.int32, device=data.device)
        else:
            idx, ln = self._direct
        _lib.check(_lib.load().mf_plan_build(self.indptr.data_ptr(), self.indices.data_ptr(), data.data_ptr(),
                                             self.N, self.n, order.data_ptr(), None,
                                             idx.data_ptr() if fresh else None, val.data_ptr(),
                                             ln.data_ptr() if fresh else None, _lib.stream_ptr()),
                   "mf_plan_build")
        if fresh:
            self._direct = (idx, ln)
        return order, idx, val, ln

    def plan_values(self, data, ordered: bool):
        """ELL values of `data` in the plan's layout (the first call also builds the
        structure arrays in the same pass over the CSR)."""
        ordered = ordered and self.positions_d is not None
        total = ((self.N + 31) // 32) * 32 * self.n
        val = torch.empty(max(total, 1), dtype=torch.float64, device=data.device)
        fresh = ordered not in self._plans
        if fresh:
            order, inv = self._order(ordered)
            ell_idx = torch.empty(max(total, 1), dtype=torch.int32, device=data.device)
            ell_len = torch.empty(max(self.N, 1), dtype=torch.int32, device=data.device)
        else:
            order, inv, ell_idx, ell_len = self._plans[ordered]
        _lib.check(_lib.load().mf_plan_build(self.indptr.data_ptr(), self.indices.data_ptr(), data.data_ptr(),
                                             self.N, self.n, _lib.ptr(order), _lib.ptr(inv),
                                             ell_idx.data_ptr() if fresh else None, val.data_ptr(),
                                             ell_len.data_ptr() if fresh else None, _lib.stream_ptr()),
                   "mf_plan_build")
        if fresh:
            self._plans[ordered] = (order, inv, ell_idx, ell_len)
        return val


class ApplyPlan:
    """A matrix's apply plan: Morton-ordered (or node-ordered) ELL-32 arrays."""

    def __init__(self, order, inv, ell_idx, ell_val, ell_len, N, W):
        self.order, self.inv = order, inv
        self.ell_idx, self.ell_val, self.ell_len = ell_idx, ell_val, ell_len
        self.N, self.W = N, W

    @property
    def ordered(self) -> bool:
        return self.order is not None


class DeviceCSR:
    """N x N CSR on the device in the reference's canonical layout.

    ``indptr``/``indices``/``data`` return host numpy arrays (int32, int32,
    float64, as scipy stores them); ``*_device`` give the device tensors.
    ``A @ u`` applies on the GPU (numpy in -> numpy out, CUDA tensor in ->
    CUDA tensor out).
    """

    def __init__(self, structure: _CsrStructure, data_d: torch.Tensor):
        self._s = structure
        self.data_device = data_d
        self.shape = (structure.N, structure.N)
        self._host = {}
        self._plan = {}
        self._scratch = None

    @property
    def nnz(self) -> int:
        return self._s.nnz

    @property
    def indptr_device(self):
        return self._s.indptr

    @property
    def indices_device(self):
        return self._s.indices[: self.nnz]

    def _get(self, name, t):
        self._s.check()
        if name not in self._host:
            self._host[name] = t.cpu().numpy()
        return self._host[name]

    @property
    def indptr(self):
        return self._get("indptr", self._s.indptr)

    @property
    def indices(self):
        return self._get("indices", self._s.indices[: self.nnz])

    @property
    def data(self):
        return self._get("data", self.data_device[: self.nnz])

    def plan(self, ordered: bool = True) -> ApplyPlan:
        """The apply plan of this matrix (built once per ordering)."""
        if ordered not in self._plan:
            val = self._s.plan_values(self.data_device, ordered)
            order, inv, idx, ln = self._s.plan(ordered)
            self._plan[ordered] = ApplyPlan(order, inv, idx, val, ln, self._s.N, self._s.n)
        return self._plan[ordered]

    def plan_direct(self):
        """The Morton-row plan with node-numbered columns (built once per matrix)."""
        if getattr(self, "_pd", None) is None:
            self._pd = self._s.plan_direct(self.data_device)
        return self._pd

    def apply_device(self, u_d: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """y = A u on the device: the Morton-row plan read with node-numbered columns
        (mf_plan_apply_direct, one launch; the field is L2-resident), or the
        node-ordered plan when the store has no positions."""
        lib = _lib.load()
        N = self._s.N
        y = out if out is not None else torch.empty(N, dtype=torch.float64, device=u_d.device)
        pd = self.plan_direct()
        if pd is not None:
            order, idx, val, ln = pd
            _lib.check(lib.mf_plan_apply_direct(idx.data_ptr(), val.data_ptr(), ln.data_ptr(), N, self._s.n,
                                                order.data_ptr(), u_d.data_ptr(), y.data_ptr(), _lib.stream_ptr()),
                       "mf_plan_apply_direct")
            return y
        p = self.plan(True)
        su = sy = None
        if p.ordered:
            if self._scratch is None or self._scratch.device != u_d.device:
                self._scratch = torch.empty((2, N), dtype=torch.float64, device=u_d.device)
            su, sy = self._scratch[0], self._scratch[1]
        _lib.check(lib.mf_plan_apply(p.ell_idx.data_ptr(), p.ell_val.data_ptr(), p.ell_len.data_ptr(), N, p.W,
                                     _lib.ptr(p.order), u_d.data_ptr(), y.data_ptr(), _lib.ptr(su), _lib.ptr(sy),
                                     _lib.stream_ptr()), "mf_plan_apply")
        return y

    def apply_csr_device(self, u_d: torch.Tensor) -> torch.Tensor:
        """Same product straight from the CSR arrays (mf_apply)."""
        lib = _lib.load()
        y = torch.empty(self._s.N, dtype=torch.float64, device=u_d.device)
        _lib.check(lib.mf_apply(self._s.indptr.data_ptr(), self._s.indices.data_ptr(),
                                self.data_device.data_ptr(), u_d.data_ptr(), y.data_ptr(), self._s.N,
                                _lib.stream_ptr()), "mf_apply")
        return y

    def __matmul__(self, field):
        u_d, host = _to_field(field, self._s.N)
        y = self.apply_device(u_d)
        if host:
            return _result_to_host(y, self._s)
        return y

    def to_scipy(self):
        """The same matrix as a scipy csr_matrix over host copies of the arrays (built once)."""
        if getattr(self, "_sp", None) is None:
            import scipy.sparse

            self._sp = scipy.sparse.csr_matrix((self.data, self.indices, self.indptr), shape=self.shape)
        return self._sp

    tocsr = to_scipy

    # The reference hands out a scipy csr_matrix (storage.py:156-170), and callers
    # inspect it with scipy's own vocabulary (abs(A).sum(axis=1), A.diagonal(),
    # A[i], A.toarray(), A.T, A + B ...).  The product A @ u is the hot path and
    # runs on the device; every other matrix operation is answered by the scipy
    # view of the same arrays.
    def __getattr__(self, name):
        if name.startswith("_"):
            raise AttributeError(name)
        return getattr(self.to_scipy(), name)

    def __abs__(self):
        return abs(self.to_scipy())

    def __neg__(self):
        return -self.to_scipy()

    def __getitem__(self, key):
        return self.to_scipy()[key]

    def __add__(self, other):
        return self.to_scipy() + (other.to_scipy() if isinstance(other, DeviceCSR) else other)

    __radd__ = __add__

    def __sub__(self, other):
        return self.to_scipy() - (other.to_scipy() if isinstance(other, DeviceCSR) else other)

    def __rsub__(self, other):
        return (other.to_scipy() if isinstance(other, DeviceCSR) else other) - self.to_scipy()

    def __mul__(self, other):
        # scipy's `A * x` is the matrix-vector product: that one stays on the device
        if np.isscalar(other):
            return self.to_scipy() * other
        return self @ other

    def __rmul__(self, other):
        if np.isscalar(other):
            return other * self.to_scipy()
        return NotImplemented

    def dot(self, other):
        """A.dot(x): the device product, as A @ x."""
        return self @ other

    def __truediv__(self, other):
        return self.to_scipy() / other

    def __repr__(self):
        return f"DeviceCSR(shape={self.shape}, nnz={self.nnz})"


# ---------------------------------------------------------------------------
# weight store
# ---------------------------------------------------------------------------

class _LazyValues(Mapping):
    """{family: flat f64 host array aligned with cols}, copied from the device on
    first access.  A read-only Mapping: get(), items(), ==, dict(...) all go
    through __getitem__ (the reference's ``values`` is a plain dict)."""

    def __init__(self, store):
        self._store = store
        self._host = {}

    def __getitem__(self, key):
        if key not in self._host:
            t = self._store._values_d[key]  # KeyError for unknown families, as a dict
            self._host[key] = t.reshape(-1).cpu().numpy()
        return self._host[key]

    def __iter__(self):
        return iter(self._store._values_d)

    def __len__(self):
        return len(self._store._values_d)

    def copy(self):
        return {k: self[k] for k in self}

    def __repr__(self):
        return f"{{{', '.join(repr(k) for k in self)}}} (device-backed)"


class WeightStore:
    """Per-node stencil weights for a set of operator families, on the device.

    Weights are kept in stencil order (self first) as (m, n) float64 tensors;
    sparse-matrix views sort each row by column index, the canonical layout
    the implicit assembly uses, so explicit and assembled applications agree
    bitwise (storage.py:111-118).
    """

    def __init__(self, n_nodes, rows, stencils_d, values_d, n, rows_d=None, positions_d=None):
        self.n_nodes = int(n_nodes)
        self.positions_device = positions_d
        self._rows = np.asarray(rows, dtype=np.int64)
        self._rows_dev_hint = rows_d
        self.stencils_device = stencils_d
        self._values_d = values_d
        self.n = int(n)
        self._node_row = None
        self.values = _LazyValues(self)
        self._cols = None
        self._structure = None
        self._matrices: dict[str, DeviceCSR] = {}
        self._rows_d = None
        self._node_row_d = None

    # -- reference fields -------------------------------------------------

    @property
    def node_row(self):
        if self._node_row is None:
            nr = np.full(self.n_nodes, -1, dtype=np.int64)
            nr[self._rows] = np.arange(self._rows.shape[0])
            self._node_row = nr
        return self._node_row

    @property
    def rows(self):
        return self._rows

    @property
    def offsets(self):
        return np.arange(self._rows.shape[0] + 1, dtype=np.int64) * self.n

    @property
    def stencil_sizes(self):
        return np.full(self._rows.shape[0], self.n, dtype=np.int64)

    @property
    def cols(self):
        if self._cols is None:
            self._cols = self.stencils_device.reshape(-1).cpu().numpy().astype(np.int64)
        return self._cols

    @property
    def families(self):
        return list(self._values_d.keys())

    def values_device(self, key: str) -> torch.Tensor:
        return self._family(key)

    def rows_device(self):
        if self._rows_d is None and isinstance(self._rows_dev_hint, torch.Tensor):
            self._rows_d = self._rows_dev_hint
        if self._rows_d is None:
            self._rows_d = _lib.to_device(self._rows, torch.int64)
        return self._rows_d

    def node_row_device(self):
        if self._node_row_d is None:
            self._node_row_d = _lib.to_device(self.node_row, torch.int64)
        return self._node_row_d

    def _row(self, i: int) -> int:
        r = self.node_row[i]
        if r < 0:
            raise StorageError(f"no weights stored for node {i}")
        return int(r)

    def _family(self, key: str) -> torch.Tensor:
        try:
            return self._values_d[key]
        except KeyError:
            raise StorageError(
                f"family {key!r} not stored; available: {', '.join(self.families)}"
            ) from None

    def stencil(self, i: int):
        r = self._row(i)
        return self.cols[r * self.n:(r + 1) * self.n]

    def weights(self, key: str, i: int):
        """Weight vector for one node, aligned with its stencil."""
        self._family(key)
        r = self._row(i)
        return self.values[key][r * self.n:(r + 1) * self.n]

    def _adopt_structure(self, s, ev):
        self._structure = s
        self._structure_ev = ev

    def structure(self) -> _CsrStructure:
        """The canonical CSR structure every family shares (built once)."""
        ev = getattr(self, "_structure_ev", None)
        if ev is not None:  # built on the side stream: order after it
            torch.cuda.current_stream().wait_event(ev)
            self._structure_ev = None
        if self._structure is None:
            self._structure = _CsrStructure(self.n_nodes, self.rows_device(), self.stencils_device, self.n,
                                            self.positions_device)
        return self._structure

    @_lib.traced("meshfree.WeightStore.matrix")
    def matrix(self, key: str) -> DeviceCSR:
        """Canonical CSR view: N x N, rows only for stored nodes."""
        if key not in self._matrices:
            vals = self._family(key)
            s = self.structure()
            data = torch.empty(max(s.nnz, 1), dtype=torch.float64, device=vals.device)
            _lib.check(_lib.load().mf_csr_gather(s.perm.data_ptr(), vals.data_ptr(), s.nnz, data.data_ptr(),
                                                 _lib.stream_ptr()), "mf_csr_gather")
            self._matrices[key] = DeviceCSR(s, data)
        return self._matrices[key]

    # -- explicit application ---------------------------------------------

    def apply(self, key: str, field, i):
        """(L u)(p_i) from stored weights; matches the assembled matrix row bitwise.

        ``i`` an int gives a float (the reference's call); an index array gives
        the values at those nodes from one launch."""
        scalar = np.ndim(i) == 0
        out = self._combine([[(key, 0)]], [field], i)
        return float(out[0][0]) if scalar else out[0]

    @_lib.traced("meshfree.WeightStore.apply_all")
    def apply_all(self, key: str, field):
        """(L u) at every stored node as a length-N vector (zeros elsewhere)."""
        if isinstance(field, torch.Tensor) and field.is_cuda:
            return self.matrix(key) @ field
        arr = np.asarray(field, dtype=float)
        if arr.shape != (self.n_nodes,):
            try:
                arr = np.broadcast_to(arr, (self.n_nodes,))
            except ValueError:
                raise ValueError(f"field of shape {arr.shape} does not match the {self.n_nodes} nodes") from None
        # the field's host-to-device copy overlaps the CSR and apply-plan builds
        u_d, ready = _lib.to_device_async(arr, torch.float64)
        mat = self.matrix(key)
        mat.plan_direct()
        torch.cuda.current_stream(u_d.device).wait_event(ready)
        y = mat.apply_device(u_d)
        return _result_to_host(y, mat._s)

    def apply_families(self, keys, field):
        """{key: L_key u} at every stored node for several families in ONE pass
        over the shared stencil structure (index stream and field gathers read
        once); each result is bitwise apply_all(key, field)."""
        keys = list(keys)
        out = self._combine([[(k, 0)] for k in keys], [field], None)
        return dict(zip(keys, out))

    # -- vector calculus (storage.py:190-222).  ``i`` an int: the reference's
    # per-node result; an index array: those nodes; None: the whole field
    # (zeros at nodes without weights), each from one launch.

    def gradient(self, field, i=None):
        d = self._dim()
        out = self._combine([[(f"d1_{a}", 0)] for a in range(d)], [field], i)
        return self._shape_out(out, i)

    def divergence(self, vec_field, i=None):
        d = self._dim()
        cols = self._components(vec_field, d)
        out = self._combine([[(f"d1_{a}", a) for a in range(d)]], cols, i)
        return float(out[0][0]) if np.ndim(i) == 0 and i is not None else out[0]

    def vector_laplacian(self, vec_field, i=None):
        vec = vec_field if isinstance(vec_field, torch.Tensor) else np.asarray(vec_field, dtype=float)
        d = int(vec.shape[1])
        cols = self._components(vec, d)
        out = self._combine([[("laplacian", a)] for a in range(d)], cols, i)
        return self._shape_out(out, i)

    def grad_div(self, vec_field, i=None):
        """grad(div u); needs the hessian families."""
        d = self._dim()
        cols = self._components(vec_field, d)
        spec = [[(f"d2_{min(a, b)}_{max(a, b)}", b) for b in range(d)] for a in range(d)]
        out = self._combine(spec, cols, i)
        return self._shape_out(out, i)

    @staticmethod
    def _shape_out(out, i):
        if i is not None and np.ndim(i) == 0:
            return np.array([float(o[0]) for o in out])
        return np.stack(out, axis=-1) if isinstance(out[0], np.ndarray) else torch.stack(out, dim=-1)

    def _components(self, vec_field, d):
        if isinstance(vec_field, torch.Tensor) and vec_field.is_cuda:
            if vec_field.ndim != 2 or vec_field.shape[1] < d:
                raise ValueError(f"vector field of shape {tuple(vec_field.shape)} has fewer than {d} components")
            return [vec_field[:, a] for a in range(d)]
        vec = np.asarray(vec_field, dtype=float)
        if vec.ndim != 2 or vec.shape[1] < d:
            raise ValueError(f"vector field of shape {vec.shape} has fewer than {d} components")
        return [np.ascontiguousarray(vec[:, a]) for a in range(d)]

    def _combine(self, spec, fields, i):
        """Outputs o = ((0.0 + s_o0) + s_o1) + ... with s = row sums of (family,
        field index) terms (spec: list of outputs, each a list of terms), at node
        i / nodes i / every node (i None).  Returns host arrays for host fields,
        device tensors for device fields."""
        terms = [t for o in spec for t in o]
        if len(terms) > _lib.MF_MAX_TERMS or len(spec) > _lib.MF_MAX_TERMS:
            raise ConfigError(f"at most {_lib.MF_MAX_TERMS} terms per combination")
        for key, _ in terms:
            self._family(key)
        device_in = all(isinstance(f, torch.Tensor) and f.is_cuda for f in fields)
        flds = [_to_field(f, self.n_nodes)[0] for f in fields]
        lib = _lib.load()
        mats = {key: self.matrix(key) for key, _ in terms}
        s = self._structure
        tt = _lib.TermsT()
        tt.nterm, tt.nout = len(terms), len(spec)
        t0 = 0
        for o, out_terms in enumerate(spec):
            tt.out_t0[o] = t0
            t0 += len(out_terms)
        tt.out_t0[len(spec)] = t0
        dev = flds[0].device
        if i is None:
            order, _, ell_idx, ell_len = s.plan(True)
            n = self.n_nodes
            if order is not None:
                plan_f = []
                for f in flds:
                    g = torch.empty(n, dtype=torch.float64, device=dev)
                    _lib.check(lib.mf_permute(f.data_ptr(), order.data_ptr(), n, 0, g.data_ptr(),
                                              _lib.stream_ptr()), "mf_permute")
                    plan_f.append(g)
            else:
                plan_f = flds
            outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in spec]
            for k, (key, fi) in enumerate(terms):
                tt.val[k] = mats[key].plan(True).ell_val.data_ptr()
                tt.fld[k] = plan_f[fi].data_ptr()
            for o, y in enumerate(outs):
                tt.out[o] = y.data_ptr()
            _lib.check(lib.mf_plan_apply_terms(ell_idx.data_ptr(), ell_len.data_ptr(), n, s.n,
                                               _lib.ptr(order), ctypes.byref(tt), _lib.stream_ptr()),
                       "mf_plan_apply_terms")
        else:
            sel = np.atleast_1d(np.asarray(i, dtype=np.int64))
            for node in sel:
                self._row(int(node))  # StorageError for nodes without weights, as the reference
            sel_d = _lib.to_device(sel, torch.int64)
            outs = [torch.empty(max(sel.size, 1), dtype=torch.float64, device=dev)[: sel.size] for _ in spec]
            for k, (key, fi) in enumerate(terms):
                tt.val[k] = mats[key].data_device.data_ptr()
                tt.fld[k] = flds[fi].data_ptr()
            for o, y in enumerate(outs):
                tt.out[o] = y.data_ptr()
            _lib.check(lib.mf_apply_terms_rows(s.indptr.data_ptr(), s.indices.data_ptr(), sel_d.data_ptr(),
                                               sel.size, ctypes.byref(tt), _lib.stream_ptr()),
                       "mf_apply_terms_rows")
        if device_in:
            return outs
        host = _result_to_host(torch.stack(outs) if outs else outs, s)
        return [host[o] for o in range(len(spec))]

    def _dim(self) -> int:
        axes = [int(k[3:]) for k in self._values_d if k.startswith("d1_")]
        if not axes:
            raise StorageError("no first-derivative families stored")
        return max(axes) + 1

    # -- boundary handling ---------------------------------------------------

    def normal_combination(self, i: int, normal):
        """Stencil-ordered weights of the normal derivative at node i."""
        normal = np.asarray(normal, dtype=float)
        acc = None
        for a, na in enumerate(normal):
            part = na * self.weights(f"d1_{a}", i)
            acc = part if acc is None else acc + part
        return acc

    def neumann_plane(self, d: int) -> torch.Tensor:
        """(d, m*n) stacked d1_* weights for the Neumann kernel."""
        for a in range(d):
            self._family(f"d1_{a}")
        return torch.stack([self._values_d[f"d1_{a}"].reshape(-1) for a in range(d)]).contiguous()

    def neumann_values_device(self, nodes_idx, normals, gn, u_d, *, plane=None, normals_d=None):
        """Batched neumann_value on the GPU -> (values tensor, lowest bad list position or None)."""
        lib = _lib.load()
        nodes_idx = np.asarray(nodes_idx, dtype=np.int64)
        for i in nodes_idx:
            self._row(int(i))
        d = normals.shape[1]
        plane = self.neumann_plane(d) if plane is None else plane
        nd = _lib.to_device(nodes_idx, torch.int64)
        normals_d = _lib.to_device(normals, torch.float64) if normals_d is None else normals_d
        g_d = _lib.to_device(np.broadcast_to(np.asarray(gn, dtype=float), nodes_idx.shape), torch.float64)
        nm = _lib.NeumannT(self.stencils_device.data_ptr(), self.n, plane.data_ptr(), plane.shape[1], d,
                           normals_d.data_ptr(), nd.data_ptr(), self.node_row_device().data_ptr(),
                           g_d.data_ptr(), nodes_idx.shape[0], None)
        out = torch.empty(max(nodes_idx.shape[0], 1), dtype=torch.float64, device=u_d.device)
        bad = torch.empty(1, dtype=torch.int64, device=u_d.device)
        _lib.check(lib.mf_neumann_values(ctypes.byref(nm), u_d.data_ptr(), out.data_ptr(), None, None,
                                         bad.data_ptr(), _lib.stream_ptr()), "mf_neumann_values")
        b = int(bad.item())
        return out[: nodes_idx.shape[0]], (None if b == _lib.SENTINEL_OK else b)

    def neumann_value(self, field, i: int, normal, gn: float) -> float:
        """Value at node i enforcing w . u = gn with the node's own weight as pivot."""
        u_d, _ = _to_field(field, self.n_nodes)
        normal = np.asarray(normal, dtype=float).reshape(1, -1)
        vals, bad = self.neumann_values_device([int(i)], normal, [float(gn)], u_d)
        if bad is not None:
            raise NumericalError(
                f"node {i}: negligible self-weight in the normal derivative; "
                "the stencil cannot enforce a Neumann condition explicitly"
            )
        return float(vals[0].item())

    def rows_in_order(self):
        return self._rows


# ---------------------------------------------------------------------------
# compute_weights
# ---------------------------------------------------------------------------

_HOST_ARANGE = {}


def _host_arange(n: int) -> np.ndarray:
    """Cached read-only int64 0..n-1 (row lists of full node sets)."""
    a = _HOST_ARANGE.get(n)
    if a is None:
        a = np.arange(n, dtype=np.int64)
        a.flags.writeable = False
        if len(_HOST_ARANGE) > 8:
            _HOST_ARANGE.clear()
        _HOST_ARANGE[n] = a
    return a


@_lib.traced("meshfree.compute_weights")
def compute_weights(nodes, engine, families, for_which=None) -> WeightStore:
    """Evaluate ``engine`` on every selected node for all families (storage.py:258-307).

    ``engine`` is a single engine, or a mapping from family specs to engines.
    ``for_which=None`` means every node that has a stencil; nodes selected
    explicitly must all have stencils.
    """
    full = nodes.full_block_matrix() if for_which is None else None
    if full is not None:
        # every node has a stencil, in index order: no host index bookkeeping
        rows = _host_arange(len(nodes))
    elif for_which is None:
        rows = np.flatnonzero(nodes._blk >= 0).astype(np.int64)
        if rows.size == 0:
            raise StencilError("no node has a stencil; run find_closest_stencils first")
    else:
        rows = nodes.select(for_which).astype(np.int64)
        if rows.size > 1 and not np.all(rows[1:] > rows[:-1]) and np.unique(rows).size != rows.size:
            # the canonical CSR keeps one row per node; the reference would store the
            # duplicated row twice and let scipy sum both copies (a caller error)
            raise StorageError("stored rows must be distinct node indices")

    fams = expand_families(families, nodes.dim)
    if isinstance(engine, dict):
        assign = {}
        for spec, eng in engine.items():
            try:
                keys = list(expand_families([spec], nodes.dim))
            except StorageError:
                keys = [str(spec)]
            for key in keys:
                if key in assign:
                    raise StorageError(f"family {key!r} mapped to two engines")
                assign[key] = eng
        missing_f = [k for k in fams if k not in assign]
        if missing_f:
            raise StorageError(f"no engine given for families {missing_f}")
        groups = []
        for eng in dict.fromkeys(assign.values()):
            sub = {k: op for k, op in fams.items() if assign[k] is eng}
            if sub:
                groups.append((eng, sub))
    else:
        groups = [(engine, fams)]
    for eng, sub in groups:
        _check_engine(eng, sub)
    if rows.size == 0:
        # nothing selected (e.g. "boundary" on a set without boundary nodes): an
        # empty store, as the reference returns
        dev = _lib.device()
        empty = torch.empty((0, 0), dtype=torch.int32, device=dev)
        return WeightStore(len(nodes), rows, empty, {k: torch.empty((0, 0), dtype=torch.float64, device=dev)
                                                     for k in fams}, 0,
                           rows_d=torch.empty(0, dtype=torch.int64, device=dev),
                           positions_d=nodes.positions_device())
    if full is not None:
        stencils_d = full
        rows_d = _lib.device_arange(len(nodes))
    else:
        missing = np.flatnonzero(nodes._blk[rows] < 0)
        if missing.size:
            raise StencilError(f"node {int(rows[missing[0]])} has no stencil")
        stencils_d = nodes.stencil_matrix_device(rows)
        rows_d = _lib.to_device(rows, torch.int64)
    n = int(stencils_d.shape[1]) if rows.size else 0
    # the canonical CSR structure and the locality order depend on the stencils
    # only: on large stores they are built on a side stream while the shape
    # solve (and its re-solve pass, which leaves most SMs idle) runs
    pre = _structure_async(len(nodes), rows_d, stencils_d, n, nodes.positions_device()) \
        if rows.size >= ASYNC_STRUCTURE_ROWS else None
    values = {}
    for eng, sub in groups:
        if _batchable(eng, sub):
            values.update(_run_batch(nodes, eng, sub, rows, rows_d, stencils_d, n))
        else:
            values.update(_run_general(nodes, eng, sub, rows, rows_d, stencils_d, n))
    values = {k: values[k] for k in fams}
    store = WeightStore(len(nodes), rows, stencils_d, values, n, rows_d=rows_d,
                       positions_d=nodes.positions_device())
    if pre is not None:
        store._adopt_structure(*pre)
    return store


_ELEMENTARY = (Identity, FirstDerivative, SecondDerivative, Laplacian)
_GENERAL_TERMS = _ELEMENTARY + (Directional,)
_RBF_CODES = {Polyharmonic: _lib.MF_RBF_PHS, Gaussian: _lib.MF_RBF_GAUSSIAN,
              Multiquadric: _lib.MF_RBF_MQ, InverseMultiquadric: _lib.MF_RBF_IMQ}


def _batchable(engine, fams) -> bool:
    """The reference's own batch criterion (storage.py:310-322)."""
    return (isinstance(engine, RbfFd) and isinstance(engine.rbf, Polyharmonic)
            and engine.solver == "lu" and engine.rbf.exponent >= 3
            and engine.scale in SCALE_CODES
            and all(isinstance(op, _ELEMENTARY) for op in fams.values()))


def _check_engine(engine, fams):
    """ConfigError for what cannot run on the GPU at all (Python-defined
    kernels, weights or operators); everything else is batched or general."""
    if isinstance(engine, RbfFd):
        if type(engine.rbf) not in _RBF_CODES:
            raise ConfigError(f"{engine!r}: kernel {engine.rbf!r} has no GPU implementation")
    elif isinstance(engine, WeightedLeastSquares):
        if not isinstance(engine.weight, (ConstantWeight, GaussianWeight)):
            raise ConfigError(f"{engine!r}: weight function {engine.weight!r} has no GPU implementation")
    else:
        raise ConfigError(f"{engine!r}: unknown weight engine")
    for key, op in fams.items():
        for _, elem in op.terms():
            if not isinstance(elem, _GENERAL_TERMS):
                raise ConfigError(f"family {key!r}: operator {elem!r} has no GPU implementation")
    if _batchable(engine, fams):
        _check_batchable(engine)


ASYNC_STRUCTURE_ROWS = 1 << 16


def _structure_async(n_nodes, rows_d, stencils_d, n, positions_d):
    """(_CsrStructure, event): the structure and its Morton order built on the
    side stream after the stencils are ready; the event marks completion."""
    main = torch.cuda.current_stream()
    side = _lib.side_stream()
    side.wait_stream(main)
    with torch.cuda.stream(side):
        s = _CsrStructure(n_nodes, rows_d, stencils_d, n, positions_d)
        s._order(True)
        ev = torch.cuda.Event()
        ev.record(side)
    for t in (rows_d, stencils_d, positions_d):
        if isinstance(t, torch.Tensor):
            t.record_stream(side)
    for t in (s.indptr, s.indices, s.perm, s._dup) + tuple(s._morton or ()):
        t.record_stream(main)
    return s, ev


def _check_batchable(engine):
    if not isinstance(engine, RbfFd) or not isinstance(engine.rbf, Polyharmonic):
        raise ConfigError(
            f"{engine!r}: the GPU path implements the batched RbfFd(Polyharmonic) engine only"
        )
    if engine.solver != "lu":
        raise ConfigError(f"{engine!r}: the GPU path implements solver='lu' only")
    if engine.rbf.exponent < 3:
        raise ConfigError(f"{engine!r}: polyharmonic exponent must be >= 3 on the batched path")
    if engine.scale not in SCALE_CODES:
        raise ConfigError(f"unknown scale rule {engine.scale!r}; use none, nearest or support")
    if engine.mode not in MODES:
        raise ConfigError(f"unknown shape-solve mode {engine.mode!r}; use hybrid, replay or fast")


def encode_families(fams: dict, dim: int, degree: int):
    """(kinds, ax_a, ax_b, orders, expos, base_bot) as in storage.py:349-380."""
    kinds, ax_a, ax_b, orders = [], [], [], []
    for key, op in fams.items():
        if isinstance(op, Identity):
            kinds.append(KIND_IDENTITY); ax_a.append(0); ax_b.append(0)
        elif isinstance(op, FirstDerivative):
            kinds.append(KIND_D1); ax_a.append(op.axis); ax_b.append(0)
        elif isinstance(op, SecondDerivative):
            kinds.append(KIND_D2); ax_a.append(op.a); ax_b.append(op.b)
        elif isinstance(op, Laplacian):
            kinds.append(KIND_LAPLACIAN); ax_a.append(0); ax_b.append(0)
        else:
            raise ConfigError(f"family {key!r}: custom operators are not supported on the GPU path")
        orders.append(op.order)
    if degree >= 0:
        expos = np.array(graded_lex_exponents(dim, degree), dtype=np.int32).reshape(-1, dim)
        basis = MonomialBasis(dim, degree)
        base_bot = np.stack([basis.origin_row(op) for op in fams.values()], axis=0)
    else:
        expos = np.empty((0, dim), dtype=np.int32)
        base_bot = np.zeros((len(fams), 0))
    as32 = lambda v: np.ascontiguousarray(np.array(v, dtype=np.int32))
    return (as32(kinds), as32(ax_a), as32(ax_b), as32(orders), np.ascontiguousarray(expos),
            np.ascontiguousarray(base_bot, dtype=np.float64))


def phs_weights_device(pos_d, rows_d, stencils_d, engine, fams: dict, dim: int, *, mode=None,
                       threshold: float = 0.0, kappa=None, min_separation: float = 0.0):
    """Run mf_phs_weights -> ((m, nf, n) f64 weights, status, first_fail, n_replayed) tensors.

    ``threshold`` overrides the HYBRID re-solve threshold; ``kappa`` (a device
    f64 tensor of m entries) receives the per-stencil conditioning estimate.
    """
    lib = _lib.load()
    kinds, ax_a, ax_b, orders, expos, base_bot = encode_families(fams, dim, engine.degree)
    m, n = int(stencils_d.shape[0]), int(stencils_d.shape[1])
    nf = len(fams)
    if nf > _lib.MF_MAX_FAMILIES or expos.shape[0] > _lib.MF_MAX_MONOMIALS:
        raise ConfigError("too many families or monomials for the batched kernel")
    dev = pos_d.device
    out = torch.empty((m, nf, n), dtype=torch.float64, device=dev)
    status = torch.empty(max(m, 1), dtype=torch.int8, device=dev)
    first_fail = torch.empty(1, dtype=torch.int64, device=dev)
    n_rep = torch.empty(1, dtype=torch.int64, device=dev)
    mode_code = MODES[mode or engine.mode]
    size = ctypes.c_size_t(0)
    _lib.check(lib.mf_phs_workspace_size(m, ctypes.byref(size)), "mf_phs_workspace_size")
    ws = _lib.workspace(size.value)
    opts = _lib.PhsOptions(float(threshold), _lib.ptr(kappa), float(min_separation))
    _lib.check(lib.mf_phs_weights(
        pos_d.data_ptr(), int(pos_d.shape[0]), dim, rows_d.data_ptr(), stencils_d.data_ptr(), m, n,
        engine.rbf.exponent, int(engine.rbf.even), expos.ctypes.data, int(expos.shape[0]),
        base_bot.ctypes.data, kinds.ctypes.data, ax_a.ctypes.data, ax_b.ctypes.data, orders.ctypes.data,
        nf, SCALE_CODES[engine.scale], mode_code, out.data_ptr(), status.data_ptr(),
        first_fail.data_ptr(), n_rep.data_ptr(), ctypes.byref(opts), ws.data_ptr(), size.value,
        _lib.stream_ptr()),
        "mf_phs_weights")
    return out, status, first_fail, n_rep


def _run_batch(nodes, engine, fams, rows, rows_d, stencils_d, n):
    _check_batchable(engine)
    dim = nodes.dim
    if engine.degree >= 0:
        l = len(graded_lex_exponents(dim, engine.degree))
        if l > n:
            raise WeightError(
                int(rows[0]),
                f"augmentation of degree {engine.degree} needs at least {l} stencil nodes, got {n}",
            )
    pos_d = nodes.positions_device()
    out, status, first_fail, _ = phs_weights_device(pos_d, rows_d, stencils_d, engine, fams, dim)
    bad = int(first_fail.item())
    if bad != _lib.SENTINEL_OK:
        node = int(rows[bad])
        if int(status[bad].item()) == 2:
            raise WeightError(node, "all stencil nodes coincide with the center")
        raise WeightError(node, "singular local collocation system; try a larger stencil")
    # (m, nf, n) -> per family (m, n)
    return {key: out[:, f, :].contiguous() for f, key in enumerate(fams)}


_ENGINE_MESSAGES = {
    2: "all stencil nodes coincide with the center",
    4: "weight function must be positive on the stencil",
}
_NONFINITE = {
    True: "least squares fit produced non-finite weights (singular local system); use the qr or svd solver",
    False: "local collocation produced non-finite weights (degenerate stencil geometry?); try a larger stencil",
}


def encode_engine(engine, fams: dict, dim: int, n: int):
    """mf_engine_t for the general kernel, or raise the reference's per-node error
    text for the first family (rows are checked by the caller)."""
    e = _lib.EngineT()
    wls = isinstance(engine, WeightedLeastSquares)
    e.engine = _lib.MF_ENGINE_WLS if wls else _lib.MF_ENGINE_RBFFD
    e.d = dim
    first = next(iter(fams))
    if engine.scale not in SCALE_CODES:
        raise _EngineSetupError(first, f"unknown scale rule {engine.scale!r}; use none, nearest or support", True)
    e.scale_code = SCALE_CODES[engine.scale]
    solvers = {"lu": _lib.MF_SOLVER_LU, "qr": _lib.MF_SOLVER_QR, "svd": _lib.MF_SOLVER_SVD}
    if wls:
        try:
            basis = engine._resolve_basis(dim)
        except ConfigError as exc:
            raise _EngineSetupError(first, str(exc), True) from None
        expos = [tuple(x) for x in basis.exponents]
        if isinstance(engine.weight, GaussianWeight):
            e.weight, e.weight_sigma = _lib.MF_WEIGHT_GAUSSIAN, engine.weight.sigma
        else:
            e.weight = _lib.MF_WEIGHT_CONSTANT
        if engine.solver == "lu" and len(expos) != n:
            raise _EngineSetupError(
                first, f"lu needs a square local system, got {(len(expos), n)}; use qr or svd")
    else:
        rbf = engine.rbf
        e.rbf = _RBF_CODES[type(rbf)]
        if isinstance(rbf, Polyharmonic):
            e.k = rbf.exponent
        else:
            e.sigma = rbf.sigma
        expos = graded_lex_exponents(dim, engine.degree) if engine.degree >= 0 else []
        if len(expos) > n:
            raise _EngineSetupError(
                first, f"augmentation of degree {engine.degree} needs at least {len(expos)} stencil nodes, got {n}")
    if engine.solver not in solvers:
        raise _EngineSetupError(first, f"unknown dense solver {engine.solver!r}; use lu, qr or svd", True)
    e.solver = solvers[engine.solver]
    if len(expos) > _lib.MF_MAX_MONOMIALS or len(fams) > _lib.MF_MAX_FAMILIES:
        raise ConfigError("too many families or monomials for the general engine kernel")
    unknowns = (min(len(expos), n) if wls else n + len(expos))
    if (engine.solver == "svd" and unknowns > 128) or (engine.solver == "qr" and unknowns > 256):
        raise ConfigError("local system too large for the GPU svd (128 unknowns) / qr (256) solver")
    e.l = len(expos)
    for j, ex in enumerate(expos):
        for a in range(dim):
            e.expos[j * _lib.MF_MAX_DIM + a] = int(ex[a])
    e.nf = len(fams)
    t = 0
    e.term0[0] = 0
    for f, (key, op) in enumerate(fams.items()):
        for coeff, elem in op.terms():
            if t >= _lib.MF_MAX_ENGINE_TERMS:
                raise ConfigError(f"more than {_lib.MF_MAX_ENGINE_TERMS} operator terms in one call")
            e.term_coeff[t] = float(coeff)
            e.term_order[t] = int(elem.order)
            if isinstance(elem, Identity):
                e.term_kind[t] = _lib.MF_TERM_IDENTITY
            elif isinstance(elem, FirstDerivative):
                e.term_kind[t], e.term_a[t] = _lib.MF_TERM_D1, elem.axis
            elif isinstance(elem, SecondDerivative):
                e.term_kind[t], e.term_a[t], e.term_b[t] = _lib.MF_TERM_D2, elem.a, elem.b
            elif isinstance(elem, Laplacian):
                e.term_kind[t] = _lib.MF_TERM_LAPLACIAN
            else:
                e.term_kind[t] = _lib.MF_TERM_DIRECTIONAL
                for a, v in enumerate(np.asarray(elem.vector, dtype=float)[:dim]):
                    e.term_vec[t * _lib.MF_MAX_DIM + a] = float(v)
            axes = [e.term_a[t], e.term_b[t]]
            if max(axes) >= dim:
                raise _EngineSetupError(key, f"axis out of range for dimension {dim}")
            t += 1
        e.term0[f + 1] = t
    return e


class _EngineSetupError(Exception):
    """A failure the reference raises from engine.weights() before any solve; `config`
    marks the ones it raises as ConfigError there (unknown scale rule / solver, basis
    dimension), the rest are NumericalError.  compute_weights wraps either into
    WeightError (storage.py:333-337); engine.weights() re-raises the original class."""

    def __init__(self, key, msg, config=False):
        self.key, self.msg, self.config = key, msg, config


def engine_weights_device(pos_d, rows_d, stencils_d, engine, fams: dict, dim: int):
    """Run mf_engine_weights -> ((m, nf, n) f64 weights, (m, nf) status, first_fail)."""
    lib = _lib.load()
    m, n = int(stencils_d.shape[0]), int(stencils_d.shape[1])
    e = encode_engine(engine, fams, dim, n)
    dev = pos_d.device
    out = torch.empty((m, len(fams), n), dtype=torch.float64, device=dev)
    status = torch.empty((max(m, 1), len(fams)), dtype=torch.int8, device=dev)
    first_fail = torch.empty(1, dtype=torch.int64, device=dev)
    _lib.check(lib.mf_engine_weights(pos_d.data_ptr(), int(pos_d.shape[0]), rows_d.data_ptr(),
                                     stencils_d.data_ptr(), m, n, ctypes.byref(e), out.data_ptr(),
                                     status.data_ptr(), first_fail.data_ptr(), _lib.stream_ptr()),
               "mf_engine_weights")
    return out, status, first_fail


def _run_general(nodes, engine, fams, rows, rows_d, stencils_d, n):
    """The per-node loop of the reference (storage.py:325-339), batched on the
    GPU: same weights up to rounding, same WeightError (lowest failing node,
    first failing family, the engine's message)."""
    dim = nodes.dim
    pos_d = nodes.positions_device()
    try:
        out, status, first_fail = engine_weights_device(pos_d, rows_d, stencils_d, engine, fams, dim)
    except _EngineSetupError as exc:
        err = WeightError(int(rows[0]), f"family {exc.key!r}: {exc.msg}")
        err.config = exc.config
        raise err from None
    bad = int(first_fail.item())
    if bad != _lib.SENTINEL_OK:
        codes = status[bad].cpu().numpy()
        f = int(np.flatnonzero(codes)[0])
        code = int(codes[f])
        key = list(fams)[f]
        if code == 1:
            msg = _NONFINITE[isinstance(engine, WeightedLeastSquares)]
        elif code == 3:
            msg = (f"derivatives of polyharmonic r^{engine.rbf.exponent} are singular "
                   "at the stencil center; use an exponent of 3 or more")
        else:
            msg = _ENGINE_MESSAGES[code]
        raise WeightError(int(rows[bad]), f"family {key!r}: {msg}")
    return {key: out[:, f, :].contiguous() for f, key in enumerate(fams)}
