"""Preconditioned iterative solution of assembled systems, on the GPU.

Drop-in for the reference's solve module (solve.py:1-108): ``SolverConfig``,
``SolveResult``, ``make_preconditioner`` and ``solve_sparse`` with the same
arguments, validation, convergence rule (scipy's bicgstab recurrence, stop at
||r|| < max(atol, tol ||b||), x0 = one preconditioned Richardson step) and
NumericalError texts.

The reference preconditions with SuperLU's ILUT (``spilu``, dual threshold,
fill_factor / drop_tol); that factorisation is sequential.  Here the
preconditioner is ILU(0) in a multicolour order (``mf_ilu0_build``): the
pattern is coloured so rows of one colour never couple, and the factorisation
and both substitutions run colour by colour on the device.  ``"ilut"`` (the
reference's default) selects it, as does ``"ilu0"``; fill_factor and drop_tol
are validated as in the reference but have no effect.  BiCGStab then reaches
the same relative residual as the reference's run, so the solutions agree to
cond(A) * tol; iteration counts differ (reported in ``info``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, NumericalError


@dataclass
class SolverConfig:
    """Iterative solver settings (solve.py:14-38)."""

    method: str = "bicgstab"
    preconditioner: str = "ilut"
    fill_factor: float = 5.0
    drop_tol: float = 1e-2
    tol: float = 1e-10
    max_iter: int = 0

    def validate(self):
        if self.method != "bicgstab":
            raise ConfigError(f"unknown solver method {self.method!r}")
        if self.preconditioner not in ("ilut", "ilu0", "none"):
            raise ConfigError(f"unknown preconditioner {self.preconditioner!r}")
        if self.tol <= 0 or self.fill_factor < 1 or self.drop_tol < 0 or self.max_iter < 0:
            raise ConfigError("solver parameters out of range")


@dataclass
class SolveResult:
    u: np.ndarray
    iterations: int
    residual: float  # recomputed |M u - r| / |r|
    converged: bool
    info: dict = field(default_factory=dict)


class SystemMatrix:
    """Square CSR matrix on the device (canonical: rows ascending, columns
    ascending within a row).  ``indptr`` / ``indices`` / ``data`` give host
    arrays (int32, int32, float64, as scipy stores them); ``@`` multiplies on
    the GPU (row sums in storage order from 0.0, bitwise scipy's csr_matvec)."""

    def __init__(self, indptr_d, indices_d, data_d, n):
        self.indptr_device = indptr_d
        self.indices_device = indices_d
        self.data_device = data_d
        self.shape = (int(n), int(n))
        self._host = {}

    @property
    def nnz(self) -> int:
        return int(self.data_device.shape[0])

    def _get(self, name, t):
        if name not in self._host:
            self._host[name] = t.cpu().numpy()
        return self._host[name]

    @property
    def indptr(self):
        return self._get("indptr", self.indptr_device)

    @property
    def indices(self):
        return self._get("indices", self.indices_device)

    @property
    def data(self):
        return self._get("data", self.data_device)

    def matvec_device(self, x_d: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        y = out if out is not None else torch.empty(self.shape[0], dtype=torch.float64, device=x_d.device)
        _lib.check(_lib.load().mf_apply(self.indptr_device.data_ptr(), self.indices_device.data_ptr(),
                                        self.data_device.data_ptr(), x_d.data_ptr(), y.data_ptr(),
                                        self.shape[0], _lib.stream_ptr()), "mf_apply")
        return y

    def __matmul__(self, x):
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return self.matvec_device(x.to(torch.float64).contiguous())
        x = np.asarray(x, dtype=float)
        if x.shape != (self.shape[1],):
            raise ValueError(f"dimension mismatch: {x.shape} for a {self.shape} matrix")
        return self.matvec_device(_lib.to_device(x, torch.float64)).cpu().numpy()

    def to_scipy(self):
        """The same matrix as a scipy csr_matrix over host copies of the arrays (built once)."""
        if self._host.get("scipy") is None:
            import scipy.sparse

            self._host["scipy"] = scipy.sparse.csr_matrix((self.data, self.indices, self.indptr), shape=self.shape)
        return self._host["scipy"]

    tocsr = to_scipy

    # finalize() hands out a scipy csr_matrix in the reference (assembly.py:96-105): the
    # product runs on the device, any other scipy operation on the view of the same arrays
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
        return self.to_scipy() + (other.to_scipy() if hasattr(other, "to_scipy") else other)

    __radd__ = __add__

    def __sub__(self, other):
        return self.to_scipy() - (other.to_scipy() if hasattr(other, "to_scipy") else other)

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

    @classmethod
    def from_any(cls, matrix):
        """SystemMatrix from a SystemMatrix, a weight store's DeviceCSR, or anything
        scipy.sparse.csr_matrix accepts (uploaded with sorted column indices)."""
        if isinstance(matrix, SystemMatrix):
            return matrix
        from .storage import DeviceCSR

        if isinstance(matrix, DeviceCSR):
            return cls(matrix.indptr_device, matrix.indices_device, matrix.data_device[: matrix.nnz],
                       matrix.shape[0])
        import scipy.sparse

        m = scipy.sparse.csr_matrix(matrix)
        if m.shape[0] != m.shape[1]:
            raise ConfigError(f"the system matrix must be square, got {m.shape}")
        m = m.copy()
        m.sum_duplicates()
        m.sort_indices()
        return cls(_lib.to_device(m.indptr.astype(np.int32), torch.int32),
                   _lib.to_device(m.indices.astype(np.int32), torch.int32),
                   _lib.to_device(m.data.astype(np.float64), torch.float64), m.shape[0])

    def __repr__(self):
        return f"SystemMatrix(shape={self.shape}, nnz={self.nnz})"


class Ilu0Preconditioner:
    """Multicolour ILU(0) of a SystemMatrix on the device (``mf_ilu0_build``).

    ``matvec`` mirrors the reference's LinearOperator (numpy in, numpy out);
    ``apply_device`` works on device tensors."""

    def __init__(self, matrix: SystemMatrix):
        lib = _lib.load()
        dev = matrix.data_device.device
        N, nnz = matrix.shape[0], matrix.nnz
        self.matrix = matrix
        self.color = torch.empty(N, dtype=torch.int32, device=dev)
        self.order = torch.empty(N, dtype=torch.int32, device=dev)
        self.part = torch.empty(max(nnz, 1), dtype=torch.int8, device=dev)
        self.diag = torch.empty(N, dtype=torch.int32, device=dev)
        self.lu = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
        self.desc = _lib.Ilu0T()
        zp = torch.empty(1, dtype=torch.int64, device=dev)
        size = ctypes.c_size_t(0)
        _lib.check(lib.mf_ilu0_workspace_size(N, ctypes.byref(size)), "mf_ilu0_workspace_size")
        ws = _lib.workspace(size.value)
        _lib.check(lib.mf_ilu0_build(matrix.indptr_device.data_ptr(), matrix.indices_device.data_ptr(),
                                     matrix.data_device.data_ptr(), N, nnz, self.color.data_ptr(),
                                     self.order.data_ptr(), self.part.data_ptr(), self.diag.data_ptr(),
                                     self.lu.data_ptr(), ctypes.byref(self.desc), zp.data_ptr(), ws.data_ptr(),
                                     size.value, _lib.stream_ptr()), "mf_ilu0_build")
        bad = int(zp.item())
        if bad != _lib.SENTINEL_OK:
            raise NumericalError(f"incomplete LU factorization failed: row {bad} has no diagonal entry")
        piv = self.lu[self.diag.long()]
        ok = torch.isfinite(piv) & (piv != 0)
        if not bool(ok.all()):
            row = int(torch.nonzero(~ok)[0, 0])
            raise NumericalError(f"incomplete LU factorization failed: zero or non-finite pivot in row {row}")
        self.shape = matrix.shape
        self.ncolors = int(self.desc.ncolors)

    def apply_device(self, x_d: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        y = out if out is not None else torch.empty_like(x_d)
        _lib.check(_lib.load().mf_ilu0_apply(ctypes.byref(self.desc), x_d.data_ptr(), y.data_ptr(),
                                             _lib.stream_ptr()), "mf_ilu0_apply")
        return y

    def matvec(self, x):
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return self.apply_device(x.to(torch.float64).contiguous())
        return self.apply_device(_lib.to_device(np.asarray(x, dtype=float), torch.float64)).cpu().numpy()

    def __repr__(self):
        return f"Ilu0Preconditioner(n={self.shape[0]}, colors={self.ncolors})"


def make_preconditioner(matrix, config: SolverConfig):
    """Multicolour ILU(0) on the device, or None (solve.py:49-62)."""
    if config.preconditioner == "none":
        return None
    return Ilu0Preconditioner(SystemMatrix.from_any(matrix))


def _finalize(system):
    # (device matrices answer unknown attributes through their scipy view: ask the type, not the object)
    if hasattr(type(system), "finalize"):
        return system.finalize()
    raise ConfigError("solve_sparse needs a SparseSystem or a matrix and a right-hand side")


@_lib.traced("meshfree.solve_sparse")
def solve_sparse(system, rhs=None, config: SolverConfig | None = None,
                 preconditioner=None, *, return_device: bool = False) -> SolveResult:
    """Solve ``M u = r`` from a SparseSystem or an explicit (matrix, rhs) (solve.py:65-108).

    The reported residual is recomputed from the returned solution, not taken
    from the iteration, so it holds whatever the solver claims.
    """
    if rhs is None:
        matrix, rhs = _finalize(system)
    else:
        matrix = system
    matrix = SystemMatrix.from_any(matrix)
    config = config or SolverConfig()
    config.validate()
    N = matrix.shape[0]
    if isinstance(rhs, torch.Tensor) and rhs.is_cuda:
        b_d = rhs.to(torch.float64).contiguous()
    else:
        rhs = np.asarray(rhs, dtype=float)
        if rhs.shape != (N,):
            raise ValueError(f"right-hand side of shape {rhs.shape} for a {matrix.shape} system")
        b_d = _lib.to_device(rhs, torch.float64)

    if preconditioner is None:
        preconditioner = make_preconditioner(matrix, config)
    max_iter = config.max_iter if config.max_iter > 0 else 10 * N

    # one preconditioned Richardson step as the initial guess (solve.py:88-94)
    if preconditioner is not None:
        x_d = preconditioner.apply_device(b_d)
        desc = ctypes.byref(preconditioner.desc)
    else:
        x_d = b_d.clone()
        desc = None
    iters, info, rnorm = _bicgstab_graph(matrix, desc, b_d, x_d, float(config.tol), int(max_iter))
    r_d = matrix.matvec_device(x_d)
    r_d.sub_(b_d)
    rhs_norm = float(torch.linalg.vector_norm(b_d))
    residual = float(torch.linalg.vector_norm(r_d)) / (rhs_norm if rhs_norm else 1.0)
    if info != 0:
        raise NumericalError(
            f"bicgstab failed to converge in {iters} iterations "
            f"(info={info}, residual={residual:.3e})"
        )
    u = x_d if return_device else x_d.cpu().numpy()
    extra = {"preconditioner": repr(preconditioner), "recurrence_residual": rnorm}
    return SolveResult(u=u, iterations=int(iters), residual=residual, converged=True, info=extra)


_STATE_DT = np.dtype([("d", "<f8", 10), ("it", "<i8"), ("maxiter", "<i8"), ("done", "<i4"), ("info", "<i4"),
                      ("pad", "<i4"), ("pad2", "<i4")])


def _bicgstab_graph(matrix, desc, b_d, x_d, tol, max_iter, replays=8):
    """scipy's bicgstab (mf_bicgstab_init / _iter): one iteration captured as a
    CUDA graph and replayed in batches; the device state stops every kernel at
    convergence, so over-shooting a batch changes nothing.  Returns (iterations,
    info, last ||r||)."""
    lib = _lib.load()
    N = matrix.shape[0]
    dev = x_d.device
    size = ctypes.c_size_t(0)
    _lib.check(lib.mf_bicgstab_workspace_size(N, ctypes.byref(size)), "mf_bicgstab_workspace_size")
    ws = torch.empty(max(size.value, 1), dtype=torch.uint8, device=dev)  # owned: the graph holds its pointers
    st_size = ctypes.c_size_t(0)
    _lib.check(lib.mf_bicgstab_state_size(ctypes.byref(st_size)), "mf_bicgstab_state_size")
    state = torch.zeros(max(st_size.value, _STATE_DT.itemsize), dtype=torch.uint8, device=dev)
    ptrs = (matrix.indptr_device.data_ptr(), matrix.indices_device.data_ptr(), matrix.data_device.data_ptr())
    _lib.check(lib.mf_bicgstab_init(*ptrs, N, b_d.data_ptr(), x_d.data_ptr(), tol, 0.0, int(max_iter),
                                    state.data_ptr(), ws.data_ptr(), size.value, _lib.stream_ptr()),
               "mf_bicgstab_init")

    def read():
        return np.frombuffer(state[: _STATE_DT.itemsize].cpu().numpy().tobytes(), dtype=_STATE_DT)[0]

    s = read()
    if s["done"] == 3:  # b == 0: x = b (solve.py: scipy returns b)
        x_d.copy_(b_d)
        return 0, 0, 0.0
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        # (capture_begin/end directly: the torch.cuda.graph context manager runs a
        # full gc.collect() on entry, which costs more than a short solve)
        graph.capture_begin()
        try:
            _lib.check(lib.mf_bicgstab_iter(*ptrs, N, desc, x_d.data_ptr(), state.data_ptr(), ws.data_ptr(),
                                            size.value, _lib.stream_ptr()), "mf_bicgstab_iter")
        finally:
            graph.capture_end()
    torch.cuda.current_stream(dev).wait_stream(side)
    while True:
        for _ in range(replays):
            graph.replay()
        s = read()
        if s["done"]:
            return int(s["it"]), int(s["info"]), float(np.sqrt(s["d"][6]))
        replays = min(replays * 2, 256)
