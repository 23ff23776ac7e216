"""ctypes binding of libmeshfree_b200.so (the C ABI in include/meshfree_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every GPU entry point raises.  Device memory, streams and the caching
allocator come from PyTorch; the library itself never allocates.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MF_LIB_PATH") or os.path.join(HERE, "libmeshfree_b200.so")  # override: A/B builds

MF_OK = 0
MF_ERR_UNSUPPORTED = 3
MF_MAX_FAMILIES = 16
MF_MAX_MONOMIALS = 128
PHS_REPLAY, PHS_FAST, PHS_HYBRID = 0, 1, 2

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double
_SZ = ctypes.c_size_t


class PhsOptions(ctypes.Structure):
    _fields_ = [("hybrid_threshold", _D), ("kappa", _P), ("min_separation", _D)]


class NeumannT(ctypes.Structure):
    _fields_ = [
        ("stencils", _P), ("n", _I32), ("w_d1", _P), ("mn", _I64), ("d", _I32),
        ("normals", _P), ("nodes", _P), ("node_row", _P), ("gn", _P), ("count", _I64),
        ("mask", _P),
    ]


MF_MAX_TERMS = 16


class TermsT(ctypes.Structure):
    """mf_terms_t (include/meshfree_b200.h): row sums of (family, field) terms, summed per output."""
    _fields_ = [("nterm", _I32), ("nout", _I32), ("val", _P * MF_MAX_TERMS), ("fld", _P * MF_MAX_TERMS),
                ("out_t0", _I32 * (MF_MAX_TERMS + 1)), ("out", _P * MF_MAX_TERMS)]


class HeatPackT(ctypes.Structure):
    """mf_heat_pack_t (include/meshfree_b200.h)."""
    _fields_ = [("ell_d16", _P), ("meta", _P), ("tile_wide", _P)]


MF_MAX_DIM = 3
MF_MAX_ENGINE_TERMS = 32
MF_ENGINE_RBFFD, MF_ENGINE_WLS = 0, 1
MF_RBF_PHS, MF_RBF_GAUSSIAN, MF_RBF_MQ, MF_RBF_IMQ = 0, 1, 2, 3
MF_WEIGHT_CONSTANT, MF_WEIGHT_GAUSSIAN = 0, 1
MF_SOLVER_LU, MF_SOLVER_QR, MF_SOLVER_SVD = 0, 1, 2
MF_TERM_IDENTITY, MF_TERM_D1, MF_TERM_D2, MF_TERM_LAPLACIAN, MF_TERM_DIRECTIONAL = 0, 1, 2, 3, 4


class EngineT(ctypes.Structure):
    """mf_engine_t (include/meshfree_b200.h): a general weight engine and its families."""
    _fields_ = [
        ("engine", _I32), ("rbf", _I32), ("k", _I32), ("solver", _I32), ("scale_code", _I32),
        ("weight", _I32), ("sigma", _D), ("weight_sigma", _D), ("d", _I32), ("l", _I32),
        ("expos", _I32 * (MF_MAX_MONOMIALS * MF_MAX_DIM)), ("nf", _I32),
        ("term0", _I32 * (MF_MAX_FAMILIES + 1)),
        ("term_kind", _I32 * MF_MAX_ENGINE_TERMS), ("term_a", _I32 * MF_MAX_ENGINE_TERMS),
        ("term_b", _I32 * MF_MAX_ENGINE_TERMS), ("term_order", _I32 * MF_MAX_ENGINE_TERMS),
        ("term_coeff", _D * MF_MAX_ENGINE_TERMS), ("term_vec", _D * (MF_MAX_ENGINE_TERMS * MF_MAX_DIM)),
    ]


MF_MAX_COLORS = 128


class Ilu0T(ctypes.Structure):
    """mf_ilu0_t (include/meshfree_b200.h): a multicolour ILU(0) factorisation."""
    _fields_ = [("indptr", _P), ("indices", _P), ("part", _P), ("diag", _P), ("lu", _P), ("order", _P),
                ("ncolors", _I32), ("rounds", _I32), ("color_off", _I32 * (MF_MAX_COLORS + 1))]


class FillGridT(ctypes.Structure):
    """mf_fill_grid_t (include/meshfree_b200.h)."""
    _fields_ = [("lo", _D * 3), ("cell", _D), ("dims", _I32 * 3), ("d", _I32)]


_SIGNATURES = {
    "mf_abi_version": ([], _I32),
    "mf_last_error": ([], ctypes.c_char_p),
    "mf_launch_count": ([], ctypes.c_longlong),
    "mf_dfma_probe": ([_I32, _I32, _I32, _P, _P, ctypes.POINTER(_D)], _I32),
    "mf_knn_workspace_size": ([_I64, _I32, _I64, _I64, _I32, ctypes.POINTER(_SZ)], _I32),
    "mf_knn": ([_P, _I64, _I32, _P, _I64, _P, _I64, _I32, _P, _P, _P, _SZ, _P], _I32),
    "mf_phs_workspace_size": ([_I64, ctypes.POINTER(_SZ)], _I32),
    "mf_phs_weights": ([_P, _I64, _I32, _P, _P, _I64, _I32, _I32, _I32, _P, _I32, _P, _P, _P, _P,
                        _P, _I32, _I32, _I32, _P, _P, _P, _P, ctypes.POINTER(PhsOptions), _P, _SZ, _P],
                       _I32),
    "mf_csr_workspace_size": ([_I64, ctypes.POINTER(_SZ)], _I32),
    "mf_csr_build": ([_P, _P, _I64, _I32, _I64, _P, _P, _P, _P, _P, _SZ, _P], _I32),
    "mf_csr_gather": ([_P, _P, _I64, _P, _P], _I32),
    "mf_apply": ([_P, _P, _P, _P, _P, _I64, _P], _I32),
    "mf_apply_rows": ([_P, _P, _P, _P, _P, _I64, _P, _P], _I32),
    "mf_order_workspace_size": ([_I64, ctypes.POINTER(_SZ)], _I32),
    "mf_locality_order": ([_P, _I64, _I32, _P, _P, _P, _SZ, _P], _I32),
    "mf_plan_build": ([_P, _P, _P, _I64, _I32, _P, _P, _P, _P, _P, _P], _I32),
    "mf_plan_apply_direct": ([_P, _P, _P, _I64, _I32, _P, _P, _P, _P], _I32),
    "mf_plan_apply": ([_P, _P, _P, _I64, _I32, _P, _P, _P, _P, _P, _P], _I32),
    "mf_permute": ([_P, _P, _I64, _I32, _P, _P], _I32),
    "mf_plan_apply_terms": ([_P, _P, _I64, _I32, _P, ctypes.POINTER(TermsT), _P], _I32),
    "mf_apply_terms_rows": ([_P, _P, _P, _I64, ctypes.POINTER(TermsT), _P], _I32),
    "mf_neumann_values": ([ctypes.POINTER(NeumannT), _P, _P, _P, _P, _P, _P], _I32),
    "mf_engine_weights": ([_P, _I64, _P, _P, _I64, _I32, ctypes.POINTER(EngineT), _P, _P, _P, _P], _I32),
    "mf_coo_workspace_size": ([_I64, ctypes.POINTER(_SZ)], _I32),
    "mf_coo_to_csr": ([_P, _P, _P, _I64, _I64, _P, _P, _P, _P, _SZ, _P], _I32),
    "mf_assemble_workspace_size": ([_I64, ctypes.POINTER(_SZ)], _I32),
    "mf_assemble_rows": ([_P, _P, _I64, _P, _P, ctypes.POINTER(_I64), _P, _SZ, _P], _I32),
    "mf_assemble_fill": ([_P, _P, _P, _I32, _P, _P, _P, _P, _I64, _P, _P, _P, _P], _I32),
    "mf_ilu0_workspace_size": ([_I64, ctypes.POINTER(_SZ)], _I32),
    "mf_ilu0_build": ([_P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, ctypes.POINTER(Ilu0T), _P, _P, _SZ, _P],
                      _I32),
    "mf_ilu0_apply": ([ctypes.POINTER(Ilu0T), _P, _P, _P], _I32),
    "mf_bicgstab_workspace_size": ([_I64, ctypes.POINTER(_SZ)], _I32),
    "mf_bicgstab": ([_P, _P, _P, _I64, ctypes.POINTER(Ilu0T), _P, _P, _D, _D, _I64, ctypes.POINTER(_I64),
                     ctypes.POINTER(_I32), ctypes.POINTER(_D), _P, _SZ, _P], _I32),
    "mf_fill_workspace_size": ([_I64, ctypes.POINTER(_SZ)], _I32),
    "mf_fill_insert": ([_P, _I64, _I64, ctypes.POINTER(FillGridT), _P, _P, _P], _I32),
    "mf_fill_accept": ([_P, _P, _P, _I64, _I64, ctypes.POINTER(FillGridT), _P, _P, _P, _P, _I64, _D, _P,
                        ctypes.POINTER(_I64), ctypes.POINTER(_I32), _P, _SZ, _P], _I32),
    "mf_heat_rows": ([_P, _P, _P, _P, _P, _P, _D, _D, _I64, _P, _P, _P], _I32),
    "mf_bicgstab_state_size": ([ctypes.POINTER(_SZ)], _I32),
    "mf_bicgstab_init": ([_P, _P, _P, _I64, _P, _P, _D, _D, _I64, _P, _P, _SZ, _P], _I32),
    "mf_bicgstab_iter": ([_P, _P, _P, _I64, ctypes.POINTER(Ilu0T), _P, _P, _P, _SZ, _P], _I32),
    "mf_heat_pack": ([_P, _P, _P, _P, _I64, _I32, _P, _P, _P, _P], _I32),
    "mf_heat_steps": ([_P, _P, _P, _I64, _I32, _P, _P, _P, _P, _D, _D, ctypes.POINTER(NeumannT),
                       _I64, _P, _P, _P, ctypes.POINTER(HeatPackT), _P], _I32),
}

EXPORTS = tuple(_SIGNATURES)

_lib = None


class LibraryError(RuntimeError):
    """The CUDA library is missing, failed to load, or rejected a call."""


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes handle; raises if the .so is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise LibraryError(
            f"{path} is not built; run `python -m paper_1912_13282_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.mf_abi_version() != 1:
        raise LibraryError("libmeshfree_b200 ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, what: str):
    if rc != MF_OK:
        msg = load().mf_last_error().decode(errors="replace")
        raise LibraryError(f"{what} failed (code {rc}): {msg}")


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise LibraryError("no CUDA device: the meshfree B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


_ARANGE = {}


def device_arange(n: int) -> torch.Tensor:
    """Cached int64 0..n-1 on the current device (full selections need no H2D copy)."""
    dev = device()  # raises LibraryError without a CUDA device
    key = (dev.index, int(n))
    t = _ARANGE.get(key)
    if t is None:
        t = torch.arange(int(n), dtype=torch.int64, device=dev)
        _ARANGE.clear() if len(_ARANGE) > 8 else None
        _ARANGE[key] = t
    return t


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    """Raw pointer of a tensor / numpy array (None passes NULL)."""
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    raise TypeError(type(t))


_WORKSPACES: dict = {}


def workspace(nbytes: int) -> torch.Tensor:
    """Scratch bytes for one C-ABI call, reused across calls on the same stream.

    Every entry point uses its workspace only for work it enqueues on the
    caller's stream, so the next call on that stream may take the same buffer;
    the buffer grows to the largest request and is kept (release_workspaces()
    drops them).  No call's outputs live in it.
    """
    dev = device()
    stream = torch.cuda.current_stream(dev)
    key = (dev.index, stream.cuda_stream)
    buf = _WORKSPACES.get(key)
    need = max(int(nbytes), 1)
    if buf is None or buf.numel() < need:
        if buf is not None:
            del _WORKSPACES[key]
            buf = None
        # round up (1 MiB) so small growth does not reallocate every call
        buf = torch.empty(((need + (1 << 20) - 1) >> 20) << 20, dtype=torch.uint8, device=dev)
        _WORKSPACES[key] = buf
    return buf[:need]


def release_workspaces() -> None:
    """Free the cached per-stream workspaces."""
    _WORKSPACES.clear()


_COPY_STREAM = None
_SIDE_STREAMS: dict = {}


def side_stream() -> torch.cuda.Stream:
    """A second (lower-priority) stream of the current device for work that may
    overlap the main stream's kernels (created once)."""
    dev = device()
    st = _SIDE_STREAMS.get(dev.index)
    if st is None:
        st = torch.cuda.Stream(device=dev, priority=0)
        _SIDE_STREAMS[dev.index] = st
    return st


def to_device_async(a, dtype):
    """Host array -> (device tensor, event): the copy runs on a side stream (async
    from pinned memory) so the caller can enqueue independent work meanwhile; the
    current stream must wait on the event before using the tensor."""
    global _COPY_STREAM
    if _COPY_STREAM is None:
        _COPY_STREAM = torch.cuda.Stream(device=device())
    arr = np.ascontiguousarray(a)
    if not arr.flags.writeable:
        arr = arr.copy()
    t = torch.from_numpy(arr)
    if t.dtype != dtype:
        t = t.to(dtype)
    main = torch.cuda.current_stream(device())
    with torch.cuda.stream(_COPY_STREAM):
        d = t.to(device(), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(_COPY_STREAM)
    d.record_stream(main)
    return d, ev


def to_device(a, dtype) -> torch.Tensor:
    """Host array or tensor -> contiguous device tensor of `dtype`."""
    if isinstance(a, torch.Tensor):
        return a.to(device=device(), dtype=dtype).contiguous()
    arr = np.ascontiguousarray(a)
    if not arr.flags.writeable:  # broadcast views: torch.from_numpy needs a writable buffer
        arr = arr.copy()
    t = torch.from_numpy(arr)
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.to(device(), non_blocking=False).contiguous()


SENTINEL_OK = int.from_bytes(b"\x7f" * 8, "little", signed=True)


class nvtx_range:
    """NVTX range around a public entry point (a no-op without a CUDA device)."""

    def __init__(self, name):
        self.name = name
        self.on = False

    def __enter__(self):
        if torch.cuda.is_available():
            torch.cuda.nvtx.range_push(self.name)
            self.on = True
        return self

    def __exit__(self, *exc):
        if self.on:
            torch.cuda.nvtx.range_pop()
        return False


def traced(name):
    """Decorator: run the function inside an NVTX range `name`."""
    def wrap(fn):
        import functools

        @functools.wraps(fn)
        def inner(*a, **k):
            with nvtx_range(name):
                return fn(*a, **k)
        return inner
    return wrap
