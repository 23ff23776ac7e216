"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the CPU oracle.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arms may import this module.  It is the checker, never the product:
the package ``paper_1912_13282_b200`` never imports it.

The C restatement (``meshfree_oracle.c``) replays the reference kernels
bit-for-bit; this module adds the small host-side pieces of the reference that
feed them (family encoding ``storage.py:342-384``, graded-lex exponents
``approx/basis.py:25-33``, monomial constraint right-hand side
``approx/basis.py:73-82`` at the origin).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from itertools import product

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

KIND_IDENTITY, KIND_D1, KIND_D2, KIND_LAPLACIAN = 0, 1, 2, 3
SCALE_CODES = {"none": 0, "nearest": 1, "support": 2}


def build() -> str:
    """Compile the oracle with its Makefile (no-op when up to date)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        src = os.path.join(_HERE, "meshfree_oracle.c")
        if not os.path.exists(_LIB_PATH) or (
            os.path.exists(src) and os.path.getmtime(src) > os.path.getmtime(_LIB_PATH)
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        i32 = ctypes.c_int
        L.oracle_phs_weights.argtypes = [P, i64, i32, P, P, i64, i32, i64, i32, P, i32, P,
                                         P, P, P, P, i32, i32, P, P, i32]
        L.oracle_phs_weights.restype = i32
        L.oracle_knn.argtypes = [P, i64, i32, P, i64, P, i64, i32, P, P, i32]
        L.oracle_knn.restype = i32
        L.oracle_csr_canonical.argtypes = [P, P, P, i64, i32, i64, P, P, P]
        L.oracle_csr_canonical.restype = i32
        L.oracle_apply.argtypes = [P, P, P, P, P, i64, i32]
        L.oracle_apply.restype = i32
        L.oracle_heat_steps.argtypes = [P, P, P, i64, P, P, P, P, ctypes.c_double,
                                        ctypes.c_double, i64, P, P, i32]
        L.oracle_heat_steps.restype = i64
        L.oracle_max_threads.restype = i32
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# -- host-side restatements of the reference's encoding ----------------------

def graded_lex_exponents(dim: int, degree: int):
    """approx/basis.py:25-33."""
    expos = [e for e in product(range(degree + 1), repeat=dim) if sum(e) <= degree]
    expos.sort(key=lambda e: (sum(e), tuple(-x for x in e)))
    return expos


def family_code(key: str, dim: int):
    """(kind, ax_a, ax_b, order) of a canonical family name (storage.py:349-363)."""
    if key == "identity":
        return KIND_IDENTITY, 0, 0, 0
    if key == "laplacian":
        return KIND_LAPLACIAN, 0, 0, 2
    if key.startswith("d1_"):
        return KIND_D1, int(key[3:]), 0, 1
    if key.startswith("d2_"):
        a, b = (int(x) for x in key[3:].split("_"))
        return KIND_D2, a, b, 2
    raise ValueError(key)


def expand(families, dim):
    out = []
    for f in families:
        if f == "gradient":
            out += [f"d1_{a}" for a in range(dim)]
        elif f == "hessian":
            out += [f"d2_{a}_{b}" for a in range(dim) for b in range(a, dim)]
        else:
            out.append(f)
    return out


def base_bot_row(key: str, expos):
    """(L x^e)(0) for each exponent tuple (approx/operators.py _mono_* at 0)."""
    kind, a, b, _ = family_code(key, len(expos[0]) if expos else 1)
    row = []
    for e in expos:
        e = list(e)
        if kind == KIND_IDENTITY:
            v = 1.0 if sum(e) == 0 else 0.0
        elif kind == KIND_D1:
            v = 1.0 if (sum(e) == 1 and e[a] == 1) else 0.0
        elif kind == KIND_D2:
            if a == b:
                v = 2.0 if (sum(e) == 2 and e[a] == 2) else 0.0
            else:
                v = 1.0 if (sum(e) == 2 and e[a] == 1 and e[b] == 1) else 0.0
        else:
            v = 2.0 if (sum(e) == 2 and max(e) == 2) else 0.0
        row.append(v)
    return row


def encode(families, dim, degree):
    keys = expand(families, dim)
    codes = np.array([family_code(k, dim) for k in keys], dtype=np.int64).reshape(-1, 4)
    if degree >= 0:
        expos = graded_lex_exponents(dim, degree)
        expos_arr = np.array(expos, dtype=np.int64).reshape(-1, dim)
        base_bot = np.array([base_bot_row(k, expos) for k in keys], dtype=np.float64)
    else:
        expos_arr = np.empty((0, dim), dtype=np.int64)
        base_bot = np.zeros((len(keys), 0))
    return keys, codes, expos_arr, base_bot.reshape(len(keys), expos_arr.shape[0])


# -- kernels --------------------------------------------------------------

def phs_weights(pts, rows, stencils, families, *, k=3, degree=2, scale="support", threads=0):
    """_batch_numba restatement -> (out (m, nf, n), fail (m,) int8, keys)."""
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    stencils = np.ascontiguousarray(stencils, dtype=np.int64)
    m, n = stencils.shape
    N, d = pts.shape
    keys, codes, expos, base_bot = encode(families, d, degree)
    nf = len(keys)
    kinds = np.ascontiguousarray(codes[:, 0])
    ax_a = np.ascontiguousarray(codes[:, 1])
    ax_b = np.ascontiguousarray(codes[:, 2])
    orders = np.ascontiguousarray(codes[:, 3])
    base_bot = np.ascontiguousarray(base_bot)
    out = np.zeros((m, nf, n))
    fail = np.zeros(m, dtype=np.int8)
    rc = lib().oracle_phs_weights(_p(pts), N, d, _p(rows), _p(stencils), m, n, int(k),
                                  int(k % 2 == 0), _p(expos), expos.shape[0], _p(base_bot),
                                  _p(kinds), _p(ax_a), _p(ax_b), _p(orders), nf,
                                  SCALE_CODES[scale], _p(out), _p(fail), int(threads))
    if rc != 0:
        raise ValueError("oracle_phs_weights rejected its arguments")
    return out, fail, keys


def knn(pts, n, targets=None, pool=None, threads=0):
    """find_closest_stencils restatement -> (T, n) int64 and straddle count."""
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    N, d = pts.shape
    targets = np.arange(N, dtype=np.int64) if targets is None else np.ascontiguousarray(targets, dtype=np.int64)
    pool = np.arange(N, dtype=np.int64) if pool is None else np.ascontiguousarray(pool, dtype=np.int64)
    T = targets.shape[0]
    out = np.zeros((T, n), dtype=np.int64)
    ns = np.zeros(1, dtype=np.int64)
    rc = lib().oracle_knn(_p(pts), N, d, _p(targets), T, _p(pool), pool.shape[0], int(n),
                          _p(out), _p(ns), int(threads))
    if rc != 0:
        raise ValueError("oracle_knn rejected its arguments")
    return out, int(ns[0])


def csr_canonical(rows, stencils, w, N):
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    stencils = np.ascontiguousarray(stencils, dtype=np.int64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    m, n = stencils.shape
    indptr = np.zeros(N + 1, dtype=np.int64)
    indices = np.zeros(m * n, dtype=np.int64)
    data = np.zeros(m * n)
    rc = lib().oracle_csr_canonical(_p(rows), _p(stencils), _p(w), m, n, N, _p(indptr),
                                    _p(indices), _p(data))
    if rc != 0:
        raise ValueError("oracle_csr_canonical: rows out of range or repeated")
    return indptr, indices, data


def apply(indptr, indices, data, u, threads=0):
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    data = np.ascontiguousarray(data, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    N = indptr.shape[0] - 1
    y = np.zeros(N)
    lib().oracle_apply(_p(indptr), _p(indices), _p(data), _p(u), _p(y), N, int(threads))
    return y


def heat_steps(indptr, indices, data, interior, dirichlet, g_dir, u0, *, dt, steps,
               diffusivity=1.0, source=None, threads=0):
    """Step-invariant run_heat_explicit loop -> (u, blowup_step, peak)."""
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    indices = np.ascontiguousarray(indices, dtype=np.int64)
    data = np.ascontiguousarray(data, dtype=np.float64)
    N = indptr.shape[0] - 1
    interior = np.ascontiguousarray(interior, dtype=np.uint8)
    dirichlet = np.ascontiguousarray(dirichlet, dtype=np.uint8)
    g_dir = np.ascontiguousarray(g_dir, dtype=np.float64)
    u = np.array(u0, dtype=np.float64, copy=True)
    src = None if source is None else np.ascontiguousarray(source, dtype=np.float64)
    peak = np.zeros(1)
    bad = lib().oracle_heat_steps(_p(indptr), _p(indices), _p(data), N, _p(interior),
                                  _p(dirichlet), _p(g_dir),
                                  None if src is None else _p(src), float(dt),
                                  float(diffusivity), int(steps), _p(u), _p(peak), int(threads))
    return u, int(bad), float(peak[0])


def monomial_count(degree, dim):
    return math.comb(degree + dim, dim)
