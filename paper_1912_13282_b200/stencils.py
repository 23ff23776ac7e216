"""Nearest-neighbour stencil selection on the GPU.

Drop-in for the reference's find_closest_stencils (geometry/stencils.py:19-93):
same arguments, preconditions, error messages and result -- for each target the
n closest pool nodes ordered by (squared distance, node index), the target
first when it belongs to the pool -- computed by the cell-list kNN kernel
``mf_knn`` (csrc/knn.cu).  The stencils stay on the device as an int32 block
of the returned NodeSet.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, StencilError
from .nodeset import NodeSet


def knn_device(nodes: NodeSet, n: int, targets: np.ndarray, pool: np.ndarray):
    """Run mf_knn -> ((T, n) int32 device stencils, straddle-row count tensor)."""
    lib = _lib.load()
    dev = _lib.device()
    N, d = nodes.positions.shape
    if d > 3:
        raise ConfigError(f"GPU stencil selection supports d <= 3, got {d}")
    T, P = int(targets.shape[0]), int(pool.shape[0])  # host arrays or resident device tensors
    pos = nodes.positions_device()
    t_d = _lib.to_device(targets, torch.int64)
    p_d = _lib.to_device(pool, torch.int64)
    out = torch.empty((T, n), dtype=torch.int32, device=dev)
    nstr = torch.zeros(1, dtype=torch.int64, device=dev)
    size = ctypes.c_size_t(0)
    _lib.check(lib.mf_knn_workspace_size(N, d, T, P, n, ctypes.byref(size)), "mf_knn_workspace_size")
    ws = _lib.workspace(size.value)
    _lib.check(lib.mf_knn(pos.data_ptr(), N, d, t_d.data_ptr(), T, p_d.data_ptr(), P, n,
                          out.data_ptr(), nstr.data_ptr(), ws.data_ptr(), size.value,
                          _lib.stream_ptr()), "mf_knn")
    return out, nstr


def find_closest_stencils(nodes: NodeSet, n: int, for_which=None, search_among=None) -> NodeSet:
    """Attach n-nearest-neighbour stencils to the selected nodes.

    ``for_which`` selects the nodes that receive stencils and ``search_among``
    the pool stencil members are drawn from (selector syntax as in NodeSet).
    Returns a new NodeSet.
    """
    targets = nodes.select(for_which)
    pool = nodes.select(search_among)
    if n < 1:
        raise StencilError(f"stencil size must be at least 1, got {n}")
    if n > pool.shape[0]:
        raise StencilError(
            f"stencil size {n} exceeds search pool of {pool.shape[0]} nodes"
        )
    if targets.shape[0] == 0:
        return nodes
    mat, _ = knn_device(nodes, int(n), targets, pool)
    return nodes._with_device_stencils(targets, mat)
