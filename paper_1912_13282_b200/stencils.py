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


def _is_all(which) -> bool:
    return which is None or (isinstance(which, str) and which == "all")


@_lib.traced("meshfree.find_closest_stencils")
def find_closest_stencils(nodes: NodeSet, n: int, for_which=None, search_among=None) -> NodeSet:
    """Attach n-nearest-neighbour stencils to the selected nodes.

    ``for_which`` selects the nodes that receive stencils and ``search_among``
    the pool stencil members are drawn from (selector syntax as in NodeSet).
    Returns a new NodeSet.
    """
    N = len(nodes)
    all_t, all_p = _is_all(for_which), _is_all(search_among)
    targets = None if all_t else nodes.select(for_which)
    pool = None if all_p else nodes.select(search_among)
    P = N if all_p else pool.shape[0]
    T = N if all_t else targets.shape[0]
    if n < 1:
        raise StencilError(f"stencil size must be at least 1, got {n}")
    if n > P:
        raise StencilError(
            f"stencil size {n} exceeds search pool of {P} nodes"
        )
    if T == 0:
        return nodes
    # full selections go to the device as a cached arange (no host array, no H2D)
    t_arg = _lib.device_arange(N) if all_t else targets
    p_arg = _lib.device_arange(N) if all_p else pool
    mat, _ = knn_device(nodes, int(n), t_arg, p_arg)
    return nodes._with_device_stencils(None if all_t else targets, mat)
