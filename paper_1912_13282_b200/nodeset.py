"""Node container: positions, type tags, boundary normals, stencils.

Mirrors the reference NodeSet (geometry/nodeset.py:25-147): same
constructor, selectors, accessors and errors.  The difference is storage:
stencils produced on the GPU stay on the GPU as dense (T, n) int32 blocks, and
the reference's Python list-of-arrays view (``.stencils``, ``.stencil(i)``)
is materialised lazily, only when host code asks for it.

Selectors (nodeset.py:8-15): ``None``/``"all"``, ``"interior"``,
``"boundary"``, an int tag, a list/tuple of tags, a boolean mask of length N,
or an integer index array (kept in the given order).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import GeometryError, StencilError


class _DevicePositions:
    """Device copy of the positions, shared by NodeSets derived from one another."""

    def __init__(self, positions: np.ndarray):
        self.host = positions
        self._dev = None

    def get(self) -> torch.Tensor:
        if self._dev is None:
            self._dev = _lib.to_device(self.host, torch.float64)
        return self._dev


class _Block:
    """Stencils of `nodes` (host int64), either a device (T, n) int32 matrix or host rows.

    ``nodes=None`` with ``full=N`` is the block of every node in index order
    (the common find_closest_stencils() case): no index array is materialised.
    """

    def __init__(self, nodes, mat=None, rows=None, full=None):
        self.full = full
        self._nodes = None if full is not None else np.asarray(nodes, dtype=np.int64)
        self.mat = mat
        self._rows = rows
        self._host = None

    @property
    def nodes(self):
        if self._nodes is None:
            self._nodes = np.arange(self.full, dtype=np.int64)
        return self._nodes

    @property
    def size(self):
        if self.mat is not None:
            return int(self.mat.shape[1])
        sizes = {len(r) for r in self._rows}
        return sizes.pop() if len(sizes) == 1 else None

    def host_matrix(self):
        if self._host is None:
            self._host = self.mat.cpu().numpy().astype(np.int64)
        return self._host

    def row(self, k):
        if self.mat is not None:
            return self.host_matrix()[k]
        return self._rows[k]

    def device_matrix(self):
        if self.mat is None:
            sizes = {len(r) for r in self._rows}
            if len(sizes) != 1:
                raise StencilError(f"stencil sizes differ: {sorted(sizes)}")
            self.mat = _lib.to_device(np.stack(self._rows).astype(np.int32), torch.int32)
        return self.mat


class NodeSet:
    def __init__(self, positions, types, normals=None, stencils=None):
        self.positions = np.ascontiguousarray(positions, dtype=float)
        if self.positions.ndim != 2:
            raise GeometryError("positions must be an (N, d) array")
        n, d = self.positions.shape
        self.types = np.asarray(types, dtype=np.int64)
        if self.types.shape != (n,):
            raise GeometryError("types must be a length-N vector")
        if normals is not None:
            normals = np.asarray(normals, dtype=float)
            if normals.shape != (n, d):
                raise GeometryError("normals must be an (N, d) array")
        self._normals = normals  # None: all NaN, materialised on first access
        self._pos = _DevicePositions(self.positions)
        self._blocks: list[_Block] = []
        # node -> block / row-in-block maps, materialised on demand (None: derived
        # from _full, the block covering every node in order, or "no stencil")
        self._blk_arr = None
        self._row_arr = None
        self._full = -1
        self._list_cache = None
        if stencils is not None:
            stencils = list(stencils)
            if len(stencils) != n:
                raise GeometryError("stencil list length must match node count")
            have = [i for i, s in enumerate(stencils) if s is not None]
            if have:
                rows = [np.asarray(stencils[i], dtype=np.int64) for i in have]
                self._add_block(_Block(np.array(have, dtype=np.int64), rows=rows))

    @property
    def _blk(self) -> np.ndarray:
        if self._blk_arr is None:
            self._blk_arr = np.full(len(self), self._full, dtype=np.int32)
        return self._blk_arr

    @property
    def _row(self) -> np.ndarray:
        if self._row_arr is None:
            self._row_arr = (np.arange(len(self), dtype=np.int64) if self._full >= 0
                             else np.zeros(len(self), dtype=np.int64))
        return self._row_arr

    @property
    def normals(self) -> np.ndarray:
        if self._normals is None:
            self._normals = np.full(self.positions.shape, np.nan)
        return self._normals

    @normals.setter
    def normals(self, value):
        self._normals = value

    # -- internal stencil bookkeeping ------------------------------------

    def _add_block(self, block: _Block):
        b = len(self._blocks)
        self._blocks.append(block)
        if block.full is not None:
            self._blk_arr = None  # implied: every node -> block b, row = node
            self._row_arr = None
            self._full = b
        else:
            blk, row = self._blk, self._row  # materialise before the maps change meaning
            blk[block.nodes] = b
            row[block.nodes] = np.arange(block.nodes.shape[0])
            self._full = -1
        self._list_cache = None

    def _derive(self, copy_maps: bool = True) -> "NodeSet":
        new = NodeSet.__new__(NodeSet)
        new.positions = self.positions
        new.types = self.types
        new._normals = self._normals
        new._pos = self._pos
        new._blocks = list(self._blocks)
        new._blk_arr = self._blk_arr.copy() if (copy_maps and self._blk_arr is not None) else None
        new._row_arr = self._row_arr.copy() if (copy_maps and self._row_arr is not None) else None
        new._full = self._full
        new._list_cache = None
        return new

    def _with_device_stencils(self, targets, mat: torch.Tensor) -> "NodeSet":
        if targets is None:  # every node, in index order: the maps are rebuilt, not copied
            new = self._derive(copy_maps=False)
            new._add_block(_Block(None, mat=mat, full=len(self)))
            return new
        new = self._derive()
        new._add_block(_Block(np.asarray(targets, dtype=np.int64), mat=mat))
        return new

    def full_block_matrix(self):
        """The (N, n) device stencil matrix when one block covers every node in order, else None."""
        if self._full < 0:
            return None
        return self._blocks[self._full].device_matrix()

    def positions_device(self) -> torch.Tensor:
        return self._pos.get()

    def stencil_matrix_device(self, idx) -> torch.Tensor:
        """(M, n) int32 device matrix of the stencils of node indices `idx`."""
        idx = np.asarray(idx, dtype=np.int64)
        if idx.size == 0:
            return torch.empty((0, 0), dtype=torch.int32, device=_lib.device())
        if self._full >= 0 and idx.shape[0] == len(self) and idx[0] == 0 and idx[-1] == len(self) - 1 \
                and np.array_equal(idx, np.arange(len(self))):
            return self._blocks[self._full].device_matrix()
        blk = self._blk[idx]
        missing = np.flatnonzero(blk < 0)
        if missing.size:
            raise StencilError(f"node {int(idx[missing[0]])} has no stencil")
        bmin, bmax = int(blk.min()), int(blk.max())
        used = np.array([bmin]) if bmin == bmax else np.unique(blk)  # (one block: no sort)
        sizes = sorted({self._blocks[b].size for b in used} - {None})
        if len(sizes) != 1 or any(self._blocks[b].size is None for b in used):
            all_sizes = set()
            for b in used:
                blkobj = self._blocks[b]
                rows = self._row[idx[blk == b]]
                all_sizes |= {len(blkobj.row(int(k))) for k in rows}
            if len(all_sizes) != 1:
                raise StencilError(f"stencil sizes differ: {sorted(all_sizes)}")
        b0 = self._blocks[int(blk[0])]
        n = b0.size if b0.mat is not None else len(b0.row(int(self._row[idx[0]])))  # (no host copy of a device block)

        def rows_of(b, sel_rows):
            """Device (k, n) int32 stencils of block b's rows sel_rows: blocks held as
            host rows upload only the selected rows (they may mix stencil sizes)."""
            blkobj = self._blocks[int(b)]
            if blkobj.mat is None:
                host = np.stack([blkobj.row(int(k)) for k in sel_rows]).astype(np.int32)
                return _lib.to_device(host, torch.int32)
            mat = blkobj.mat
            if sel_rows.shape[0] == mat.shape[0] and np.array_equal(sel_rows, np.arange(sel_rows.shape[0])):
                return mat
            return mat.index_select(0, _lib.to_device(sel_rows, torch.int64))

        if used.size == 1:
            return rows_of(used[0], self._row[idx])
        out = torch.empty((idx.shape[0], n), dtype=torch.int32, device=_lib.device())
        for b in used:
            sel = np.flatnonzero(blk == b)
            out.index_copy_(0, _lib.to_device(sel, torch.int64), rows_of(b, self._row[idx[sel]]))
        return out

    # -- basic queries ---------------------------------------------------

    def __len__(self):
        return self.positions.shape[0]

    @property
    def dim(self) -> int:
        return self.positions.shape[1]

    def interior_indices(self):
        return np.flatnonzero(self.types > 0)

    def boundary_indices(self):
        return np.flatnonzero(self.types < 0)

    def normal(self, i: int):
        """Outward normal of boundary node i (nodeset.py:85-88)."""
        if self.types[i] >= 0:
            raise GeometryError(f"node {i} is not a boundary node")
        return self.normals[i]

    def select(self, which):
        """Resolve a node selector (see module docstring) to an index array."""
        n = len(self)
        if which is None or (isinstance(which, str) and which == "all"):
            return np.arange(n)
        if isinstance(which, str):
            if which == "interior":
                return self.interior_indices()
            if which == "boundary":
                return self.boundary_indices()
            raise GeometryError(f"unknown node selector {which!r}")
        if isinstance(which, (int, np.integer)):
            return np.flatnonzero(self.types == which)
        if isinstance(which, (list, tuple, set, frozenset)):
            mask = np.isin(self.types, list(which))
            return np.flatnonzero(mask)
        if isinstance(which, torch.Tensor):
            which = which.cpu().numpy()
        arr = np.asarray(which)
        if arr.dtype == bool:
            if arr.shape != (n,):
                raise GeometryError("boolean selector must have length N")
            return np.flatnonzero(arr)
        if np.issubdtype(arr.dtype, np.integer):
            if arr.size and (arr.min() < 0 or arr.max() >= n):
                raise GeometryError("index selector out of range")
            return arr.astype(np.int64)
        raise GeometryError(f"cannot interpret node selector {which!r}")

    def normal(self, i: int):
        if self.types[i] >= 0:
            raise GeometryError(f"node {i} is not a boundary node")
        return self.normals[i]

    @property
    def stencils(self) -> list:
        """Reference-style list of N stencils (np.int64 arrays or None), built lazily."""
        if self._list_cache is None:
            out = [None] * len(self)
            for i in np.flatnonzero(self._blk >= 0):
                out[int(i)] = self.stencil(int(i))
            self._list_cache = out
        return self._list_cache

    def stencil(self, i: int):
        b = self._blk[i]
        if b < 0:
            raise StencilError(f"node {i} has no stencil")
        return np.asarray(self._blocks[b].row(int(self._row[i])), dtype=np.int64)

    def has_stencil(self, i: int) -> bool:
        return bool(self._blk[i] >= 0)

    # -- derived forms -----------------------------------------------------

    def stencil_matrix(self, indices=None):
        """Stack stencils of the given nodes into an (M, n) int64 host matrix."""
        idx = self.select(indices)
        if idx.size == 0:
            return np.empty((0, 0), dtype=np.int64)
        missing = np.flatnonzero(self._blk[idx] < 0)
        if missing.size:
            raise StencilError(f"node {int(idx[missing[0]])} has no stencil")
        rows = [self.stencil(int(i)) for i in idx]
        sizes = {r.shape[0] for r in rows}
        if len(sizes) != 1:
            raise StencilError(f"stencil sizes differ: {sorted(sizes)}")
        return np.vstack(rows).astype(np.int64)

    def append(self, positions, types, normals=None):
        """New NodeSet with extra nodes appended; existing stencils kept."""
        positions = np.atleast_2d(np.asarray(positions, dtype=float))
        m = positions.shape[0]
        types = np.broadcast_to(np.asarray(types, dtype=np.int64), (m,))
        if normals is None:
            normals = np.full((m, self.dim), np.nan)
        new = NodeSet(
            np.concatenate([self.positions, positions], axis=0),
            np.concatenate([self.types, types]),
            np.concatenate([self.normals, normals], axis=0),
        )
        new._pos = _DevicePositions(new.positions)
        new._blocks = list(self._blocks)
        n_old = len(self)
        blk, row = new._blk, new._row  # fresh maps (new._full is -1)
        blk[:n_old] = self._blk
        row[:n_old] = self._row
        return new

    def with_stencils(self, indices, stencils):
        """New NodeSet where nodes ``indices[k]`` get ``stencils[k]``."""
        indices = np.asarray(indices, dtype=np.int64)
        if isinstance(stencils, torch.Tensor) and stencils.is_cuda:
            return self._with_device_stencils(indices, stencils.to(torch.int32).contiguous())
        rows = [np.asarray(s, dtype=np.int64) for s in stencils]
        new = self._derive()
        if rows:
            new._add_block(_Block(indices, rows=rows))
        return new

    def __repr__(self):
        nb = len(self.boundary_indices())
        ni = len(self.interior_indices())
        return (
            f"NodeSet(N={len(self)}, d={self.dim}, interior={ni}, "
            f"boundary={nb}, other={len(self) - ni - nb})"
        )
