"""The five graph algorithms (drop-in for the reference's algorithms.py).

Each algorithm validates its input exactly like the reference and then runs
a FUSED device loop: one native driver call per algorithm that executes the
reference's operator composition level by level with the elementwise and
reduce steps folded into the traversal kernels (north star (5)).  Results --
and the direction trace in ``desc.direction_log`` -- equal the reference's.

``desc.fused = False`` instead replays the reference's literal composition
through the unfused kernels (kernels.py), so ``desc.counters`` carries the
reference's exact work tallies.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _lib
from .algebra import LESS, MINUS, TIMES, builtin_monoid, builtin_semiring
from .containers import INDEX_DTYPE, Descriptor, Direction, SparseMatrix, Vector, empty
from .errors import ShapeError
from .kernels import (
    DirectionDecision,
    apply,
    assign,
    assign_scatter,
    ewise_add,
    ewise_mult,
    extract_gather,
    mxm_masked,
    mxv,
    reduce,
    reduce_scalar_matrix,
    transpose,
    vxm,
)

_INT_INF = np.iinfo(np.int64).max

_POLICY = {Direction.AUTO: _lib.DIR_AUTO, Direction.FORCE_PUSH: _lib.DIR_PUSH,
           Direction.FORCE_PULL: _lib.DIR_PULL}


def _require_square(A):
    if A.nrows != A.ncols:
        raise ShapeError(f"adjacency matrix must be square, got {A.nrows}x{A.ncols}")


def _require_symmetric(A):
    """algorithms.py:41-45 -- O(1) once the build has compared CSR and CSC."""
    if not A.is_symmetric():
        raise ValueError("adjacency matrix must be symmetric (undirected graph)")


def _log_decisions(desc, A, dirs, nvals, ests, count):
    total = A.nnz
    thr = total * desc.switch_ratio
    for i in range(count):
        chosen = "pull" if dirs[i] == _lib.DIR_PULL else "push"
        desc.direction_log.append(
            DirectionDecision(chosen, int(nvals[i]), int(ests[i]), total, thr))


# ---------------------------------------------------------------------------
# BFS
# ---------------------------------------------------------------------------


def bfs(A: SparseMatrix, source: int, desc=None, early_exit=True) -> Vector:
    """Level labels of a breadth-first search: source 1, unreached 0 (algorithms.py:48-77)."""
    _require_square(A)
    if not 0 <= source < A.nrows:
        raise IndexError(f"source {source} out of range")
    desc = desc if desc is not None else Descriptor()
    desc.early_exit = early_exit
    if not desc.fused:
        return _bfs_composed(A, source, desc)
    n = A.nrows
    iters = min(desc.max_niter, n + 1)
    levels = empty(n, np.int64)
    push, _k1 = A.orient(False).csr_struct()          # vxm push walks rows of A (CSR)
    pull_o = A.orient(True) if A.has_csc else None    # vxm pull walks rows of A^T (CSC)
    pull, _k2 = pull_o.csr_struct() if pull_o is not None else (None, None)
    cap = max(iters, 1)
    dirs = np.zeros(cap, np.int32)
    nv = np.zeros(cap, np.int64)
    est = np.zeros(cap, np.int64)
    done = C.c_int64(0)
    _lib.context().call(
        "gb_bfs", C.byref(push), C.byref(pull) if pull is not None else None,
        _lib.ptr(pull_o.nonempty()) if pull_o is not None else None,
        int(source), int(iters), float(desc.switch_ratio), _POLICY[desc.direction],
        _lib.ptr(levels), dirs.ctypes.data_as(C.c_void_p), nv.ctypes.data_as(C.c_void_p),
        est.ctypes.data_as(C.c_void_p), C.byref(done))
    _log_decisions(desc, A, dirs, nv, est, int(done.value))
    return Vector._wrap(n, None, levels, 0, np.int64)


def _bfs_composed(A, source, desc):
    boolean = builtin_semiring("LogicalOrAnd")
    plus = builtin_monoid("Plus")
    n = A.nrows
    frontier = Vector.from_entries([source], [1], n, dtype=np.int64)
    visited = Vector.filled(n, 0, dtype=np.int64)
    depth = 1
    for _ in range(min(desc.max_niter, n + 1)):
        assign(visited, depth, mask=frontier, desc=desc)
        desc.toggle("mask")
        frontier = vxm(boolean, frontier, A, mask=visited, desc=desc)
        desc.toggle("mask")
        if int(reduce(plus, frontier)) == 0:
            break
        depth += 1
    return visited


def sssp(A, source, desc=None, on_iteration=None):
    raise NotImplementedError("sssp is not wired yet")


def pagerank(A, alpha=0.85, eps=1e-7, max_iters=10_000, desc=None):
    raise NotImplementedError("pagerank is not wired yet")


def connected_components(A, desc=None, sparsify=True):
    raise NotImplementedError("connected_components is not wired yet")


def triangle_count(A, desc=None):
    raise NotImplementedError("triangle_count is not wired yet")
