"""Operator layer (drop-in for the reference's kernels.py) on the GPU.

Every public function keeps the reference signature and semantics
(kernels.py:52-676); the arithmetic runs in libgraphblast_sm100a through the
C ABI.  Host-decidable argument errors are raised before any device work,
with the reference's exception types.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .algebra import Monoid, OpLike, Semiring, add_op_of, fold_op_id, mult_op_of, pair_op_id
from .containers import (
    INDEX_DTYPE,
    Counters,
    Descriptor,
    Direction,
    MaskMode,
    Partition,
    SparseMatrix,
    Vector,
    _Orient,
    compact,
    empty,
    full,
    scatter_dense,
)
from .errors import FormatError, ShapeError


@dataclass(frozen=True)
class DirectionDecision:
    """One push-or-pull choice with the numbers that produced it (kernels.py:52-60)."""

    chosen: str
    frontier_nvals: int
    estimated_frontier_edges: int
    total_edges: int
    threshold_edges: float


def _default_desc(desc):
    return desc if desc is not None else Descriptor()


_POLICY = {Direction.AUTO: _lib.DIR_AUTO, Direction.FORCE_PUSH: _lib.DIR_PUSH,
           Direction.FORCE_PULL: _lib.DIR_PULL}


def direction_rule(total, nrows, nnz_u, switch_ratio, policy):
    """kernels.py:108-126 as a pure function: (chosen, estimate, threshold)."""
    d = total / nrows if nrows else 0.0
    estimate = int(round(d * nnz_u))
    threshold = total * switch_ratio
    if policy is Direction.FORCE_PUSH:
        chosen = "push"
    elif policy is Direction.FORCE_PULL:
        chosen = "pull"
    else:
        chosen = "pull" if estimate > threshold else "push"
    return chosen, estimate, threshold


def decide_direction(u: Vector, A: SparseMatrix, desc=None, zero=0) -> DirectionDecision:
    """Choose push or pull for multiplying A (or A^T) by u (kernels.py:108-126)."""
    desc = _default_desc(desc)
    total = A.nnz
    nnz_u = u.nvals_for(zero)
    chosen, estimate, threshold = direction_rule(total, A.nrows, nnz_u, desc.switch_ratio,
                                                 desc.direction)
    return DirectionDecision(chosen, nnz_u, estimate, total, threshold)


def transpose(A: SparseMatrix) -> SparseMatrix:
    """Reverse every edge; O(1) when both layouts are stored (kernels.py:668-676)."""
    if not A.has_csc:
        A._build_csc()
    return SparseMatrix._wrap(A.ncols, A.nrows, A._csc, A._csr, A._dt, A._sym)


def _todo(name):
    def f(*a, **k):
        raise NotImplementedError(f"{name} is not wired yet")
    f.__name__ = name
    return f


mxv = _todo("mxv")
vxm = _todo("vxm")
spmv_pull = _todo("spmv_pull")
spmspv_push = _todo("spmspv_push")
mxm_masked = _todo("mxm_masked")
ewise_add = _todo("ewise_add")
ewise_mult = _todo("ewise_mult")
assign = _todo("assign")
assign_scatter = _todo("assign_scatter")
extract_gather = _todo("extract_gather")
apply = _todo("apply")
reduce = _todo("reduce")
reduce_rows = _todo("reduce_rows")
reduce_scalar_matrix = _todo("reduce_scalar_matrix")
