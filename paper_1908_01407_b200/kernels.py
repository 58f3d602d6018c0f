"""Operator layer (drop-in for the reference's kernels.py) on the GPU.

Every public function keeps the reference signature and semantics
(kernels.py:52-676); the arithmetic runs in libgraphblast_sm100a through the
C ABI.  Host-decidable argument errors are raised before any device work,
with the reference's exception types.  These are the UNFUSED kernels: they
reproduce the reference exactly, including ``desc.counters`` and the
direction log; the algorithms call fused drivers instead (algorithms.py).
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .algebra import Monoid, OpLike, Semiring, add_op_of, fold_op_id, mult_op_of, pair_op_id
from .containers import (
    INDEX_DTYPE,
    Descriptor,
    Direction,
    MaskMode,
    Partition,
    SparseMatrix,
    Vector,
    _Orient,
    _TORCH,
    cast,
    compact,
    device_dtype,
    empty,
    full,
    gather32,
    iota,
    to_dev,
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


def _ctx():
    return _lib.context()


def _code(dt):
    return _lib.dtype_code(dt)


def _buf(value, dt):
    return _lib.scalar_buf(value, dt)


def _as(t, dt):
    return cast(t, dt)


def _counters_tensor():
    return torch.zeros(3, dtype=torch.int64, device=torch.device("cuda", torch.cuda.current_device()))


def _merge_counters(desc, t):
    r, m, a = (int(x) for x in t.cpu().tolist())
    desc.counters.matrix_entries_read += r
    desc.counters.semiring_multiplies += m
    desc.counters.semiring_adds += a


# ---------------------------------------------------------------------------
# masks  (kernels.py:67-84)
# ---------------------------------------------------------------------------


def _mask_bitmap(mask, size, mode):
    """Device bitmap of allowed output positions, or None when unmasked."""
    if mask is None:
        return None
    if mask.size != size:
        raise ShapeError(f"mask size {mask.size} does not match output size {size}")
    W = max((size + 31) // 32, 1)
    out = torch.empty(W, dtype=torch.int32, device=mask._vals.device)
    k = -1 if mask._idx is None else int(mask._idx.numel())  # -1: dense mask
    _ctx().call("gb_mask_bitmap", int(size), k, _lib.ptr(mask._idx), _lib.ptr(mask._vals),
                _code(mask._dt), 1 if mode is MaskMode.COMPLEMENT else 0, _lib.ptr(out))
    return out


def _bitmap_count(bm, size):
    c = C.c_int64(0)
    _ctx().call("gb_bitmap_count", int(size), _lib.ptr(bm), C.byref(c))
    return int(c.value)


def _bitmap_of_indices(idx_t, size):
    """Bitmap with the given int32 positions set."""
    W = max((size + 31) // 32, 1)
    out = torch.empty(W, dtype=torch.int32, device=idx_t.device)
    ones = torch.ones(int(idx_t.numel()), dtype=torch.int64, device=idx_t.device)
    _ctx().call("gb_mask_bitmap", int(size), int(idx_t.numel()), _lib.ptr(idx_t), _lib.ptr(ones),
                _lib.GB_I64, 0, _lib.ptr(out))
    return out


def _filter(idx_t, vals_t, dt, bm):
    """Keep sparse entries whose index the bitmap allows."""
    k = int(idx_t.numel())
    if bm is None or k == 0:
        return idx_t, vals_t
    oi = empty(k, np.int32)
    ov = empty(k, dt)
    cnt = C.c_int64(0)
    _ctx().call("gb_filter_mask", _code(dt), k, _lib.ptr(idx_t), _lib.ptr(vals_t), _lib.ptr(bm),
                _lib.ptr(oi), _lib.ptr(ov), C.byref(cnt))
    c = int(cnt.value)
    return oi[:c], ov[:c]


# ---------------------------------------------------------------------------
# direction choice  (kernels.py:108-126)
# ---------------------------------------------------------------------------


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


# ---------------------------------------------------------------------------
# pull / push  (kernels.py:153-286)
# ---------------------------------------------------------------------------


def _spmv_pull(semiring, A, u, mask, desc, transpose):
    o = A.orient(transpose)                      # row_view: CSR, or CSC when transposed
    in_size = A.nrows if transpose else A.ncols
    if u.is_sparse:
        raise FormatError("pull kernel requires a dense input vector (dispatcher bug)")
    if u.size != in_size:
        raise ShapeError(f"matrix has {in_size} columns but vector has size {u.size}")
    dtype = np.result_type(A.dtype, u.dtype)
    identity = semiring.add.identity_for(dtype)
    add, mult = fold_op_id(semiring.add.op), pair_op_id(semiring.multiply)
    bm = _mask_bitmap(mask, o.nrows, desc.mask_mode)
    early = 1 if (desc.early_exit and semiring.add.name == "LogicalOr") else 0
    s, keep = o.csr_struct(dtype)
    uv = _as(u._vals, dtype)
    out = empty(o.nrows, dtype)
    cnt = _counters_tensor()
    part = _lib.PART_ROW if desc.partition is Partition.ROW_SPLIT else _lib.PART_NONZERO
    view = None
    if _use_bins(bm, add, early, part, o):
        nst = _stripe_count(o)
        if nst > 1:
            csrs, plans, _sk = o.stripes(nst)
            if dtype != o.dt:  # the stripes carry the orientation's own dtype tag
                csrs = _retag(csrs, dtype)
            _ctx().call("gb_mxv_pull_striped", add, mult, nst, C.cast(csrs, C.c_void_p),
                        C.cast(plans, C.c_void_p), _lib.ptr(uv), _lib.ptr(bm), _lib.ptr(out),
                        _lib.ptr(cnt))
        else:
            bins, _bk = o.bin_plan()
            _ctx().call("gb_mxv_pull_binned", add, mult, C.byref(s), C.byref(bins),
                        _lib.ptr(uv), _lib.ptr(bm), _lib.ptr(out), _lib.ptr(cnt))
    elif (view := _ordered_view(A, o, transpose, add, early, part)) is not None:
        ov, oplan, _keep, order, reach = view
        so, _ko = ov.csr_struct(dtype)
        _ctx().call("gb_mxv_pull_ordered", add, mult, C.byref(so), C.byref(oplan), _lib.ptr(order),
                    reach, _lib.ptr(uv), _lib.ptr(bm), _lib.ptr(out), _lib.ptr(cnt))
    else:
        plan, _pk = o.row_plan()
        _ctx().call("gb_mxv_pull", add, mult, C.byref(s), C.byref(plan), _lib.ptr(uv),
                    _lib.ptr(bm), early, part, _lib.ptr(out), _lib.ptr(cnt))
    _merge_counters(desc, cnt)
    return Vector._wrap(o.nrows, None, out, identity, dtype)


# The masked pull runs on the degree-ordered layout (gb_mxv_pull_ordered) for
# large power-law matrices: the layout is built once per matrix (~0.2 s and
# one relabelled copy of the structure at s24, shared with bfs) and makes the
# gathered part of u a dense, L2-resident prefix whose head sits in shared
# memory.  Measured at s24 with a 50 % mask it gains 5 % in the kernel and
# loses it to the per-call permutation (1.32 + 0.08 vs 1.40 ms), and the
# shared-memory head made it slower (2.2 ms: the L1 it displaces held more
# hits), so it is opt-in: GB_MV_ORDERED=1.
_MV_ORDERED = os.environ.get("GB_MV_ORDERED", "")


# Row bins (gb_mxv_pull_binned) for masked pulls and Partition.ROW_SPLIT:
# rows are mask-tested before their entries are read, so masked-out rows cost
# one bit probe instead of their share of the edge-balanced tiles.
# GB_MV_BINS=0 disables, =1 also takes unmasked pulls.
_MV_BINS = os.environ.get("GB_MV_BINS", "")


# Column stripes for the binned pull (gb_mxv_pull_striped): when the gathered
# vector is larger than GB_MV_STRIPE_BYTES (default 48 MB, under half of the
# 126 MB L2) a structure-only matrix whose degrees are not skewed (under
# 10 % of its entries in rows longer than 512) is cut into ceil(8*ncols /
# that) column stripes, multiplied one after the other, so every stripe's
# slice of the vector stays L2-resident while it is gathered.  Measured at
# s24, 50 % mask: uniform 2.68 -> 1.90 ms with 4 stripes; R-MAT 1.27 -> 1.78
# ms (its gathers concentrate on the hubs, which stay cached anyway, so the
# extra passes only cost) -- hence the skew test.  Stripe budget at uniform
# s24 (masked f64, kernel ms): 16 MB (8 stripes) 2.97, 32 MB (4) 1.85, 48 MB
# (3) 1.80, 64 MB (2) 2.72; the unmasked int64 min-pull 3.04 (32 MB) vs 3.10
# (48 MB).  0 disables.
_MV_STRIPE_BYTES = int(os.environ.get("GB_MV_STRIPE_BYTES", str(48 << 20)))
_MV_STRIPE_SKEW = float(os.environ.get("GB_MV_STRIPE_SKEW", "0.1"))


def _stripe_count(o):
    if _MV_STRIPE_BYTES <= 0 or o.values is not None:
        return 1
    k = max(1, -(-8 * o.ncols // _MV_STRIPE_BYTES))
    if k > 1 and _MV_STRIPE_SKEW < 1.0:
        plan, _pk = o.bin_plan()
        if plan.n_long_tiles * 512 >= _MV_STRIPE_SKEW * max(o.nnz, 1):
            return 1
    return k


def _retag(csrs, dtype):
    out = (_lib.gb_csr * len(csrs))()
    for k, c in enumerate(csrs):
        out[k] = c
        out[k].dtype = _lib.dtype_code(dtype)
        out[k].iso_i64, out[k].iso_f64 = c.iso_i64, c.iso_f64
    return out


def _use_bins(bm, add, early, part, o):
    if _MV_BINS == "0" or early or add not in _lib.COMMUTATIVE_FOLD_IDS:
        return False
    # unmasked too when the matrix takes column stripes (large gathered
    # vector, degrees not skewed): uniform s24 min-pull 5.18 -> 3.04 ms
    return bm is not None or part == _lib.PART_ROW or _MV_BINS == "1" or _stripe_count(o) > 1


def _ordered_view(A, o, transpose, add, early, part):
    if _MV_ORDERED != "1" or early or part == _lib.PART_ROW:
        return None
    if add not in _lib.COMMUTATIVE_FOLD_IDS or A.nrows != A.ncols or A._csc is None:
        return None
    return A.ordered_pull(transpose)


def spmv_pull(semiring: Semiring, A: SparseMatrix, u: Vector, mask=None, desc=None) -> Vector:
    """Row-walking multiply over a dense vector; mask applied first (kernels.py:232-235)."""
    desc = _default_desc(desc)
    return _spmv_pull(semiring, A, u, mask, desc, desc.transpose_inp0)


def _spmspv_push(semiring, A, u, mask, desc, transpose):
    o = A.orient(not transpose)                  # col_view: CSC, or CSR when transposed
    out_size = A.ncols if transpose else A.nrows
    if not u.is_sparse:
        raise FormatError("push kernel requires a sparse input vector (dispatcher bug)")
    if u.size != o.nrows:
        raise ShapeError(f"matrix has {o.nrows} columns but vector has size {u.size}")
    dtype = np.result_type(A.dtype, u.dtype)
    identity = semiring.add.identity_for(dtype)
    add, mult = fold_op_id(semiring.add.op), pair_op_id(semiring.multiply)
    bm = _mask_bitmap(mask, out_size, desc.mask_mode)
    k = int(u._idx.numel())
    s, keep = o.csr_struct(dtype)
    uv = _as(u._vals, dtype)
    cap = max(min(out_size, o.nnz), 1)
    oi = empty(cap, np.int32)
    ov = empty(cap, dtype)
    cnt = _counters_tensor()
    c = C.c_int64(0)
    _ctx().call("gb_mxv_push", add, mult, C.byref(s), int(out_size), k, _lib.ptr(u._idx),
                _lib.ptr(uv), _lib.ptr(bm), _lib.ptr(oi), _lib.ptr(ov), C.byref(c), _lib.ptr(cnt))
    _merge_counters(desc, cnt)
    n = int(c.value)
    return Vector._wrap(out_size, oi[:n], ov[:n], identity, dtype)


def spmspv_push(semiring: Semiring, A: SparseMatrix, u: Vector, mask=None, desc=None) -> Vector:
    """Column-gathering multiply over a sparse vector; mask applied after (kernels.py:283-286)."""
    desc = _default_desc(desc)
    return _spmspv_push(semiring, A, u, mask, desc, desc.transpose_inp0)


def _mv_dispatch(semiring, A, u, mask, desc, transpose):
    """kernels.py:293-310."""
    out_size = A.ncols if transpose else A.nrows
    in_size = A.nrows if transpose else A.ncols
    if u.size != in_size:
        raise ShapeError(f"matrix expects input of size {in_size}, got {u.size}")
    if mask is not None and mask.size != out_size:
        raise ShapeError(f"mask size {mask.size} does not match output size {out_size}")
    dtype = np.result_type(A.dtype, u.dtype)
    identity = semiring.add.identity_for(dtype)
    decision = decide_direction(u, A, desc, zero=identity)
    desc.direction_log.append(decision)
    if decision.chosen == "pull":
        u_run = u if not u.is_sparse else u.to_dense(identity)
        return _spmv_pull(semiring, A, u_run, mask, desc, transpose)
    u_run = u if u.is_sparse else u.to_sparse(identity)
    return _spmspv_push(semiring, A, u_run, mask, desc, transpose)


def mxv(semiring: Semiring, A: SparseMatrix, u: Vector, mask=None, desc=None) -> Vector:
    """w = A u over the semiring, masked, with automatic push/pull (kernels.py:313-316)."""
    desc = _default_desc(desc)
    return _mv_dispatch(semiring, A, u, mask, desc, desc.transpose_inp0)


def vxm(semiring: Semiring, u: Vector, A: SparseMatrix, mask=None, desc=None) -> Vector:
    """w = u A, i.e. mxv against the transposed matrix (kernels.py:319-322)."""
    desc = _default_desc(desc)
    return _mv_dispatch(semiring, A, u, mask, desc, not desc.transpose_inp1)


# ---------------------------------------------------------------------------
# masked matrix-matrix  (kernels.py:329-391)
# ---------------------------------------------------------------------------


def mxm_masked(semiring: Semiring, A: SparseMatrix, B: SparseMatrix,
               mask: SparseMatrix, desc=None) -> SparseMatrix:
    """C = (A B) .* mask, computing only the dot products the mask names."""
    desc = _default_desc(desc)
    if desc.mask_mode is MaskMode.COMPLEMENT:
        raise ValueError("complemented matrix masks are not supported")
    bo = B.orient(not desc.transpose_inp1)       # col_view(transpose_inp1)
    b_rows = B.ncols if desc.transpose_inp1 else B.nrows
    b_cols = B.nrows if desc.transpose_inp1 else B.ncols
    if A.ncols != b_rows:
        raise ShapeError(f"inner dimensions differ: {A.ncols} vs {b_rows}")
    if mask.nrows != A.nrows or mask.ncols != b_cols:
        raise ShapeError("mask shape must match the product shape")
    dtype = np.result_type(A.dtype, B.dtype)
    add, mult = fold_op_id(semiring.add.op), pair_op_id(semiring.multiply)
    sa, ka = A.orient(False).csr_struct(dtype)
    sb, kb = bo.csr_struct(dtype)
    sm, km = mask.orient(False).csr_struct()
    nnz_m = mask.nnz
    off = empty(mask.nrows + 1, np.int64)
    oi = empty(max(nnz_m, 1), np.int32)
    ov = empty(max(nnz_m, 1), dtype)
    cnt = _counters_tensor()
    c = C.c_int64(0)
    _ctx().call("gb_mxm_masked", add, mult, C.byref(sa), C.byref(sb), C.byref(sm), _lib.ptr(off),
                _lib.ptr(oi), _lib.ptr(ov), C.byref(c), _lib.ptr(cnt))
    _merge_counters(desc, cnt)
    nnz = int(c.value)
    return SparseMatrix.from_csr(mask.nrows, mask.ncols, off, oi[:nnz], ov[:nnz], build_csc=True)


# ---------------------------------------------------------------------------
# element-wise  (kernels.py:398-512)
# ---------------------------------------------------------------------------


def _add_identity(op, dtype):
    if isinstance(op, Semiring):
        return op.add.identity_for(dtype)
    if isinstance(op, Monoid):
        return op.identity_for(dtype)
    raise TypeError(
        f"{op.name!r} has no identity; pass a monoid or semiring for this operation")


def _maybe_identity(op, dtype):
    if isinstance(op, (Semiring, Monoid)):
        return _add_identity(op, dtype)
    return None


def _sparse_result(idx_t, vals_t, size, dt, mask, mode):
    bm = _mask_bitmap(mask, size, mode)
    idx_t, vals_t = _filter(idx_t, vals_t, dt, bm)
    return Vector._wrap(size, idx_t, vals_t, 0, dt)


def _dense_pair(opid, dt, a_t, b_t, scalar, swap, bm, zero, n):
    out = empty(n, dt)
    if n:
        _ctx().call("gb_ewise_dense", opid, _code(dt), int(n), _lib.ptr(_as(a_t, dt)),
                    _lib.ptr(None if b_t is None else _as(b_t, dt)),
                    _buf(0 if scalar is None else scalar, dt), 1 if swap else 0, _lib.ptr(bm),
                    _buf(zero, dt), _lib.ptr(out))
    return out


def ewise_add(op: OpLike, u: Vector, v, mask=None, desc=None) -> Vector:
    """Union combine: both present -> op, one present -> copy (kernels.py:422-478)."""
    desc = _default_desc(desc)
    add = add_op_of(op)
    if not isinstance(v, Vector):
        dtype = device_dtype(np.result_type(u.dtype, v))
        identity = _maybe_identity(op, dtype)
        if u.is_sparse:
            if identity is None:
                _add_identity(op, dtype)
            base = u.to_dense(identity)
        else:
            base = u
        zero = identity if identity is not None else dtype.type(0)
        bm = _mask_bitmap(mask, u.size, desc.mask_mode)
        out = _dense_pair(pair_op_id(add), dtype, base._vals, None, dtype.type(v), False, bm,
                          zero, u.size)
        return Vector._wrap(u.size, None, out, zero, dtype)
    if u.size != v.size:
        raise ShapeError(f"vector sizes differ: {u.size} vs {v.size}")
    dtype = device_dtype(np.result_type(u.dtype, v.dtype))
    if u.is_sparse and v.is_sparse:
        ka, kb = int(u._idx.numel()), int(v._idx.numel())
        if ka + kb == 0:
            return _sparse_result(empty(0, np.int32), empty(0, dtype), u.size, dtype, mask,
                                  desc.mask_mode)
        fop = fold_op_id(add)               # Monoid(add, 0).segment_reduce (kernels.py:463-464)
        oi = empty(ka + kb, np.int32)
        ov = empty(ka + kb, dtype)
        c = C.c_int64(0)
        _ctx().call("gb_union_sparse", fop, _code(dtype), ka, _lib.ptr(u._idx),
                    _lib.ptr(_as(u._vals, dtype)), kb, _lib.ptr(v._idx),
                    _lib.ptr(_as(v._vals, dtype)), _lib.ptr(oi), _lib.ptr(ov), C.byref(c))
        n = int(c.value)
        return _sparse_result(oi[:n], ov[:n], u.size, dtype, mask, desc.mask_mode)
    identity = _maybe_identity(op, dtype)
    if identity is None and (u.is_sparse or v.is_sparse or mask is not None):
        _add_identity(op, dtype)
    ud = u._vals if not u.is_sparse else u.to_dense(identity)._vals
    vd = v._vals if not v.is_sparse else v.to_dense(identity)._vals
    zero = identity if identity is not None else dtype.type(0)
    bm = _mask_bitmap(mask, u.size, desc.mask_mode)
    out = _dense_pair(pair_op_id(add), dtype, ud, vd, None, False, bm, zero, u.size)
    return Vector._wrap(u.size, None, out, zero, dtype)


def ewise_mult(op: OpLike, u: Vector, v: Vector, mask=None, desc=None) -> Vector:
    """Intersection combine; dense operands are present everywhere (kernels.py:481-512)."""
    desc = _default_desc(desc)
    mult = mult_op_of(op)
    if u.size != v.size:
        raise ShapeError(f"vector sizes differ: {u.size} vs {v.size}")
    dtype = device_dtype(np.result_type(u.dtype, v.dtype))
    opid = pair_op_id(mult)
    if u.is_sparse and v.is_sparse:
        ka, kb = int(u._idx.numel()), int(v._idx.numel())
        bm = _mask_bitmap(mask, u.size, desc.mask_mode)
        oi = empty(max(ka, 1), np.int32)
        ov = empty(max(ka, 1), dtype)
        c = C.c_int64(0)
        if ka:
            _ctx().call("gb_intersect_sparse", opid, _code(dtype), ka, _lib.ptr(u._idx),
                        _lib.ptr(_as(u._vals, dtype)), kb, _lib.ptr(v._idx),
                        _lib.ptr(_as(v._vals, dtype)), _lib.ptr(bm), _lib.ptr(oi), _lib.ptr(ov),
                        C.byref(c))
        n = int(c.value)
        return Vector._wrap(u.size, oi[:n], ov[:n], 0, dtype)
    if u.is_sparse or v.is_sparse:
        sp, dn = (u, v) if u.is_sparse else (v, u)
        k = int(sp._idx.numel())
        out = empty(k, dtype)
        if k:
            _ctx().call("gb_gather_pair", opid, _code(dtype), k, _lib.ptr(sp._idx),
                        _lib.ptr(_as(sp._vals, dtype)), _lib.ptr(_as(dn._vals, dtype)),
                        0 if u.is_sparse else 1, _lib.ptr(out))
        return _sparse_result(sp._idx.clone(), out, u.size, dtype, mask, desc.mask_mode)
    bm = _mask_bitmap(mask, u.size, desc.mask_mode)
    out = _dense_pair(opid, dtype, u._vals, v._vals, None, False, None, 0, u.size)
    if bm is not None:
        i, vals = _filter(iota(u.size), out, dtype, bm)
        return Vector._wrap(u.size, i, vals, 0, dtype)
    return Vector._wrap(u.size, None, out, 0, dtype)


# ---------------------------------------------------------------------------
# assign / scatter / gather / apply / reduce  (kernels.py:519-665)
# ---------------------------------------------------------------------------


def _densify_in_place(w):
    if w.is_sparse:
        d = w.to_dense(w.zero)
        w._idx, w._vals = None, d._vals


def assign(w: Vector, value, mask=None, desc=None, indices=None) -> Vector:
    """Write a scalar at every mask-allowed position of w, in place (kernels.py:519-535)."""
    desc = _default_desc(desc)
    bm = _mask_bitmap(mask, w.size, desc.mask_mode)
    if indices is not None:
        sel = to_dev(np.asarray(indices, dtype=INDEX_DTYPE), np.int32)
        if bm is not None:
            sel, _ = _filter(sel, empty(int(sel.numel()), np.int64), np.int64, bm)
        bm = _bitmap_of_indices(sel, w.size)
    if w.size == 0:
        return w
    if bm is not None and _bitmap_count(bm, w.size) == 0:
        return w
    _densify_in_place(w)
    _ctx().call("gb_assign_scalar", _code(w._dt), int(w.size), _lib.ptr(w._vals),
                _buf(w._dt.type(value), w._dt), _lib.ptr(bm))
    return w


def _stored_positions(vec):
    """(positions int32 tensor or None=all, values tensor) of a vector's stored entries."""
    return vec._idx, vec._vals


def _targets_and_values(values, indices):
    """kernels.py:544-559: the (target, value) pairs an assign_scatter consumes."""
    dev = values._vals.device
    if not (indices.is_sparse or values.is_sparse):
        return indices._vals, values._vals
    if indices.is_sparse and values.is_sparse:
        # k = intersect1d(indices.k, values.k); tgt/val at k
        ki, kv = int(indices._idx.numel()), int(values._idx.numel())
        out_t = empty(max(ki, 1), indices._dt)
        out_v = empty(max(ki, 1), values._dt)
        idx_buf = empty(max(ki, 1), np.int32)
        c = C.c_int64(0)
        if ki:
            _ctx().call("gb_intersect_sparse", _lib.OP_FIRST, _code(indices._dt), ki,
                        _lib.ptr(indices._idx), _lib.ptr(indices._vals), kv,
                        _lib.ptr(values._idx), _lib.ptr(_as(values._vals, indices._dt)), None,
                        _lib.ptr(idx_buf), _lib.ptr(out_t), C.byref(c))
        n = int(c.value)
        common = idx_buf[:n]
        tgt = out_t[:n]
        # values at the common positions: gather from the dense image of `values`
        vd = values.to_dense(values.zero)._vals
        val = gather32(vd, common) if n else empty(0, values._dt)
        return tgt, val
    if indices.is_sparse:
        k = indices._idx
        return indices._vals, gather32(values._vals, k)
    k = values._idx
    return gather32(indices._vals, k), values._vals


def assign_scatter(w: Vector, values: Vector, indices: Vector, mask=None, desc=None) -> Vector:
    """w(indices(k)) <- values(k); colliding targets keep the minimum (kernels.py:538-583)."""
    desc = _default_desc(desc)
    if values.size != indices.size:
        raise ShapeError("values and indices must have equal size")
    tgt, val = _targets_and_values(values, indices)
    tgt = _as(tgt, np.int64)
    k = int(tgt.numel())
    if k:
        bad = C.c_int32(0)
        _ctx().call("gb_check_bounds", k, _lib.ptr(tgt), int(w.size), C.byref(bad))
        if bad.value:
            raise IndexError("scatter target index out of range")
    bm = _mask_bitmap(mask, w.size, desc.mask_mode)
    if bm is not None and k:
        t32, v2 = _filter(_as(tgt, np.int32), val, values._dt, bm)
        tgt, val = _as(t32, np.int64), v2
        k = int(tgt.numel())
    if k == 0:
        return w
    _densify_in_place(w)
    _ctx().call("gb_scatter_min", _code(w._dt), int(w.size), _lib.ptr(w._vals), k, _lib.ptr(tgt),
                _lib.ptr(_as(val, w._dt)), None)
    return w


def extract_gather(w: Vector, u: Vector, indices: Vector, mask=None, desc=None) -> Vector:
    """w(k) = u(indices(k)) for stored k of ``indices``; replaces w (kernels.py:586-619)."""
    desc = _default_desc(desc)
    dev = u._vals.device
    if indices.is_sparse:
        k = indices._idx
    else:
        k = iota(indices.size)
    gather = _as(indices._vals, np.int64)
    n = int(gather.numel())
    dt = u._dt
    if u.is_sparse:
        present = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        vals = empty(max(n, 1), dt)
        if n:
            _ctx().call("gb_gather_sparse", _code(dt), n, _lib.ptr(gather), int(u.size),
                        int(u._idx.numel()), _lib.ptr(u._idx), _lib.ptr(u._vals),
                        _lib.ptr(present), _lib.ptr(vals))
            ko = empty(n, np.int32)
            vo = empty(n, dt)
            c = C.c_int64(0)
            _ctx().call("gb_select_flags", n, _lib.ptr(present), _lib.ptr(k), _lib.ptr(vals),
                        _code(dt), _lib.ptr(ko), _lib.ptr(vo), C.byref(c))
            k, vals = ko[:c.value], vo[:c.value]
        else:
            vals = vals[:0]
        sparse_out = True
    else:
        vals = empty(n, dt)
        if n:
            _ctx().call("gb_gather", _code(dt), n, _lib.ptr(gather), int(u.size), _lib.ptr(u._vals),
                        _lib.ptr(vals))
        sparse_out = indices.is_sparse
    bm = _mask_bitmap(mask, w.size, desc.mask_mode)
    if bm is not None:
        k, vals = _filter(_as(k, np.int32), vals, dt, bm)
        sparse_out = True
    w._idx = _as(k, np.int32).clone() if sparse_out else None
    w._vals = vals.clone()
    w._dt = dt
    w.zero = dt.type(w.zero)
    return w


def _affine_of(fn, dt):
    """(scale, shift) when fn is exactly affine on integer probes, else None."""
    probe = np.array([0, 1, 2, 3, -7, 1000], dtype=dt)
    try:
        out = np.asarray(fn(probe.copy()))
    except Exception:
        return None
    if out.shape != probe.shape or out.dtype != dt:
        return None
    b = out[0]
    a = out[1] - out[0]
    with np.errstate(over="ignore"):
        if np.array_equal(out, probe * a + b):
            return a, b
    return None


def apply(fn, u: Vector, mask=None, desc=None) -> Vector:
    """Map a unary function over stored entries, dropping masked-off ones (kernels.py:622-639).

    Identity maps and exact integer affine maps run in the native kernel; any
    other ``fn`` is evaluated on the device tensor of values (it must accept
    array-likes, as the reference requires)."""
    desc = _default_desc(desc)
    bm = _mask_bitmap(mask, u.size, desc.mask_mode)
    if bm is None:
        idx, vals = u._idx, u._vals
    elif u.is_sparse:
        idx, vals = _filter(u._idx, u._vals, u._dt, bm)
    else:
        idx, vals = _filter(iota(u.size), u._vals, u._dt, bm)
    out = _apply_values(fn, vals, u._dt)
    odt = device_dtype(np.dtype(str(out.dtype).replace("torch.", "")))
    if bm is None and not u.is_sparse:
        return Vector._wrap(u.size, None, out, u.zero, odt)
    return Vector._wrap(u.size, None if idx is None else idx.clone(), out, u.zero, odt)


def _apply_values(fn, vals, dt):
    probe = np.array([0, 1, 5, -3], dtype=dt)
    try:
        is_identity = np.array_equal(np.asarray(fn(probe.copy())), probe) and \
            np.asarray(fn(probe.copy())).dtype == dt
    except Exception:
        is_identity = False
    if is_identity:
        return vals.clone()
    if dt.kind == "i":
        ab = _affine_of(fn, dt)
        if ab is not None:
            out = empty(int(vals.numel()), dt)
            if vals.numel():
                _ctx().call("gb_apply_affine", _code(dt), int(vals.numel()), _lib.ptr(vals),
                            _buf(ab[0], dt), _buf(ab[1], dt), _lib.ptr(out))
            return out
    res = fn(vals)
    if not isinstance(res, torch.Tensor):
        res = torch.as_tensor(np.asarray(res), device=vals.device)
    return res.to(_TORCH[device_dtype(np.dtype(str(res.dtype).replace("torch.", "")))])


def _fold_values(monoid, vals_t, dt, zero=None):
    """Fold a device value array (values equal to ``zero`` skipped) -> numpy scalar."""
    n = int(vals_t.numel())
    if n == 0:
        return monoid.identity_for(dt)
    op = fold_op_id(monoid.op)
    out = C.create_string_buffer(8)
    cnt = C.c_int64(0)
    _ctx().call("gb_reduce", op, _code(dt), n, _lib.ptr(_as(vals_t, dt)),
                None if zero is None else _buf(zero, dt), out, C.byref(cnt))
    if cnt.value == 0:
        return monoid.identity_for(dt)
    return np.frombuffer(out.raw, dtype=dt)[0]


def reduce(monoid: Monoid, u: Vector):
    """Fold all stored entries of a vector down to one scalar (kernels.py:642-647)."""
    if u.is_sparse:
        return _fold_values(monoid, u._vals, u._dt)
    return _fold_values(monoid, u._vals, u._dt, zero=u.zero)


def reduce_rows(monoid: Monoid, A: SparseMatrix) -> Vector:
    """Per-row reduction of stored values; empty rows give the identity (kernels.py:650-660)."""
    dt = A.dtype
    identity = monoid.identity_for(dt)
    o = A.orient(False)
    s, keep = o.csr_struct()
    out = empty(A.nrows, dt)
    if A.nrows:
        _ctx().call("gb_reduce_rows", fold_op_id(monoid.op), C.byref(s), _lib.ptr(out))
    return Vector._wrap(A.nrows, None, out, identity, dt)


def reduce_scalar_matrix(monoid: Monoid, A: SparseMatrix):
    """Fold every stored matrix entry down to one scalar (kernels.py:663-665)."""
    return _fold_values(monoid, A.orient(False).dense_values(), A.dtype)


def transpose(A: SparseMatrix) -> SparseMatrix:
    """Reverse every edge; O(1) when both layouts are stored (kernels.py:668-676)."""
    if not A.has_csc:
        A._build_csc()
    return SparseMatrix._wrap(A.ncols, A.nrows, A._csc, A._csr, A._dt, A._sym)
