"""numpy restatement of the reference operator layer and algorithms (TEST ORACLE).

Every function cites the reference file:line whose semantics it restates
(paths relative to ``/root/reference/pkg/src/graphalg/``).  The structure is
deliberately flat -- plain records plus free functions -- and it is only ever
used as the checker for the CUDA path (see ``oracle/__init__.py``).

Value conventions restated here (the A-notes of SURVEY.md §8(a)):
* ``mult(A value, u value)``: the matrix operand is always first
  (kernels.py:172,182,261).
* semiring add-monoids fold with the plain ufunc (wrapping int add,
  algebra.py:98-126); ``Plus`` used as a *pairwise* op saturates at the int64
  bounds (algebra.py:24-38, 146).
* outputs equal to the add identity are never stored (kernels.py:229, 277).
* a stored 0 in a sparse mask blocks the write (kernels.py:67-84).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

I64 = np.int64
I64_MAX = np.iinfo(np.int64).max
I64_MIN = np.iinfo(np.int64).min

# ---------------------------------------------------------------------------
# algebra  (algebra.py:24-195)
# ---------------------------------------------------------------------------


def _sat_add(x, y):
    """algebra.py:24-38 -- int add clamped at the int64 bounds, float add plain."""
    x, y = np.asarray(x), np.asarray(y)
    if x.dtype.kind == "f" or y.dtype.kind == "f":
        return x + y
    info = np.iinfo(np.result_type(x, y))
    with np.errstate(over="ignore"):
        out = x + y
    hi = (y > 0) & (x > info.max - y)
    lo = (y < 0) & (x < info.min - y)
    return np.where(hi, info.max, np.where(lo, info.min, out))


# name -> (pairwise array function, folding ufunc)
OPS = {
    "Plus": (_sat_add, np.add),
    "Minus": (np.subtract, np.subtract),
    "Multiplies": (np.multiply, np.multiply),
    "Minimum": (np.minimum, np.minimum),
    "Maximum": (np.maximum, np.maximum),
    "LogicalOr": (np.logical_or, np.logical_or),
    "LogicalAnd": (np.logical_and, np.logical_and),
    "Less": (np.less, np.less),
    "NotEqualTo": (np.not_equal, np.not_equal),
    "SelectSecond": (lambda x, y: np.broadcast_arrays(x, y)[1].copy(), None),
}

# monoid name -> identity (algebra.py:160-167)
MONOID_IDENTITY = {"Plus": 0.0, "Multiplies": 1.0, "Minimum": math.inf, "Maximum": -math.inf,
                   "LogicalOr": 0.0, "LogicalAnd": 1.0}

# semiring name -> (add monoid, multiply op) (algebra.py:169-179)
SEMIRINGS = {
    "PlusMultiplies": ("Plus", "Multiplies"),
    "LogicalOrAnd": ("LogicalOr", "LogicalAnd"),
    "MinPlus": ("Minimum", "Plus"),
    "MaxPlus": ("Maximum", "Plus"),
    "MinMultiplies": ("Minimum", "Multiplies"),
    "MinimumSelectSecond": ("Minimum", "SelectSecond"),
    "PlusLess": ("Plus", "Less"),
    "MinimumNotEqualTo": ("Minimum", "NotEqualTo"),
}


def identity_for(monoid, dtype):
    """algebra.py:88-96 -- +/-inf become the integer bounds."""
    dtype = np.dtype(dtype)
    ident = MONOID_IDENTITY[monoid]
    if dtype.kind == "f":
        return dtype.type(ident)
    if ident == math.inf:
        return dtype.type(np.iinfo(dtype).max)
    if ident == -math.inf:
        return dtype.type(np.iinfo(dtype).min)
    return dtype.type(ident)


def pairwise(op, x, y, dtype):
    """algebra.py:62-70 -- apply and cast to the domain dtype."""
    with np.errstate(over="ignore", invalid="ignore"):
        return np.asarray(OPS[op][0](x, y)).astype(dtype, copy=False)


def fold(monoid, values, dtype):
    """algebra.py:98-110 -- fold to a scalar; empty gives the identity."""
    values = np.asarray(values)
    if values.size == 0:
        return identity_for(monoid, dtype)
    with np.errstate(over="ignore"):
        return np.dtype(dtype).type(OPS[monoid][1].reduce(values))


def segfold(monoid, values, starts, dtype):
    """algebra.py:112-126 -- reduceat over nonempty segments."""
    if len(starts) == 0:
        return np.empty(0, dtype)
    with np.errstate(over="ignore"):
        return np.asarray(OPS[monoid][1].reduceat(values, starts)).astype(dtype, copy=False)


# ---------------------------------------------------------------------------
# containers  (containers.py:49-464)
# ---------------------------------------------------------------------------


@dataclass
class Counters:
    reads: int = 0
    mults: int = 0
    adds: int = 0

    def as_list(self):
        return [self.reads, self.mults, self.adds]


@dataclass
class Desc:
    """containers.py:74-113 (only the fields the path reads)."""
    complement: bool = False
    transpose0: bool = False
    transpose1: bool = False
    direction: str = "auto"
    switch_ratio: float = 0.1
    max_niter: int = 10_000
    early_exit: bool = False
    counters: Counters = field(default_factory=Counters)
    log: list = field(default_factory=list)


@dataclass
class Vec:
    """containers.py:116-257: sparse = (sorted idx, vals); dense = vals + zero."""
    size: int
    idx: Optional[np.ndarray]
    vals: np.ndarray
    zero: object

    @property
    def sparse(self):
        return self.idx is not None

    def nvals_for(self, z):  # containers.py:179-182
        return int(self.idx.size) if self.sparse else int(np.count_nonzero(self.vals != z))

    def tuples(self):  # containers.py:209-218
        if self.sparse:
            return self.idx.copy(), self.vals.copy()
        i = np.flatnonzero(self.vals != self.zero).astype(I64)
        return i, self.vals[i].copy()

    def dense(self, z=None):  # containers.py:230-240
        z = self.zero if z is None else z
        if not self.sparse:
            return Vec(self.size, None, self.vals.copy(), self.vals.dtype.type(z))
        v = np.full(self.size, z, dtype=self.vals.dtype)
        v[self.idx] = self.vals
        return Vec(self.size, None, v, v.dtype.type(z))

    def sparsify(self, z=None):  # containers.py:242-252
        z = self.zero if z is None else z
        if self.sparse:
            k = self.vals != z
            return Vec(self.size, self.idx[k], self.vals[k], self.vals.dtype.type(z))
        i = np.flatnonzero(self.vals != z).astype(I64)
        return Vec(self.size, i, self.vals[i].copy(), self.vals.dtype.type(z))

    def copy(self):
        return Vec(self.size, None if self.idx is None else self.idx.copy(), self.vals.copy(), self.zero)


def vec_entries(idx, vals, size, dtype=None):
    """containers.py:135-147 (sorted, duplicate check)."""
    idx = np.asarray(idx, dtype=I64).ravel()
    vals = np.asarray(vals, dtype=dtype).ravel()
    o = np.argsort(idx, kind="stable")
    idx, vals = idx[o], vals[o]
    if idx.size > 1 and (np.diff(idx) == 0).any():
        raise ValueError("duplicate index")
    return Vec(size, idx, vals, vals.dtype.type(0))


def vec_filled(size, value, dtype=None):
    v = np.full(size, value, dtype=dtype)
    return Vec(size, None, v, v.dtype.type(0))


@dataclass
class Mat:
    """containers.py:276-451: CSR + optional CSC mirror."""
    nrows: int
    ncols: int
    rp: np.ndarray
    ci: np.ndarray
    cv: np.ndarray
    cp: Optional[np.ndarray] = None
    ri: Optional[np.ndarray] = None
    rv: Optional[np.ndarray] = None

    @property
    def nnz(self):
        return int(self.ci.size)

    def rows(self, transpose=False):  # containers.py:384-389
        if not transpose:
            return self.rp, self.ci, self.cv
        if self.cp is None:
            raise RuntimeError("FormatError: no CSC")
        return self.cp, self.ri, self.rv

    def cols(self, transpose=False):  # containers.py:391-396
        if transpose:
            return self.rp, self.ci, self.cv
        if self.cp is None:
            raise RuntimeError("FormatError: no CSC")
        return self.cp, self.ri, self.rv

    def tuples(self):
        r = np.repeat(np.arange(self.nrows, dtype=I64), np.diff(self.rp))
        return r, self.ci.copy(), self.cv.copy()


def mat_from_tuples(rows, cols, vals, nrows, ncols, dedup="Plus", csc=True, dtype=None):
    """containers.py:307-345 and _build_csc 357-364."""
    rows = np.asarray(rows, dtype=I64).ravel()
    cols = np.asarray(cols, dtype=I64).ravel()
    vals = np.asarray(vals, dtype=dtype).ravel()
    if vals.dtype == object:
        vals = vals.astype(np.float64)
    o = np.lexsort((cols, rows))
    rows, cols, vals = rows[o], cols[o], vals[o]
    if rows.size:
        first = np.r_[True, (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])]
        st = np.flatnonzero(first)
        vals = segfold(dedup, vals, st, vals.dtype)
        rows, cols = rows[st], cols[st]
    rp = np.zeros(nrows + 1, I64)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp).astype(I64)
    m = Mat(nrows, ncols, rp, cols, vals)
    if csc:
        add_csc(m)
    return m


def add_csc(m):
    r = np.repeat(np.arange(m.nrows, dtype=I64), np.diff(m.rp))
    o = np.argsort(m.ci, kind="stable")
    m.ri, m.rv = r[o], m.cv[o]
    cp = np.zeros(m.ncols + 1, I64)
    np.add.at(cp, m.ci + 1, 1)
    m.cp = np.cumsum(cp).astype(I64)
    return m


def transpose(m):
    """kernels.py:668-676."""
    if m.cp is None:
        add_csc(m)
    return Mat(m.ncols, m.nrows, m.cp, m.ri, m.rv, m.rp, m.ci, m.cv)


# ---------------------------------------------------------------------------
# operator layer  (kernels.py)
# ---------------------------------------------------------------------------


def allowed_of(mask, size, complement):
    """kernels.py:67-84."""
    if mask is None:
        return None
    if mask.size != size:
        raise ValueError("ShapeError: mask size")
    if mask.sparse:
        a = np.zeros(size, bool)
        a[mask.idx[mask.vals != 0]] = True
    else:
        a = mask.vals != 0
    return ~a if complement else a


def decide(nnz_u, nnz, nrows, desc):
    """kernels.py:108-126 -- Python round() is half-even."""
    d = nnz / nrows if nrows else 0.0
    est = int(round(d * nnz_u))
    thr = nnz * desc.switch_ratio
    if desc.direction == "force-push":
        ch = "push"
    elif desc.direction == "force-pull":
        ch = "pull"
    else:
        ch = "pull" if est > thr else "push"
    return [ch, nnz_u, est, thr]


def pull(sr, A, u, mask, desc, transpose):
    """kernels.py:153-229 (single span; spans never change values or counters)."""
    add, mul = SEMIRINGS[sr]
    off, ind, val = A.rows(transpose)
    out_n = A.ncols if transpose else A.nrows
    in_n = A.nrows if transpose else A.ncols
    if u.sparse:
        raise RuntimeError("FormatError: pull needs dense u")
    if u.size != in_n:
        raise ValueError("ShapeError")
    dt = np.result_type(val, u.vals)
    ident = identity_for(add, dt)
    allowed = allowed_of(mask, out_n, desc.complement)
    early = desc.early_exit and add == "LogicalOr"
    out = np.full(out_n, ident, dtype=dt)
    rows = np.arange(out_n) if allowed is None else np.flatnonzero(allowed)
    for i in rows:
        lo, hi = off[i], off[i + 1]
        if hi == lo:
            continue
        cols, av = ind[lo:hi], val[lo:hi]
        uv = u.vals[cols]
        inc = uv != ident
        if early:
            hit = inc & (pairwise(mul, av, uv, dt) != ident)
            desc.counters.reads += int(np.argmax(hit)) + 1 if hit.any() else int(hi - lo)
        else:
            desc.counters.reads += int(hi - lo)
        p = pairwise(mul, av[inc], uv[inc], dt)
        desc.counters.mults += int(p.size)
        if p.size:
            out[i] = segfold(add, p, np.array([0]), dt)[0]
            desc.counters.adds += int(p.size - 1)
    return Vec(out_n, None, out, ident)


def push(sr, A, u, mask, desc, transpose):
    """kernels.py:242-280 -- expand, stable sort by row, fold, drop identity, mask after."""
    add, mul = SEMIRINGS[sr]
    off, ind, val = A.cols(transpose)
    out_n = A.ncols if transpose else A.nrows
    in_n = A.nrows if transpose else A.ncols
    if not u.sparse:
        raise RuntimeError("FormatError: push needs sparse u")
    if u.size != in_n:
        raise ValueError("ShapeError")
    dt = np.result_type(val, u.vals)
    ident = identity_for(add, dt)
    allowed = allowed_of(mask, out_n, desc.complement)
    lens = off[u.idx + 1] - off[u.idx]
    pos = np.concatenate([np.arange(off[j], off[j + 1]) for j in u.idx]) if u.idx.size else np.empty(0, I64)
    pos = pos.astype(I64)
    rows = ind[pos]
    prods = pairwise(mul, val[pos], np.repeat(u.vals, lens), dt)
    desc.counters.mults += int(prods.size)
    if rows.size:
        o = np.argsort(rows, kind="stable")
        rows, prods = rows[o], prods[o]
        st = np.flatnonzero(np.r_[True, rows[1:] != rows[:-1]])
        oi, ov = rows[st], segfold(add, prods, st, dt)
        desc.counters.adds += int(prods.size - st.size)
    else:
        oi, ov = np.empty(0, I64), np.empty(0, dt)
    keep = ov != ident
    if allowed is not None:
        keep &= allowed[oi]
    return Vec(out_n, oi[keep], ov[keep], ident)


def mv(sr, A, u, mask, desc, transpose):
    """kernels.py:293-310 dispatch (mxv: transpose=desc.transpose0; vxm: not transpose1)."""
    out_n = A.ncols if transpose else A.nrows
    in_n = A.nrows if transpose else A.ncols
    if u.size != in_n:
        raise ValueError("ShapeError")
    if mask is not None and mask.size != out_n:
        raise ValueError("ShapeError")
    add, _ = SEMIRINGS[sr]
    dt = np.result_type(A.cv, u.vals)
    ident = identity_for(add, dt)
    dec = decide(u.nvals_for(ident), A.nnz, A.nrows, desc)
    desc.log.append(dec)
    if dec[0] == "pull":
        return pull(sr, A, u if not u.sparse else u.dense(ident), mask, desc, transpose)
    return push(sr, A, u if u.sparse else u.sparsify(ident), mask, desc, transpose)


def mxv(sr, A, u, mask=None, desc=None):
    desc = desc or Desc()
    return mv(sr, A, u, mask, desc, desc.transpose0)


def vxm(sr, u, A, mask=None, desc=None):
    desc = desc or Desc()
    return mv(sr, A, u, mask, desc, not desc.transpose1)


def mxm_masked(sr, A, B, M, desc=None):
    """kernels.py:329-391 -- one dot product per nonzero mask entry."""
    desc = desc or Desc()
    add, mul = SEMIRINGS[sr]
    boff, bidx, bval = B.cols(desc.transpose1)
    dt = np.result_type(A.cv, bval)
    ident = identity_for(add, dt)
    out = []
    mr, mc, mv_ = M.tuples()
    for i, j in zip(mr[mv_ != 0], mc[mv_ != 0]):
        ai, av = A.ci[A.rp[i]:A.rp[i + 1]], A.cv[A.rp[i]:A.rp[i + 1]]
        bi, bv = bidx[boff[j]:boff[j + 1]], bval[boff[j]:boff[j + 1]]
        common, xa, xb = np.intersect1d(ai, bi, assume_unique=True, return_indices=True)
        if common.size:
            p = pairwise(mul, av[xa], bv[xb], dt)
            desc.counters.mults += int(p.size)
            desc.counters.adds += int(p.size - 1)
            out.append((i, j, fold(add, p, dt)))
        elif ident != dt.type(0):
            out.append((i, j, ident))
    if out:
        r, c, v = zip(*out)
    else:
        r, c, v = [], [], []
    return mat_from_tuples(r, c, np.asarray(v, dtype=dt), M.nrows, M.ncols, dtype=dt)


def ewise_add(op, u, v, mask=None, desc=None, identity=None):
    """kernels.py:422-478.  ``op`` is the add-op name, ``identity`` the monoid
    identity when op came from a Semiring/Monoid (None for a bare op)."""
    desc = desc or Desc()
    if not isinstance(v, Vec):
        dt = np.result_type(u.vals, v)
        ident = None if identity is None else identity_for(identity, dt)
        if u.sparse:
            if ident is None:
                raise TypeError("no identity")
            base = u.dense(ident)
        else:
            base = u
        out = pairwise(op, base.vals, v, dt)
        z = ident if ident is not None else dt.type(0)
        a = allowed_of(mask, u.size, desc.complement)
        if a is not None:
            out[~a] = z
        return Vec(u.size, None, out, dt.type(z))
    if u.size != v.size:
        raise ValueError("ShapeError")
    dt = np.result_type(u.vals, v.vals)
    if u.sparse and v.sparse:
        idx = np.concatenate([u.idx, v.idx])
        vals = np.concatenate([u.vals.astype(dt), v.vals.astype(dt)])
        if idx.size:
            o = np.argsort(idx, kind="stable")
            idx, vals = idx[o], vals[o]
            st = np.flatnonzero(np.r_[True, idx[1:] != idx[:-1]])
            # Monoid(op, 0).segment_reduce -> reduceat of the op's ufunc, or the
            # scalar fn for ops without one (kernels.py:463-464, algebra.py:121-126)
            if OPS[op][1] is None:  # SelectSecond: fold keeps the last value
                ends = np.r_[st[1:], idx.size] - 1
                vals = vals[ends]
            else:
                vals = segfold(op, vals, st, dt)
            idx = idx[st]
        a = allowed_of(mask, u.size, desc.complement)
        if a is not None:
            k = a[idx]
            idx, vals = idx[k], vals[k]
        return Vec(u.size, idx, vals, dt.type(0))
    ident = None if identity is None else identity_for(identity, dt)
    if ident is None and (u.sparse or v.sparse or mask is not None):
        raise TypeError("no identity")
    ud = u.vals if not u.sparse else u.dense(ident).vals
    vd = v.vals if not v.sparse else v.dense(ident).vals
    out = pairwise(op, ud, vd, dt)
    z = ident if ident is not None else dt.type(0)
    a = allowed_of(mask, u.size, desc.complement)
    if a is not None:
        out = np.where(a, out, z)
    return Vec(u.size, None, out, dt.type(z))


def ewise_mult(op, u, v, mask=None, desc=None):
    """kernels.py:481-512."""
    desc = desc or Desc()
    if u.size != v.size:
        raise ValueError("ShapeError")
    dt = np.result_type(u.vals, v.vals)

    def masked(idx, vals):
        a = allowed_of(mask, u.size, desc.complement)
        if a is not None:
            k = a[idx]
            idx, vals = idx[k], vals[k]
        return Vec(u.size, idx, vals, dt.type(0))

    if u.sparse and v.sparse:
        c, ui, vi = np.intersect1d(u.idx, v.idx, assume_unique=True, return_indices=True)
        return masked(c.astype(I64), pairwise(op, u.vals[ui], v.vals[vi], dt))
    if u.sparse:
        return masked(u.idx.copy(), pairwise(op, u.vals, v.vals[u.idx], dt))
    if v.sparse:
        return masked(v.idx.copy(), pairwise(op, u.vals[v.idx], v.vals, dt))
    out = pairwise(op, u.vals, v.vals, dt)
    a = allowed_of(mask, u.size, desc.complement)
    if a is not None:
        i = np.flatnonzero(a).astype(I64)
        return Vec(u.size, i, out[a], dt.type(0))
    return Vec(u.size, None, out, dt.type(0))


def assign(w, value, mask=None, desc=None, indices=None):
    """kernels.py:519-535 (in place)."""
    desc = desc or Desc()
    a = allowed_of(mask, w.size, desc.complement)
    if a is None:
        a = np.ones(w.size, bool)
    if indices is not None:
        s = np.zeros(w.size, bool)
        s[np.asarray(indices, dtype=I64)] = True
        a = a & s
    if not a.any():
        return w
    if w.sparse:
        d = w.dense(w.zero)
        w.idx, w.vals = None, d.vals
    w.vals[a] = value
    return w


def _stored_at(vec, k):
    return vec.vals[np.searchsorted(vec.idx, k)] if vec.sparse else vec.vals[k]


def assign_scatter(w, values, indices, mask=None, desc=None):
    """kernels.py:538-583 -- w[idx(k)] = min_k val(k), overwrite."""
    desc = desc or Desc()
    if values.size != indices.size:
        raise ValueError("ShapeError")
    if indices.sparse or values.sparse:
        ki = indices.tuples()[0] if indices.sparse else None
        kv = values.tuples()[0] if values.sparse else None
        k = kv if ki is None else (ki if kv is None else np.intersect1d(ki, kv, assume_unique=True))
        tgt, val = _stored_at(indices, k), _stored_at(values, k)
    else:
        tgt, val = indices.vals, values.vals
    tgt = np.asarray(tgt, dtype=I64)
    if tgt.size and (tgt.min() < 0 or tgt.max() >= w.size):
        raise IndexError("scatter target")
    a = allowed_of(mask, w.size, desc.complement)
    if a is not None:
        keep = a[tgt]
        tgt, val = tgt[keep], val[keep]
    if tgt.size == 0:
        return w
    o = np.argsort(tgt, kind="stable")
    tgt, val = tgt[o], val[o]
    st = np.flatnonzero(np.r_[True, tgt[1:] != tgt[:-1]])
    comb = np.minimum.reduceat(val, st)
    if w.sparse:
        d = w.dense(w.zero)
        w.idx, w.vals = None, d.vals
    w.vals[tgt[st]] = comb
    return w


def extract_gather(w, u, indices, mask=None, desc=None):
    """kernels.py:586-619 -- w(k) = u(indices(k)), replaces w."""
    desc = desc or Desc()
    k = indices.idx if indices.sparse else np.arange(indices.size, dtype=I64)
    g = indices.vals.astype(I64)
    if g.size and (g.min() < 0 or g.max() >= u.size):
        raise IndexError("gather index")
    if u.sparse:
        if u.idx.size:
            p = np.searchsorted(u.idx, g)
            pc = np.minimum(p, u.idx.size - 1)
            present = (p < u.idx.size) & (u.idx[pc] == g)
        else:
            pc = np.zeros(g.size, I64)
            present = np.zeros(g.size, bool)
        k, vals = k[present], u.vals[pc[present]]
        sparse_out = True
    else:
        vals = u.vals[g]
        sparse_out = indices.sparse
    a = allowed_of(mask, w.size, desc.complement)
    if a is not None:
        keep = a[k]
        k, vals = k[keep], vals[keep]
        sparse_out = True
    w.idx = k.astype(I64) if sparse_out else None
    w.vals = vals.copy()
    return w


def apply(fn, u, mask=None, desc=None):
    """kernels.py:622-639."""
    desc = desc or Desc()
    a = allowed_of(mask, u.size, desc.complement)
    if a is None:
        return Vec(u.size, None if not u.sparse else u.idx.copy(), np.asarray(fn(u.vals)), u.zero)
    if u.sparse:
        keep = a[u.idx]
        i, vals = u.idx[keep], u.vals[keep]
    else:
        i = np.flatnonzero(a).astype(I64)
        vals = u.vals[i]
    return Vec(u.size, i, np.asarray(fn(vals)), u.zero)


def reduce(monoid, u):
    """kernels.py:642-647."""
    if u.sparse:
        return fold(monoid, u.vals, u.vals.dtype)
    return fold(monoid, u.vals[u.vals != u.zero], u.vals.dtype)


def reduce_rows(monoid, A):
    """kernels.py:650-660."""
    lens = np.diff(A.rp)
    dt = A.cv.dtype
    ident = identity_for(monoid, dt)
    out = np.full(A.nrows, ident, dtype=dt)
    ne = lens > 0
    if ne.any():
        out[ne] = segfold(monoid, A.cv, A.rp[:-1][ne], dt)
    return Vec(A.nrows, None, out, ident)


def reduce_scalar_matrix(monoid, A):
    """kernels.py:663-665."""
    return fold(monoid, A.cv, A.cv.dtype)


# ---------------------------------------------------------------------------
# algorithms  (algorithms.py:48-240)
# ---------------------------------------------------------------------------


def bfs(A, source, desc=None):
    """algorithms.py:48-77 -- levels 1-based, 0 unreached."""
    desc = desc or Desc()
    desc.early_exit = True
    n = A.nrows
    f = vec_entries([source], [1], n, dtype=I64)
    visited = vec_filled(n, 0, dtype=I64)
    depth = 1
    for _ in range(min(desc.max_niter, n + 1)):
        assign(visited, depth, mask=f, desc=desc)
        desc.complement = not desc.complement
        f = vxm("LogicalOrAnd", f, A, mask=visited, desc=desc)
        desc.complement = not desc.complement
        if int(reduce("Plus", f)) == 0:
            break
        depth += 1
    return visited


def sssp(A, source, desc=None, on_iteration=None):
    """algorithms.py:80-119 -- frontier-sparsified Bellman-Ford."""
    desc = desc or Desc()
    n = A.nrows
    dist = vec_filled(n, np.inf, dtype=np.float64)
    dist.zero = np.float64(np.inf)
    dist.vals[source] = 0.0
    f = vec_entries([source], [0.0], n, dtype=np.float64)
    ceiling = vec_filled(n, np.finfo(np.float64).max)
    last = -1.0
    for it in range(min(desc.max_niter, n)):
        cand = vxm("MinPlus", f, A, desc=desc)
        improved = ewise_mult("Less", cand, dist, desc=desc)
        dist = ewise_add("Minimum", dist, cand, desc=desc, identity="Minimum")
        f = apply(lambda x: x, cand, mask=improved, desc=desc)
        if on_iteration is not None:
            on_iteration(it, dist.copy())
        reached = ewise_mult("Less", dist, ceiling, desc=desc)
        succ = float(reduce("Plus", reached))
        if succ == last and f.nvals_for(f.zero) == 0:
            break
        last = succ
    return dist


def scale_rows(A, alpha):
    """algorithms.py:122-129."""
    lens = np.diff(A.rp)
    inv = np.zeros(A.nrows)
    inv[lens > 0] = alpha / lens[lens > 0]
    m = Mat(A.nrows, A.ncols, A.rp.copy(), A.ci.copy(), np.repeat(inv, lens))
    return add_csc(m)


def pagerank(A, alpha=0.85, eps=1e-7, max_iters=10_000, desc=None, on_iteration=None):
    """algorithms.py:132-162."""
    desc = desc or Desc()
    n = A.nrows
    S = scale_rows(A, alpha)
    tele = (1.0 - alpha) / n
    r = vec_filled(n, 1.0 / n)
    for it in range(max_iters):
        prev = r
        spread = vxm("PlusMultiplies", prev, S, desc=desc)
        r = ewise_add("Plus", spread, tele, desc=desc, identity="Plus")
        delta = ewise_mult("Minus", r, prev, desc=desc)
        sq = ewise_add("Multiplies", delta, delta, desc=desc)
        err = math.sqrt(float(reduce("Plus", sq)))
        if on_iteration is not None:
            on_iteration(it, r.vals.copy(), err)
        if err <= eps:
            break
    return r


def connected_components(A, desc=None, sparsify=True):
    """algorithms.py:165-203 -- FastSV with grandparent sparsification."""
    desc = desc or Desc()
    n = A.nrows
    parent = Vec(n, None, np.arange(n, dtype=I64), I64(0))
    mn, gp, gp_prev = parent.copy(), parent.copy(), parent.copy()
    for _ in range(desc.max_niter):
        pp = parent.copy()
        hooked = mxv("MinimumSelectSecond", A, gp, desc=desc)
        mn = ewise_add("Minimum", mn, hooked, desc=desc, identity="Minimum")
        assign_scatter(parent, mn, pp, desc=desc)
        parent = ewise_add("Minimum", parent, mn, desc=desc, identity="Minimum")
        parent = ewise_add("Minimum", parent, pp, desc=desc, identity="Minimum")
        extract_gather(gp, parent, parent, desc=desc)
        changed = ewise_mult("NotEqualTo", gp_prev, gp, desc=desc)
        if int(reduce("Plus", changed)) == 0:
            break
        gp_prev = gp.copy()
        if sparsify:
            desc.complement = not desc.complement
            assign(gp, I64_MAX, mask=changed, desc=desc)
            desc.complement = not desc.complement
    return parent


def degree_sorted_lower(A):
    """algorithms.py:206-218."""
    deg = np.diff(A.rp)
    order = np.argsort(deg, kind="stable")
    pos = np.empty(A.nrows, I64)
    pos[order] = np.arange(A.nrows, dtype=I64)
    r, c, v = A.tuples()
    pr, pc = pos[r], pos[c]
    k = pr > pc
    return mat_from_tuples(pr[k], pc[k], v[k], A.nrows, A.ncols)


def triangle_count_fast(A):
    """algorithms.py:221-240 restated as a merge count: L L^T .* L summed.
    The count is orientation-free, so this walks the degree-ordered upper
    rows (the cheaper orientation) with sorted-list intersections."""
    L = degree_sorted_lower(A)
    U = transpose(L)  # rows hold higher-ranked neighbours
    total = 0
    rp, ci = U.rp, U.ci
    for i in range(U.nrows):
        ri = ci[rp[i]:rp[i + 1]]
        for j in ri:
            total += np.intersect1d(ri, ci[rp[j]:rp[j + 1]], assume_unique=True).size
    return total


# ---------------------------------------------------------------------------
# io  (io.py:71-111, 220-315)
# ---------------------------------------------------------------------------

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def splitmix_stream(seed, start, count):
    """io.py:100-111 -- draw k is mix(seed + (k+1)*gamma), closed form."""
    ks = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + ks * GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def rmat_edges(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, d=0.05, seed=1, chunk=1 << 20):
    """io.py:275-295, chunked so the draw matrix never exceeds chunk x scale."""
    n = 1 << scale
    m = edge_factor * n
    tab = a + b
    tabc = tab + c
    rows = np.empty(m, I64)
    cols = np.empty(m, I64)
    shifts = np.arange(scale - 1, -1, -1, dtype=I64)
    for e0 in range(0, m, chunk):
        k = min(chunk, m - e0)
        x = (splitmix_stream(seed, e0 * scale, k * scale) >> np.uint64(11)) * (1.0 / (1 << 53))
        x = x.reshape(k, scale)
        rb = x >= tab
        cb = ((x >= a) & (x < tab)) | (x >= tabc)
        rows[e0:e0 + k] = (rb.astype(I64) << shifts).sum(axis=1)
        cols[e0:e0 + k] = (cb.astype(I64) << shifts).sum(axis=1)
    return rows, cols, n


def preprocess(src, dst):
    """io.py:220-249 (pattern edges): drop loops, mirror, sort, dedup."""
    k = src != dst
    src, dst = src[k], dst[k]
    s = np.concatenate([src, dst])
    t = np.concatenate([dst, src])
    o = np.lexsort((t, s))
    s, t = s[o], t[o]
    keep = np.r_[True, (s[1:] != s[:-1]) | (t[1:] != t[:-1])] if s.size else np.zeros(0, bool)
    return s[keep], t[keep]


def rmat_csr(scale, **kw):
    """(row_offsets int64, col_indices int64, n) of the preprocessed pattern graph."""
    r, c, n = rmat_edges(scale, **kw)
    s, t = preprocess(r, c)
    rp = np.zeros(n + 1, I64)
    np.add.at(rp, s + 1, 1)
    return np.cumsum(rp).astype(I64), t.astype(I64), n


def upper_weights(rp, ci, seed=1, low=1, high=64):
    """io.py:252-272 restated for a symmetric sorted CSR: the k-th upper entry
    (row-major) gets 1 + mix_k mod 64; its mirror gets the same value."""
    n = rp.size - 1
    rp = np.asarray(rp, dtype=I64)
    ci = np.asarray(ci, dtype=I64)  # int32 columns would overflow rows*n + col from n = 2^16
    rows = np.repeat(np.arange(n, dtype=I64), np.diff(rp))
    up = rows < ci
    k = np.cumsum(up) - 1
    draws = (low + (splitmix_stream(seed, 0, int(up.sum())) % np.uint64(high - low + 1)).astype(I64)).astype(np.float64)
    w = np.empty(ci.size, np.float64)
    w[up] = draws[k[up]]
    # mirror: entry (i,j) with i>j takes the weight of (j,i)
    lo = ~up
    key_up = rows[up] * n + ci[up]
    key_lo = ci[lo] * n + rows[lo]
    w[lo] = draws[np.searchsorted(key_up, key_lo)]
    return w


def mat_from_csr(rp, ci, vals, n):
    m = Mat(n, n, rp, ci, vals)
    return add_csc(m)
