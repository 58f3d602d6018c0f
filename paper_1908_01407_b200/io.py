"""Graph ingestion and synthetic generation (drop-in for the reference's io.py).

The R-MAT stream is generated ON THE GPU, bit-identical to the reference's
counter-based SplitMix64 formulation (io.py:71-111, 275-295): edge e at level
l consumes draw e*scale+l, so every thread computes its edge independently.
``preprocess`` + ``edges_to_matrix`` run as one device sort/dedup
(io.py:220-249, 298-315); ``assign_weights`` reproduces the first-appearance
draw order (io.py:252-272).  Edge lists live on the device; their
``src``/``dst``/``weight`` attributes are host numpy copies on access.

Matrix Market files are host text: they are parsed on the host and uploaded.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .algebra import builtin_monoid
from .containers import INDEX_DTYPE, SparseMatrix, _Orient, cast, empty, full, to_dev, to_host
from .errors import ParseError


class EdgeList:
    """Directed (src, dst) pairs with optional weights (io.py:27-42), on the device.

    ``_csr`` caches the CSR form when the list is known to be sorted and
    duplicate-free (the output of ``preprocess``); ``_symmetric`` records that
    it was mirrored.
    """

    __slots__ = ("_src", "_dst", "n", "_w", "_csr", "_symmetric")

    def __init__(self, src, dst, n, weight=None):
        self._src = to_dev(src, np.int32)
        self._dst = to_dev(dst, np.int32)
        self.n = int(n)
        self._w = None if weight is None else to_dev(weight, np.float64)
        self._csr = None
        self._symmetric = False

    @classmethod
    def _wrap(cls, src_t, dst_t, n, w_t=None, csr=None, symmetric=False):
        e = cls.__new__(cls)
        e._src, e._dst, e.n, e._w = src_t, dst_t, int(n), w_t
        e._csr, e._symmetric = csr, symmetric
        return e

    @property
    def src(self):
        return to_host(self._src, INDEX_DTYPE)

    @property
    def dst(self):
        return to_host(self._dst, INDEX_DTYPE)

    @property
    def weight(self):
        return None if self._w is None else to_host(self._w)

    @property
    def nedges(self) -> int:
        return int(self._src.numel())

    def copy(self) -> "EdgeList":
        return EdgeList._wrap(self._src.clone(), self._dst.clone(), self.n,
                              None if self._w is None else self._w.clone(), self._csr,
                              self._symmetric)


@dataclass(frozen=True)
class RmatParams:
    """Recursive-quadrant generator parameters (io.py:45-68)."""

    scale: int
    edge_factor: int = 16
    a: float = 0.57
    b: float = 0.19
    c: float = 0.19
    d: float = 0.05
    seed: int = 1

    def __post_init__(self):
        total = self.a + self.b + self.c + self.d
        if abs(total - 1.0) > 1e-9:
            raise ValueError(f"quadrant probabilities sum to {total}, expected 1")
        if self.scale < 0 or self.edge_factor <= 0:
            raise ValueError("scale must be >= 0 and edge_factor positive")


_GAMMA = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB
_U64 = (1 << 64) - 1


class SplitMix64:
    """Scalar SplitMix64 (io.py:77-97) -- a host utility for single draws."""

    def __init__(self, seed: int):
        self.state = seed & _U64

    def next_u64(self) -> int:
        self.state = (self.state + _GAMMA) & _U64
        z = self.state
        z = ((z ^ (z >> 30)) * _MIX1) & _U64
        z = ((z ^ (z >> 27)) * _MIX2) & _U64
        return z ^ (z >> 31)

    def next_float(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / (1 << 53))

    def next_int(self, low: int, high: int) -> int:
        return low + self.next_u64() % (high - low + 1)


def generate_rmat(params: RmatParams) -> EdgeList:
    """edge_factor * 2**scale directed R-MAT edges, generated on the GPU (io.py:275-295)."""
    n = 1 << params.scale
    m = params.edge_factor * n
    t_ab = params.a + params.b          # the same double sums as the reference
    t_abc = t_ab + params.c
    src = empty(m, np.int32)
    dst = empty(m, np.int32)
    if m:
        _lib.context().call("gb_rmat_generate", params.scale, m, params.seed & _U64,
                            float(params.a), float(t_ab), float(t_abc), _lib.ptr(src),
                            _lib.ptr(dst))
    return EdgeList._wrap(src, dst, n)


def preprocess(edges: EdgeList, make_undirected=True) -> EdgeList:
    """Drop self loops, mirror, sort by (src, dst), deduplicate (io.py:220-249)."""
    if edges._w is not None:
        return _preprocess_weighted(edges, make_undirected)
    n, m = edges.n, edges.nedges
    off = empty(n + 1, np.int64)
    idx = empty(2 * m if make_undirected else m, np.int32)
    cnt = C.c_int64(0)
    _lib.context().call("gb_edges_to_csr", n, m, _lib.ptr(edges._src), _lib.ptr(edges._dst),
                        1 if make_undirected else 0, _lib.ptr(off), _lib.ptr(idx), C.byref(cnt))
    nnz = int(cnt.value)
    idx = idx[:nnz].clone() if nnz < idx.numel() // 2 else idx[:nnz]
    csr = _Orient(n, n, off, idx, None, 1, np.int64)
    rows = empty(nnz, np.int32)
    if nnz:
        _lib.context().call("gb_csr_row_ids", n, nnz, _lib.ptr(off), _lib.ptr(rows))
    return EdgeList._wrap(rows, idx, n, None, csr, bool(make_undirected))


def _preprocess_weighted(edges, make_undirected):
    """Weighted edges: duplicates keep the minimum weight (io.py:245-247)."""
    m = edges.nedges
    cap = max(2 * m if make_undirected else m, 1)
    src, dst, w = empty(cap, np.int64), empty(cap, np.int64), empty(cap, np.float64)
    c = C.c_int64(0)
    _lib.context().call("gb_edges_clean", m, _lib.ptr(edges._src), _lib.ptr(edges._dst),
                        _lib.ptr(edges._w), 1 if make_undirected else 0, _lib.ptr(src),
                        _lib.ptr(dst), _lib.ptr(w), C.byref(c))
    k = int(c.value)
    A = SparseMatrix.from_tuples(src[:k], dst[:k], w[:k], edges.n, edges.n,
                                 dedup=builtin_monoid("Minimum"), build_csc=False)
    rows = A.row_ids()
    o = A._csr
    wv = o.dense_values()
    out = EdgeList._wrap(rows, o.indices, edges.n, wv, None, bool(make_undirected))
    return out


def assign_weights(edges: EdgeList, low=1, high=64, seed=1) -> EdgeList:
    """One integer weight in [low, high] per undirected pair (io.py:252-272)."""
    if low > high:
        raise ValueError(f"low {low} exceeds high {high}")
    w = empty(edges.nedges, np.float64)
    if edges.nedges:
        _lib.context().call("gb_assign_weights", edges.n, edges.nedges, _lib.ptr(edges._src),
                            _lib.ptr(edges._dst), seed & _U64, int(low), int(high), _lib.ptr(w))
    return EdgeList._wrap(edges._src.clone(), edges._dst.clone(), edges.n, w, edges._csr,
                          edges._symmetric)


def edges_to_matrix(edges: EdgeList, weighted=False, build_csc=True) -> SparseMatrix:
    """Adjacency matrix of a clean edge list (io.py:298-315)."""
    n = edges.n
    if weighted:
        if edges._w is None:
            raise ValueError("edge list carries no weights")
        if edges._csr is not None:
            o = edges._csr
            csr = _Orient(n, n, o.offsets, o.indices, edges._w, None, np.float64)
            iso = None
            m = SparseMatrix._wrap(n, n, csr, None, np.float64)
            if edges._symmetric:
                m._csc, m._sym = csr, True
            elif build_csc:
                m._build_csc()
            return m
        return SparseMatrix.from_tuples(cast(edges._src, np.int64), cast(edges._dst, np.int64),
                                        edges._w, n, n, dedup=builtin_monoid("Minimum"),
                                        build_csc=build_csc)
    if edges._csr is not None:
        o = edges._csr
        csr = _Orient(n, n, o.offsets, o.indices, None, 1, np.int64)
        m = SparseMatrix._wrap(n, n, csr, None, np.int64)
        if edges._symmetric:
            m._csc, m._sym = csr, True
        elif build_csc:
            m._build_csc()
        return m
    ones = full(edges.nedges, 1, np.int64)
    return SparseMatrix.from_tuples(cast(edges._src, np.int64), cast(edges._dst, np.int64), ones,
                                    n, n, dedup=builtin_monoid("Plus"), build_csc=build_csc)


def rmat_matrix(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, d=0.05, seed=1, weighted=False):
    """Convenience: the benchmark graph of cli._load_graph (cli.py:105-121) for R-MAT."""
    e = preprocess(generate_rmat(RmatParams(scale, edge_factor, a, b, c, d, seed)),
                   make_undirected=True)
    if weighted:
        e = assign_weights(e, 1, 64, seed=seed)
    return edges_to_matrix(e, weighted=weighted)


# ---------------------------------------------------------------------------
# Matrix Market (host text; io.py:114-213)
# ---------------------------------------------------------------------------

_FIELDS = ("pattern", "integer", "real")
_SYMMETRIES = ("general", "symmetric")


def read_matrix_market(path) -> EdgeList:
    with open(path, "r", encoding="ascii") as fh:
        lines = fh.read().splitlines()
    if not lines:
        raise ParseError("empty file", line=1)
    banner = lines[0].split()
    if len(banner) != 5 or banner[0] != "%%MatrixMarket" or banner[1] != "matrix":
        raise ParseError(f"bad banner {lines[0]!r}", line=1)
    layout, fld, sym = banner[2], banner[3].lower(), banner[4].lower()
    if layout != "coordinate":
        raise ParseError(f"unsupported layout {layout!r} (need coordinate)", line=1)
    if fld not in _FIELDS:
        raise ParseError(f"unsupported field {fld!r}", line=1)
    if sym not in _SYMMETRIES:
        raise ParseError(f"unsupported symmetry {sym!r}", line=1)
    lineno, body = 1, None
    for lineno, raw in enumerate(lines[1:], start=2):
        text = raw.strip()
        if text and not text.startswith("%"):
            body = text.split()
            break
    if body is None:
        raise ParseError("missing size line", line=lineno)
    try:
        nrows, ncols, nnz = (int(tok) for tok in body)
    except ValueError:
        raise ParseError(f"bad size line {body!r}", line=lineno) from None
    srcs, dsts, ws = [], [], []
    seen = 0
    want = 2 if fld == "pattern" else 3
    for here, raw in enumerate(lines[lineno:], start=lineno + 1):
        text = raw.strip()
        if not text or text.startswith("%"):
            continue
        toks = text.split()
        if len(toks) < want:
            raise ParseError(f"entry has {len(toks)} fields, expected {want}", line=here)
        try:
            i, j = int(toks[0]), int(toks[1])
            wv = 1.0 if fld == "pattern" else float(toks[2])
        except ValueError:
            raise ParseError(f"bad entry {text!r}", line=here) from None
        if not (1 <= i <= nrows and 1 <= j <= ncols):
            raise ParseError(f"entry ({i}, {j}) outside {nrows}x{ncols}", line=here)
        seen += 1
        srcs.append(i - 1)
        dsts.append(j - 1)
        ws.append(wv)
        if sym == "symmetric" and i != j:
            srcs.append(j - 1)
            dsts.append(i - 1)
            ws.append(wv)
    if seen != nnz:
        raise ParseError(f"declared {nnz} entries but found {seen}", line=len(lines))
    n = max(nrows, ncols)
    weight = None if fld == "pattern" else np.asarray(ws, dtype=np.float64)
    return EdgeList(np.asarray(srcs, dtype=np.int64), np.asarray(dsts, dtype=np.int64), n, weight)


def write_matrix_market(path, edges: EdgeList, comment=None):
    fld = "pattern" if edges._w is None else "real"
    src, dst, w = edges.src, edges.dst, edges.weight
    with open(path, "w", encoding="ascii") as fh:
        fh.write(f"%%MatrixMarket matrix coordinate {fld} general\n")
        if comment:
            fh.write(f"%{comment}\n")
        fh.write(f"{edges.n} {edges.n} {edges.nedges}\n")
        if w is None:
            for s, t in zip(src, dst):
                fh.write(f"{s + 1} {t + 1}\n")
        else:
            for s, t, x in zip(src, dst, w):
                fh.write(f"{s + 1} {t + 1} {x:g}\n")


# ---------------------------------------------------------------------------
# Binary CSR cache (an extension): a preprocessed matrix
# saved once and reloaded without re-running generation / preprocessing.
# ---------------------------------------------------------------------------


def save_matrix(path, A: SparseMatrix):
    """Write A's CSR (and whether it is symmetric) to an .npz file."""
    o = A._csr
    vals = None if o.values is None else to_host(o.values)
    np.savez(path, nrows=A.nrows, ncols=A.ncols, row_offsets=to_host(o.offsets),
             col_indices=to_host(o.indices), values=vals if vals is not None else np.empty(0),
             iso=np.asarray(o.iso if o.iso is not None else 0), has_values=vals is not None,
             dtype=str(A.dtype), symmetric=bool(A.is_symmetric()) if A.nrows == A.ncols else False)


def load_matrix(path, build_csc=True) -> SparseMatrix:
    """Read a matrix written by save_matrix onto the current device."""
    z = np.load(path, allow_pickle=False)
    nrows, ncols = int(z["nrows"]), int(z["ncols"])
    dt = np.dtype(str(z["dtype"]))
    off, idx = z["row_offsets"], z["col_indices"]
    vals = z["values"] if bool(z["has_values"]) else np.full(idx.size, z["iso"].item(), dtype=dt)
    sym = bool(z["symmetric"])
    return SparseMatrix.from_csr(nrows, ncols, off, idx, vals.astype(dt, copy=False),
                                 build_csc=build_csc, symmetric=True if sym else None)
