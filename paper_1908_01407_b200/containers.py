"""Device-resident Matrix / Vector containers, the Descriptor and Counters.

Drop-in for the reference's containers.py (containers.py:29-464).  The public
surface -- constructors, accessors, conversions, the attribute names tests
read -- is the same; the storage is not:

* ``SparseMatrix`` keeps CSR and (optionally) CSC on the GPU as int64 offsets
  + int32 indices (+ values).  Pattern matrices whose values are all equal are
  stored structure-only ("iso"): no value array at all.  A
  square matrix whose CSC equals its CSR aliases the two orientations
  (symmetric graphs, the common case) -- half the memory, and
  ``_require_symmetric`` becomes O(1).
* ``Vector`` is dense (values[n] + ``zero``) or sparse (sorted int32 indices +
  values) on the GPU; which form an operation produces follows the reference
  (kernels.py) exactly, so ``is_sparse`` and the canonical tuples agree.
* The array attributes the reference exposes (``values``, ``indices``,
  ``row_offsets``, ``col_indices``, ...) are HOST numpy copies made on access
  (the paper's canonical-GPU-copy rule): reading them is a
  device->host transfer, writing them uploads.

Values are int64 or float64 on the device (narrower numpy dtypes are widened
on upload: bool/int -> int64, float32 -> float64).
"""

from __future__ import annotations

import ctypes as C
import enum
import itertools
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .algebra import Monoid, builtin_monoid, fold_op_id
from .errors import FormatError, ShapeError

INDEX_DTYPE = np.int64


class Direction(enum.Enum):
    AUTO = "auto"
    FORCE_PUSH = "force-push"
    FORCE_PULL = "force-pull"


class MaskMode(enum.Enum):
    NORMAL = "normal"
    COMPLEMENT = "complement"


class Partition(enum.Enum):
    # GPU load balancing of pull kernels: merge-path (edge-balanced) vs row split
    NONZERO_SPLIT = "nonzero"
    ROW_SPLIT = "row"


@dataclass
class Counters:
    """Work tallies (containers.py:49-71); filled by the unfused kernels."""

    matrix_entries_read: int = 0
    semiring_multiplies: int = 0
    semiring_adds: int = 0

    def reset(self):
        self.matrix_entries_read = 0
        self.semiring_multiplies = 0
        self.semiring_adds = 0

    def merge(self, other: "Counters"):
        self.matrix_entries_read += other.matrix_entries_read
        self.semiring_multiplies += other.semiring_multiplies
        self.semiring_adds += other.semiring_adds


class DecisionLog(list):
    """The direction log (a list of DirectionDecision, kernels.py:303-304).

    An asynchronous device call (``bfs``) appends a pending resolver instead
    of its decisions; any read or further append first waits for the pending
    calls in order and materialises their decisions, so the log always reads
    exactly like the reference's eagerly filled list.
    """

    __slots__ = ("_pending",)

    def __init__(self, *args):
        super().__init__(*args)
        self._pending = []

    def _defer(self, resolve):
        self._pending.append(resolve)

    def _flush(self):
        if self._pending:
            pending, self._pending = self._pending, []
            for resolve in pending:
                list.extend(self, resolve())

    def __reduce_ex__(self, protocol):
        self._flush()
        return (DecisionLog, (list(self),))


def _flushing(name):
    base = getattr(list, name)

    def method(self, *args, **kwargs):
        self._flush()
        return base(self, *args, **kwargs)

    method.__name__ = name
    return method


for _name in ("__len__", "__iter__", "__getitem__", "__setitem__", "__delitem__", "__contains__",
              "__reversed__", "__eq__", "__ne__", "__lt__", "__le__", "__gt__", "__ge__",
              "__repr__", "__add__", "__iadd__", "__mul__", "__rmul__", "__imul__", "append",
              "extend", "insert", "pop", "remove", "clear", "index", "count", "copy", "sort",
              "reverse"):
    setattr(DecisionLog, _name, _flushing(_name))
DecisionLog.__hash__ = None


@dataclass
class Descriptor:
    """Per-call modifiers (containers.py:74-113).

    Extensions (not in the reference): ``fused`` -- algorithms run their
    fused device loops (default); ``False`` replays the reference's exact
    operator composition so ``counters`` carry the reference's tallies.
    ``count_work`` -- the fused algorithms also fill ``counters`` with the
    reference's exact tallies (BFS: recomputed on the device from the levels
    and the direction log, gb_bfs_counters; PageRank: from the direction log;
    SSSP / CC / TC: by running the operator composition), at extra cost.
    ``num_workers`` is accepted and ignored (the GPU grid replaces the
    thread pool).
    """

    mask_mode: MaskMode = MaskMode.NORMAL
    transpose_inp0: bool = False
    transpose_inp1: bool = False
    direction: Direction = Direction.AUTO
    switch_ratio: float = 0.1
    max_niter: int = 10_000
    num_workers: int = 1
    partition: Partition = Partition.NONZERO_SPLIT
    early_exit: bool = False
    counters: Counters = field(default_factory=Counters)
    direction_log: list = field(default_factory=DecisionLog)
    fused: bool = True
    count_work: bool = False

    _TOGGLES = {"mask": "mask_mode", "inp0": "transpose_inp0", "inp1": "transpose_inp1"}

    def toggle(self, which: str):
        if which == "mask":
            self.mask_mode = (
                MaskMode.COMPLEMENT if self.mask_mode is MaskMode.NORMAL else MaskMode.NORMAL
            )
        elif which in ("inp0", "inp1"):
            attr = self._TOGGLES[which]
            setattr(self, attr, not getattr(self, attr))
        else:
            raise KeyError(f"unknown descriptor toggle {which!r}")
        return self


# ---------------------------------------------------------------------------
# dtype / tensor helpers
# ---------------------------------------------------------------------------


def device_dtype(dt) -> np.dtype:
    """The device storage dtype for a numpy dtype: int64 or float64."""
    dt = np.dtype(dt)
    if dt.kind in "biu":
        return np.dtype(np.int64)
    if dt.kind == "f":
        return np.dtype(np.float64)
    if dt == object:
        return np.dtype(np.float64)
    raise NotImplementedError(f"dtype {dt} is not supported on the device")


_TORCH = {np.dtype(np.int64): torch.int64, np.dtype(np.float64): torch.float64,
          np.dtype(np.int32): torch.int32}


def _device():
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def to_dev(a, np_dtype) -> torch.Tensor:
    """Upload array-like (numpy, list, tensor) as a contiguous CUDA tensor."""
    np_dtype = np.dtype(np_dtype)
    if isinstance(a, torch.Tensor):
        return a.to(device=_device(), dtype=_TORCH[np_dtype]).contiguous()
    arr = np.ascontiguousarray(np.asarray(a).astype(np_dtype, copy=False)).ravel()
    return torch.from_numpy(arr).to(_device())


def to_host(t: torch.Tensor, np_dtype=None) -> np.ndarray:
    """Device -> host copy.  Large arrays go through a pinned staging tensor
    (torch's caching host allocator) so the copy runs at full PCIe/C2C speed;
    the returned numpy array keeps that pinned buffer alive."""
    t = t.detach()
    if t.is_cuda and t.numel() * t.element_size() >= (1 << 20):
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        torch.cuda.current_stream(t.device).synchronize()
        out = h.numpy()
    else:
        out = t.cpu().numpy()
    return out if np_dtype is None else out.astype(np_dtype, copy=False)


def empty(n, np_dtype) -> torch.Tensor:
    return torch.empty(int(n), dtype=_TORCH[np.dtype(np_dtype)], device=_device())


def full(n, value, np_dtype) -> torch.Tensor:
    return torch.full((int(n),), value, dtype=_TORCH[np.dtype(np_dtype)], device=_device())


_CODE_OF_TORCH = {torch.int64: 0, torch.float64: 1, torch.int32: 2}   # GB_I64 / GB_F64 / GB_I32


def cast(t: torch.Tensor, np_dtype) -> torch.Tensor:
    """numpy astype on a device array (gb_cast); t itself when already of dtype."""
    want = _TORCH[np.dtype(np_dtype)]
    if t.dtype == want:
        return t
    out = torch.empty(t.numel(), dtype=want, device=t.device)
    if t.numel():
        _lib.context().call("gb_cast", int(t.numel()), _CODE_OF_TORCH[t.dtype], _lib.ptr(t),
                            _CODE_OF_TORCH[want], _lib.ptr(out))
    return out


def iota(n, np_dtype=np.int32) -> torch.Tensor:
    """0, 1, ..., n-1 on the device (gb_iota)."""
    out = empty(n, np_dtype)
    if n:
        _lib.context().call("gb_iota", _CODE_OF_TORCH[out.dtype], int(n), _lib.ptr(out))
    return out


def gather32(src: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    """src[idx] with int32 device indices (gb_gather_i32)."""
    k = int(idx.numel())
    out = torch.empty(k, dtype=src.dtype, device=src.device)
    if k:
        _lib.context().call("gb_gather_i32", _CODE_OF_TORCH[src.dtype], k,
                            _lib.ptr(cast(idx, np.int32)), _lib.ptr(src), _lib.ptr(out))
    return out


def _zero_buf(zero, dt):
    return _lib.scalar_buf(zero, dt)


# ---------------------------------------------------------------------------
# Vector
# ---------------------------------------------------------------------------


class Vector:
    """A length-n vector, sparse (sorted indices + values) or dense (containers.py:116-257)."""

    __slots__ = ("size", "_idx", "_vals", "_dt", "zero", "__weakref__")

    def __init__(self, size, indices, values, zero):
        self.size = int(size)
        vals_np_dtype = _dtype_of(values)
        self._dt = device_dtype(vals_np_dtype)
        self._vals = to_dev(values, self._dt)
        self._idx = None if indices is None else to_dev(indices, np.int32)
        self.zero = self._dt.type(zero)

    @classmethod
    def _wrap(cls, size, idx_t, vals_t, zero, dt):
        v = cls.__new__(cls)
        v.size = int(size)
        v._idx = idx_t
        v._vals = vals_t
        v._dt = np.dtype(dt)
        v.zero = v._dt.type(zero)
        return v

    # -- construction -------------------------------------------------

    @classmethod
    def from_entries(cls, indices, values, size, dtype=None) -> "Vector":
        """Sparse vector from (index, value) pairs (containers.py:135-147)."""
        idx = np.asarray(indices, dtype=INDEX_DTYPE).ravel()
        vals = np.asarray(values, dtype=dtype).ravel()
        if idx.shape != vals.shape:
            raise ShapeError(f"{idx.size} indices vs {vals.size} values")
        dt = device_dtype(vals.dtype)
        if idx.size == 0:
            return cls._wrap(size, empty(0, np.int32), empty(0, dt), 0, dt)
        # sort + validate on the device through the CSR builder (one row)
        rows = full(idx.size, 0, np.int64)
        A = SparseMatrix.from_tuples(rows, idx, vals, 1, int(size), build_csc=False,
                                     _check_unique=True)
        o = A._csr
        vals_t = o.values if o.values is not None else full(o.nnz, o.iso, dt)
        return cls._wrap(size, o.indices, vals_t, 0, dt)

    @classmethod
    def filled(cls, size, value, dtype=None) -> "Vector":
        dt = device_dtype(np.asarray(value, dtype=dtype).dtype)
        return cls._wrap(size, None, full(size, dt.type(value).item(), dt), 0, dt)

    @classmethod
    def empty(cls, size, dtype=np.int64) -> "Vector":
        dt = device_dtype(dtype)
        return cls._wrap(size, empty(0, np.int32), empty(0, dt), 0, dt)

    @classmethod
    def dense_of(cls, values, zero) -> "Vector":
        if isinstance(values, torch.Tensor):
            dt = device_dtype(np.dtype(str(values.dtype).replace("torch.", "")))
            t = values.to(device=_device(), dtype=_TORCH[dt]).contiguous()
            return cls._wrap(t.numel(), None, t, zero, dt)
        values = np.asarray(values)
        dt = device_dtype(values.dtype)
        return cls._wrap(values.size, None, to_dev(values, dt), zero, dt)

    # -- accessors ----------------------------------------------------

    @property
    def is_sparse(self):
        return self._idx is not None

    @property
    def dtype(self):
        return self._dt

    @property
    def indices(self):
        return None if self._idx is None else to_host(self._idx, INDEX_DTYPE)

    @indices.setter
    def indices(self, value):
        self._idx = None if value is None else to_dev(value, np.int32)

    @property
    def values(self):
        return to_host(self._vals)

    @values.setter
    def values(self, value):
        self._vals = to_dev(value, self._dt)

    @property
    def nvals(self) -> int:
        return self.nvals_for(self.zero)

    def nvals_for(self, zero) -> int:
        if self.is_sparse:
            return int(self._idx.numel())
        return count_ne(self._vals, self._dt, zero)

    def set_element(self, i, value):
        if not 0 <= i < self.size:
            raise IndexError(f"index {i} out of range for size {self.size}")
        if not self.is_sparse:
            self._vals[i] = self._dt.type(value).item()
            return
        idx = self.indices
        pos = int(np.searchsorted(idx, i))
        if pos < idx.size and idx[pos] == i:
            self._vals[pos] = self._dt.type(value).item()
        else:
            vals = self.values
            self._idx = to_dev(np.insert(idx, pos, i), np.int32)
            self._vals = to_dev(np.insert(vals, pos, value), self._dt)

    def extract_element(self, i):
        if not 0 <= i < self.size:
            raise IndexError(f"index {i} out of range for size {self.size}")
        if self.is_sparse:
            idx = self.indices
            pos = int(np.searchsorted(idx, i))
            if pos < idx.size and idx[pos] == i:
                return self._dt.type(self._vals[pos].item())
            return None
        v = self._dt.type(self._vals[i].item())
        return None if v == self.zero else v

    def extract_tuples(self):
        """Stored (indices, values) in ascending index order (host arrays)."""
        if self.is_sparse:
            return self.indices, self.values
        idx_t, vals_t = compact(self._vals, None, self._dt, self.zero, self.size)
        return to_host(idx_t, INDEX_DTYPE), to_host(vals_t)

    def dup(self) -> "Vector":
        return Vector._wrap(self.size, None if self._idx is None else self._idx.clone(),
                            self._vals.clone(), self.zero, self._dt)

    def clear(self):
        self._idx = empty(0, np.int32)
        self._vals = empty(0, self._dt)

    # -- format conversion --------------------------------------------

    def to_dense(self, zero=None) -> "Vector":
        zero = self.zero if zero is None else zero
        if not self.is_sparse:
            out = self.dup()
            out.zero = out._dt.type(zero)
            return out
        t = scatter_dense(self._idx, self._vals, self._dt, zero, self.size)
        return Vector._wrap(self.size, None, t, zero, self._dt)

    def to_sparse(self, zero=None) -> "Vector":
        zero = self.zero if zero is None else zero
        idx_t, vals_t = compact(self._vals, self._idx, self._dt, zero, self.size)
        return Vector._wrap(self.size, idx_t, vals_t, zero, self._dt)

    def __repr__(self):
        kind = "sparse" if self.is_sparse else "dense"
        return f"<Vector {kind} size={self.size} nvals={self.nvals}>"


def _dtype_of(values):
    if isinstance(values, torch.Tensor):
        return np.dtype(str(values.dtype).replace("torch.", ""))
    return np.asarray(values).dtype


def vector_build(indices, values, size, dtype=None) -> Vector:
    return Vector.from_entries(indices, values, size, dtype=dtype)


def vector_fill(size, value, dtype=None) -> Vector:
    return Vector.filled(size, value, dtype=dtype)


def vector_convert(v: Vector, target: str, zero) -> Vector:
    if target == "dense":
        return v.to_dense(zero)
    if target == "sparse":
        return v.to_sparse(zero)
    raise KeyError(f"unknown vector format {target!r}")


# -- device vector primitives used above and by kernels.py --------------------


def count_ne(vals_t, dt, zero) -> int:
    n = int(vals_t.numel())
    if n == 0:
        return 0
    ctx = _lib.context()
    out = C.c_int64(0)
    ctx.call("gb_count_ne", n, _lib.ptr(vals_t), _lib.dtype_code(dt), _zero_buf(zero, dt),
             C.byref(out))
    return int(out.value)


def compact(vals_t, idx_t, dt, zero, size):
    """Keep entries != zero -> (int32 idx tensor, values tensor)."""
    k = int(vals_t.numel())
    out_idx = empty(k, np.int32)
    out_vals = empty(k, dt)
    if k == 0:
        return out_idx, out_vals
    ctx = _lib.context()
    cnt = C.c_int64(0)
    ctx.call("gb_compact", int(size), k if idx_t is not None else -1, _lib.ptr(idx_t), _lib.ptr(vals_t), _lib.dtype_code(dt),
             _zero_buf(zero, dt), _lib.ptr(out_idx), _lib.ptr(out_vals), C.byref(cnt))
    c = int(cnt.value)
    return out_idx[:c], out_vals[:c]


def scatter_dense(idx_t, vals_t, dt, zero, size):
    out = empty(size, dt)
    if size == 0:
        return out
    ctx = _lib.context()
    ctx.call("gb_scatter_dense", int(size), int(idx_t.numel()), _lib.ptr(idx_t), _lib.ptr(vals_t),
             _lib.dtype_code(dt), _zero_buf(zero, dt), _lib.ptr(out))
    return out


# ---------------------------------------------------------------------------
# SparseMatrix
# ---------------------------------------------------------------------------


_ORIENT_GEN = itertools.count(1)


class _Orient:
    """One orientation on the device: rows of A (CSR) or of A^T (CSC)."""

    __slots__ = ("nrows", "ncols", "offsets", "indices", "values", "iso", "dt", "_nonempty",
                 "_plan", "_bins", "_stripes", "_ordered", "_order", "_mv_ordered", "_struct", "gen",
                 "_min_cache",
                 "__weakref__")

    def __init__(self, nrows, ncols, offsets, indices, values, iso, dt):
        self.nrows, self.ncols = int(nrows), int(ncols)
        self.offsets, self.indices, self.values = offsets, indices, values
        self.iso = iso  # python scalar when values is None
        self.dt = np.dtype(dt)
        self._nonempty = None
        self._plan = None
        self._bins = None
        self._stripes = None
        self._struct = None      # cached csr_struct() of the stored dtype (immutable)
        self._ordered = None
        self._order = None       # new -> original id of the traversal layout
        self._mv_ordered = {}    # transpose -> ordered masked-pull view (SparseMatrix.ordered_pull)
        # contents identity for the native per-matrix caches (gb_csr.gen);
        # orientations are immutable, so one id per object
        self.gen = next(_ORIENT_GEN)

    @property
    def nnz(self):
        return int(self.indices.numel())

    def bin_plan(self):
        """Row bins of this orientation (gb_bin_plan_counts / _fill): short
        rows, medium rows and the 512-entry tiles of long rows, built once.
        Returns (gb_bin_plan, keepalive)."""
        if self._bins is None:
            s, _keep = self.csr_struct()
            ctx = _lib.context()
            cnt = (C.c_int64 * 3)()
            ctx.call("gb_bin_plan_counts", C.byref(s), cnt)
            ns, nm, nl = int(cnt[0]), int(cnt[1]), int(cnt[2])
            bufs = (empty(max(ns, 1), np.int32), empty(max(nm, 1), np.int32),
                    empty(max(nl, 1), np.int32), empty(max(nl, 1), np.int64),
                    empty(max(nl, 1), np.int64))
            p = _lib.gb_bin_plan()
            p.n_short, p.n_mid, p.n_long_tiles = ns, nm, nl
            (p.short_rows, p.mid_rows, p.tile_row, p.tile_beg,
             p.tile_end) = (b.data_ptr() for b in bufs)
            ctx.call("gb_bin_plan_fill", C.byref(s), C.byref(p))
            self._bins = (p, bufs)
        return self._bins

    def stripes(self, count):
        """Column stripes of this (structure-only) orientation for the striped
        pull (gb_mxv_pull_striped): `count` CSRs over the same rows, stripe k
        holding the entries with columns in [k*w, (k+1)*w), w =
        ceil(ncols/count) rounded up to 1024, each with its row bins.  Built
        once per count.  Returns (gb_csr array, gb_bin_plan array, keepalive)."""
        if self._stripes is not None and self._stripes[0] == count:
            return self._stripes[1]
        if self.values is not None:
            raise NotImplementedError("column stripes take a structure-only matrix")
        n, nc = self.nrows, self.ncols
        w = -(-nc // count)
        w = -(-w // 1024) * 1024
        ctx = _lib.context()
        s, _keep = self.csr_struct()
        subs = []
        for k in range(count):
            lo, hi = min(k * w, nc), min((k + 1) * w, nc)
            off = empty(n + 1, np.int64)
            cnt = C.c_int64(0)
            ctx.call("gb_csr_column_block", C.byref(s), lo, hi, _lib.ptr(off), None, C.byref(cnt))
            idx = empty(max(int(cnt.value), 1), np.int32)
            ctx.call("gb_csr_column_block", C.byref(s), lo, hi, _lib.ptr(off), _lib.ptr(idx),
                     C.byref(cnt))
            subs.append(_Orient(n, nc, off, idx[:int(cnt.value)], None, self.iso, self.dt))
        csrs = (_lib.gb_csr * count)()
        plans = (_lib.gb_bin_plan * count)()
        keep = []
        for k, sub in enumerate(subs):
            st, kk = sub.csr_struct()
            csrs[k] = st
            plan, pk = sub.bin_plan()
            plans[k] = plan
            keep += [kk, pk]
        self._stripes = (count, (csrs, plans, (subs, keep)))
        return self._stripes[1]

    def row_plan(self):
        """Edge-balanced work plan of this orientation (gb_row_plan_build):
        the non-empty rows and the first plan row of every 512-entry tile,
        built once.  Returns (gb_row_plan, keepalive)."""
        if self._plan is None:
            n = self.nrows
            nz_rows = empty(max(n, 1), np.int32)
            nz_off = empty(n + 1, np.int64)
            tile_first = empty(self.nnz // 512 + 2, np.int32)
            R = C.c_int64(0)
            s, _keep = self.csr_struct()
            _lib.context().call("gb_row_plan_build", C.byref(s), _lib.ptr(nz_rows),
                                _lib.ptr(nz_off), _lib.ptr(tile_first), C.byref(R))
            p = _lib.gb_row_plan()
            p.nrows_nz = R.value
            p.nz_rows, p.nz_off, p.tile_first = (nz_rows.data_ptr(), nz_off.data_ptr(),
                                                 tile_first.data_ptr())
            self._plan = (p, (nz_rows, nz_off, tile_first))
        return self._plan

    def csr_struct(self, as_dtype=None):
        """(gb_csr, keepalive) -- values converted to ``as_dtype`` when given.

        Keep the second element alive for as long as the struct is used: it
        owns the converted value array the struct points at."""
        if (as_dtype is None or np.dtype(as_dtype) == self.dt) and self._struct is not None:
            return self._struct
        s = _lib.gb_csr()
        s.nrows, s.ncols, s.nnz = self.nrows, self.ncols, self.nnz
        s.offsets = self.offsets.data_ptr()
        s.indices = self.indices.data_ptr() if self.nnz else 0
        dt = self.dt if as_dtype is None else np.dtype(as_dtype)
        keep = None
        if self.values is None:
            s.values = None
            iso = 0 if self.iso is None else self.iso
            s.iso_f64 = float(iso)
            # the int view of a float iso value is only read for int compute dtypes
            s.iso_i64 = int(iso) if np.isfinite(float(iso)) and abs(float(iso)) < 2**63 else 0
        else:
            keep = self.values_as(dt)
            s.values = keep.data_ptr() if self.nnz else 0
        s.dtype = _lib.dtype_code(dt)
        s.gen = self.gen
        if dt == self.dt:
            self._struct = (s, keep)
        return s, keep

    def values_as(self, dt):
        dt = np.dtype(dt)
        if self.values is None:
            return None
        if dt == self.dt:
            return self.values
        return cast(self.values, dt)

    def nonempty(self):
        if self._nonempty is None:
            W = (self.nrows + 31) // 32
            t = torch.empty(max(W, 1), dtype=torch.int32, device=self.offsets.device)
            _lib.context().call("gb_nonempty_rows", self.nrows, _lib.ptr(self.offsets), _lib.ptr(t))
            self._nonempty = t
        return self._nonempty

    def dense_values(self):
        if self.values is not None:
            return self.values
        return full(self.nnz, self.iso, self.dt)


def _iso_of(vals_t, dt):
    """Python scalar when every value is equal (structure-only storage)."""
    n = int(vals_t.numel())
    if n == 0:
        return None
    ctx = _lib.context()
    flag = C.c_int32(0)
    ctx.call("gb_values_iso", n, _lib.ptr(vals_t), _lib.dtype_code(dt), C.byref(flag))
    if flag.value:
        return dt.type(vals_t[0].item()).item()
    return None


class SparseMatrix:
    """An M-by-N sparse matrix on the GPU: CSR + optional CSC (containers.py:276-451)."""

    __slots__ = ("nrows", "ncols", "_csr", "_csc", "_dt", "_sym", "__weakref__")

    def __init__(self, nrows, ncols, row_offsets, col_indices, csr_values,
                 col_offsets=None, row_indices=None, csc_values=None):
        self.nrows, self.ncols = int(nrows), int(ncols)
        dt = device_dtype(_dtype_of(csr_values))
        self._dt = dt
        self._csr = _make_orient(self.nrows, self.ncols, row_offsets, col_indices, csr_values, dt)
        self._csc = None
        self._sym = None
        if col_offsets is not None:
            self._csc = _make_orient(self.ncols, self.nrows, col_offsets, row_indices,
                                     csc_values, dt)

    @classmethod
    def _wrap(cls, nrows, ncols, csr, csc, dt, sym=None):
        m = cls.__new__(cls)
        m.nrows, m.ncols = int(nrows), int(ncols)
        m._csr, m._csc, m._dt, m._sym = csr, csc, np.dtype(dt), sym
        return m

    # -- construction -------------------------------------------------

    @classmethod
    def from_tuples(cls, rows, cols, values, nrows, ncols, dedup: Optional[Monoid] = None,
                    build_csc=True, dtype=None, _check_unique=False) -> "SparseMatrix":
        """Build from (row, col, value) triples, folding duplicates (containers.py:307-345)."""
        if dedup is None:
            dedup = builtin_monoid("Plus")
        rows_t = to_dev(rows, np.int64) if not isinstance(rows, torch.Tensor) else rows.to(
            device=_device(), dtype=torch.int64).contiguous()
        cols_t = to_dev(cols, np.int64)
        if isinstance(values, torch.Tensor):
            vdt = device_dtype(_dtype_of(values)) if dtype is None else device_dtype(dtype)
            vals_t = values.to(device=_device(), dtype=_TORCH[vdt]).contiguous()
        else:
            vals = np.asarray(values, dtype=dtype).ravel()
            if vals.dtype == object:
                vals = vals.astype(np.float64)
            vdt = device_dtype(vals.dtype)
            vals_t = to_dev(vals, vdt)
        n = int(rows_t.numel())
        if not (n == int(cols_t.numel()) == int(vals_t.numel())):
            raise ShapeError("rows, cols and values must have equal length")
        nrows, ncols = int(nrows), int(ncols)
        off = empty(nrows + 1, np.int64)
        idx = empty(n, np.int32)
        outv = empty(n, vdt)
        cnt = C.c_int64(0)
        op = fold_op_id(dedup.op)
        _lib.context().call("gb_build_csr", nrows, ncols, n, _lib.ptr(rows_t), _lib.ptr(cols_t),
                            _lib.ptr(vals_t), _lib.dtype_code(vdt), op, _lib.ptr(off),
                            _lib.ptr(idx), _lib.ptr(outv), C.byref(cnt))
        nnz = int(cnt.value)
        if _check_unique and nnz != n:
            raise ValueError("duplicate index in vector build")
        idx, outv = idx[:nnz], outv[:nnz]
        iso = _iso_of(outv, vdt)
        csr = _Orient(nrows, ncols, off, idx, None if iso is not None else outv, iso, vdt)
        m = cls._wrap(nrows, ncols, csr, None, vdt)
        if build_csc:
            m._build_csc()
        return m

    @classmethod
    def from_csr(cls, nrows, ncols, row_offsets, col_indices, values, build_csc=True,
                 symmetric=None):
        """Wrap an existing CSR (containers.py:347-355).  ``symmetric=True``
        (an extension) promises A == A^T and skips the transpose build."""
        vdt = device_dtype(_dtype_of(values))
        off = to_dev(row_offsets, np.int64)
        idx = to_dev(col_indices, np.int32)
        vals_t = to_dev(values, vdt) if not isinstance(values, torch.Tensor) else values.to(
            device=_device(), dtype=_TORCH[vdt]).contiguous()
        iso = _iso_of(vals_t, vdt)
        csr = _Orient(nrows, ncols, off, idx, None if iso is not None else vals_t, iso, vdt)
        m = cls._wrap(nrows, ncols, csr, None, vdt)
        if symmetric:
            m._csc, m._sym = csr, True
        elif build_csc:
            m._build_csc()
        return m

    def _build_csc(self):
        o = self._csr
        off = empty(self.ncols + 1, np.int64)
        idx = empty(o.nnz, np.int32)
        vals = None if o.values is None else empty(o.nnz, self._dt)
        s, _k = o.csr_struct()
        _lib.context().call("gb_transpose_csr", C.byref(s), _lib.ptr(off), _lib.ptr(idx),
                            _lib.ptr(vals))
        csc = _Orient(self.ncols, self.nrows, off, idx, vals, o.iso, self._dt)
        self._csc = csc
        self._sym = None
        if self.nrows == self.ncols:
            eq = C.c_int32(0)
            (a, _ka), (b, _kb) = o.csr_struct(), csc.csr_struct()
            _lib.context().call("gb_csr_equal", C.byref(a), C.byref(b), C.byref(eq))
            self._sym = bool(eq.value)
            if self._sym:
                self._csc = self._csr  # alias: one copy of the structure
        else:
            self._sym = False

    # -- accessors ----------------------------------------------------

    @property
    def nnz(self) -> int:
        return self._csr.nnz

    @property
    def nvals(self) -> int:
        return self.nnz

    @property
    def has_csc(self) -> bool:
        return self._csc is not None

    @property
    def dtype(self):
        return self._dt

    @property
    def is_iso(self):
        return self._csr.values is None

    @property
    def row_offsets(self):
        return to_host(self._csr.offsets)

    @property
    def col_indices(self):
        return to_host(self._csr.indices, INDEX_DTYPE)

    @property
    def csr_values(self):
        return to_host(self._csr.dense_values())

    @property
    def col_offsets(self):
        return None if self._csc is None else to_host(self._csc.offsets)

    @property
    def row_indices(self):
        return None if self._csc is None else to_host(self._csc.indices, INDEX_DTYPE)

    @property
    def csc_values(self):
        return None if self._csc is None else to_host(self._csc.dense_values())

    def orient(self, transpose=False) -> _Orient:
        """Device orientation whose rows are rows of A (False) or of A^T (True)."""
        if not transpose:
            return self._csr
        self.require_csc()
        return self._csc

    def row_view(self, transpose=False):
        o = self.orient(transpose)
        return to_host(o.offsets), to_host(o.indices, INDEX_DTYPE), to_host(o.dense_values()), o.nrows

    def col_view(self, transpose=False):
        o = self.orient(not transpose)
        return to_host(o.offsets), to_host(o.indices, INDEX_DTYPE), to_host(o.dense_values()), o.nrows

    def require_csc(self):
        if not self.has_csc:
            raise FormatError(
                "column-oriented storage missing; build the matrix with build_csc=True")

    def is_symmetric(self) -> bool:
        if self._sym is None:
            if self.nrows != self.ncols:
                self._sym = False
            else:
                if self._csc is None:
                    self._build_csc()
                    return bool(self._sym)
                eq = C.c_int32(0)
                (a, _ka), (b, _kb) = self._csr.csr_struct(), self._csc.csr_struct()
                _lib.context().call("gb_csr_equal", C.byref(a), C.byref(b), C.byref(eq))
                self._sym = bool(eq.value)
        return bool(self._sym)

    def traversal(self):
        """Degree-ordered relabelling used by the traversals, built
        once per matrix: vertices renumbered by descending in-degree (ties by
        id; gb_degree_order), both orientations relabelled with sorted rows
        (gb_csr_relabel_t).  Returns (push, pull, rank) -- push walks rows of
        P A P^T, pull rows of P A^T P^T, rank[i] = new id of vertex i -- or
        None when the matrix is not square or has no column orientation."""
        o, csc = self._csr, self._csc
        if csc is None or self.nrows != self.ncols:
            return None
        c = o._ordered
        if c is not None and c[0] is csc:
            return c[1]
        n = self.nrows
        ctx = _lib.context()
        order = empty(max(n, 1), np.int32)
        rank = empty(max(n, 1), np.int32)
        ctx.call("gb_degree_order", n, _lib.ptr(csc.offsets), _lib.ptr(order), _lib.ptr(rank))

        def relabel_t(src):  # P src^T P^T
            off = empty(n + 1, np.int64)
            idx = empty(src.nnz, np.int32)
            vals = None if src.values is None else empty(src.nnz, src.dt)
            st, _k = src.csr_struct()
            ctx.call("gb_csr_relabel_t", C.byref(st), _lib.ptr(order), _lib.ptr(rank),
                     _lib.ptr(off), _lib.ptr(idx), _lib.ptr(vals))
            return _Orient(n, n, off, idx, vals, src.iso, src.dt)

        if csc is o:
            push = pull = relabel_t(o)
        else:
            pull = relabel_t(o)    # rows of P A^T P^T: in-edges
            push = relabel_t(csc)  # rows of P A P^T: out-edges
        o._ordered = (csc, (push, pull, rank))
        o._order = order
        o._mv_ordered = {}
        return o._ordered[1]

    def ordered_pull(self, transpose):
        """The masked pull SpMV's view of the degree-ordered layout
        (gb_mxv_pull_ordered): the relabelled orientation whose rows the pull
        walks (P A P^T, or P A^T P^T when transposed), its row plan with the
        non-empty rows named by their ORIGINAL ids, the new -> original
        order and the column reach.  Built once per matrix and orientation;
        None when the matrix has no traversal layout."""
        t = self.traversal()
        if t is None:
            return None
        o = self._csr
        v = o._mv_ordered.get(bool(transpose))
        if v is not None:
            return v
        push, pull, _rank = t
        ov = pull if transpose else push
        plan, keep = ov.row_plan()
        ctx = _lib.context()
        rows_old = empty(max(int(plan.nrows_nz), 1), np.int32)
        ctx.call("gb_row_plan_remap", int(plan.nrows_nz), C.c_void_p(plan.nz_rows),
                 _lib.ptr(o._order), _lib.ptr(rows_old))
        p = _lib.gb_row_plan()
        p.nrows_nz = plan.nrows_nz
        p.nz_rows, p.nz_off, p.tile_first = rows_old.data_ptr(), plan.nz_off, plan.tile_first
        mx = C.c_int64(0)
        ctx.call("gb_index_max", ov.nnz, _lib.ptr(ov.indices), C.byref(mx))
        v = (ov, p, (rows_old, keep), o._order, int(mx.value) + 1)
        o._mv_ordered[bool(transpose)] = v
        return v

    def _rank64(self):
        """int64 copy of the traversal rank (gather targets), cached with it."""
        o = self._csr
        c = o._ordered
        if c is None or len(c) < 3:
            rank = self.traversal()[2]
            c = o._ordered
        if len(c) < 3:
            o._ordered = (c[0], c[1], cast(c[1][2], np.int64))
        return o._ordered[2]

    def row_ids(self):
        o = self._csr
        out = empty(o.nnz, np.int32)
        if o.nnz:
            _lib.context().call("gb_csr_row_ids", o.nrows, o.nnz, _lib.ptr(o.offsets), _lib.ptr(out))
        return out

    def extract_tuples(self):
        o = self._csr
        return (to_host(self.row_ids(), INDEX_DTYPE), to_host(o.indices, INDEX_DTYPE),
                to_host(o.dense_values()))

    def extract_element(self, i, j):
        if not (0 <= i < self.nrows and 0 <= j < self.ncols):
            raise IndexError("matrix index out of range")
        o = self._csr
        lo, hi = int(o.offsets[i].item()), int(o.offsets[i + 1].item())
        seg = to_host(o.indices[lo:hi])
        pos = int(np.searchsorted(seg, j))
        if pos < seg.size and seg[pos] == j:
            if o.values is None:
                return self._dt.type(o.iso)
            return self._dt.type(o.values[lo + pos].item())
        return None

    def set_element(self, i, j, value):
        """Overwrite or insert one entry (O(nnz), a poke; containers.py:418-428)."""
        rows, cols, vals = self.extract_tuples()
        keep = ~((rows == i) & (cols == j))
        rows = np.append(rows[keep], i)
        cols = np.append(cols[keep], j)
        vals = np.append(vals[keep], value)
        rebuilt = SparseMatrix.from_tuples(rows, cols, vals, self.nrows, self.ncols,
                                           build_csc=self.has_csc)
        for name in ("nrows", "ncols", "_csr", "_csc", "_dt", "_sym"):
            setattr(self, name, getattr(rebuilt, name))

    def dup(self) -> "SparseMatrix":
        def cp(o):
            if o is None:
                return None
            return _Orient(o.nrows, o.ncols, o.offsets.clone(), o.indices.clone(),
                           None if o.values is None else o.values.clone(), o.iso, o.dt)
        csr = cp(self._csr)
        csc = csr if self._csc is self._csr else cp(self._csc)
        return SparseMatrix._wrap(self.nrows, self.ncols, csr, csc, self._dt, self._sym)

    def clear(self):
        had = self.has_csc
        self._csr = _Orient(self.nrows, self.ncols, torch.zeros(self.nrows + 1, dtype=torch.int64,
                            device=_device()), empty(0, np.int32), empty(0, self._dt), None, self._dt)
        self._csc = None
        if had:
            self._csc = _Orient(self.ncols, self.nrows, torch.zeros(self.ncols + 1, dtype=torch.int64,
                                device=_device()), empty(0, np.int32), empty(0, self._dt), None, self._dt)
        self._sym = None

    def __repr__(self):
        return f"<SparseMatrix {self.nrows}x{self.ncols} nnz={self.nnz}>"


def _make_orient(nrows, ncols, offsets, indices, values, dt):
    off = to_dev(offsets, np.int64)
    idx = to_dev(indices, np.int32)
    vals = to_dev(values, dt)
    iso = _iso_of(vals, dt)
    return _Orient(nrows, ncols, off, idx, None if iso is not None else vals, iso, dt)


def matrix_build(tuples, nrows, ncols, dedup: Optional[Monoid] = None,
                 build_csc=True, dtype=None) -> SparseMatrix:
    tuples = list(tuples)
    if tuples:
        rows, cols, vals = zip(*tuples)
    else:
        rows, cols, vals = [], [], []
    if dtype is None and not tuples:
        dtype = np.int64
    return SparseMatrix.from_tuples(rows, cols, vals, nrows, ncols,
                                    dedup=dedup, build_csc=build_csc, dtype=dtype)
