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
import os
import weakref

import numpy as np
import torch

from . import _lib
from .algebra import LESS, MINUS, TIMES, builtin_monoid, builtin_semiring
from .containers import (INDEX_DTYPE, DecisionLog, Descriptor, Direction, SparseMatrix, Vector,
                         empty, full, iota)
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
# bfs over the degree-ordered relabelling (SparseMatrix.traversal); GB_BFS_ORDER=0
# keeps the original labels (A/B measurement, tests of both paths)
_ORDERED_BFS = os.environ.get("GB_BFS_ORDER", "1") != "0"
# pagerank iterates on the same layout (s22 x20: 10.9-11.2 ms vs 12.1-12.5 ms
# on the stored labels); GB_PR_ORDER=0 keeps the stored labels
_ORDERED_PR = os.environ.get("GB_PR_ORDER", "1") != "0"
# sssp too (s20: 1.86 vs 1.94 ms); GB_SSSP_ORDER=0 keeps the stored labels
_ORDERED_SSSP = os.environ.get("GB_SSSP_ORDER", "1") != "0"

_POLICY = {Direction.AUTO: _lib.DIR_AUTO, Direction.FORCE_PUSH: _lib.DIR_PUSH,
           Direction.FORCE_PULL: _lib.DIR_PULL}


def _require_square(A):
    if A.nrows != A.ncols:
        raise ShapeError(f"adjacency matrix must be square, got {A.nrows}x{A.ncols}")


def _require_symmetric(A):
    """algorithms.py:41-45 -- O(1) once the build has compared CSR and CSC."""
    if not A.is_symmetric():
        raise ValueError("adjacency matrix must be symmetric (undirected graph)")


_ASYNC_CAP = 65000   # loop caps the asynchronous entry accepts (16-bit device levels)
# GB_BFS_ASYNC=0: every bfs() call synchronises and fills the log eagerly
_ASYNC_BFS = os.environ.get("GB_BFS_ASYNC", "1") != "0"
_TINY_K = 4096   # gb_bfs.cu kTinyK: push levels up to this many entries take the one-kernel path
_LOG_PREFIX = 21     # decisions gb_bfs_ordered_async copies to the pinned log


class _PendingBfs:
    """Resolver of one asynchronous bfs: waits for it, then returns its
    DirectionDecision list (and books its kernel launches).  Its log lives in
    a slot of the context's ring (pinned prefix + device buffer); the slot is
    settled -- copied out -- before the ring reuses it."""

    def __init__(self, ctx, A, switch_ratio, info):
        self.ctx = ctx
        self.total = A.nnz
        self.thr = A.nnz * switch_ratio
        self.info = info
        self.row = None
        self.dev = None
        self.event = None
        self.raw = None

    def settle(self):
        if self.raw is None:
            self.event.sync()
            raw = self.row.numpy().copy()
            iters = int(raw[0])
            if iters > _LOG_PREFIX:
                tail = self.dev[1 + 3 * _LOG_PREFIX:1 + 3 * iters].cpu().numpy()
                raw = np.concatenate([raw, tail])
            self.raw = raw
            self.row = self.dev = None

    def __call__(self):
        self.settle()
        raw = self.raw
        iters = int(raw[0])
        dirs = raw[1:1 + 3 * iters:3]
        info = self.info
        if info[0]:
            push = dirs == _lib.DIR_PUSH
            kk = raw[2:2 + 3 * iters:3]
            npush1 = int(np.count_nonzero(push & (kk == 1)))
            ntiny = int(np.count_nonzero(push & (kk > 1) & (kk <= _TINY_K)))
            npush = int(np.count_nonzero(push)) - npush1 - ntiny
            # single-entry push levels skip the degree scan, tiny ones take the
            # one-kernel path; + the no-op g_steps of the device loop's last pass
            u = int(info[3])
            self.ctx.lib.gb_count_launches(self.ctx.ptr, int(info[0] + npush * info[1] +
                                                            npush1 * info[4] +
                                                            ntiny * info[5] +
                                                            (iters - npush - npush1 - ntiny) *
                                                            info[2] +
                                                            (u - iters % u) % u))
        return [DirectionDecision("pull" if dirs[i] == _lib.DIR_PULL else "push",
                                  int(raw[2 + 3 * i]), int(raw[3 + 3 * i]), self.total, self.thr)
                for i in range(iters)]


class _LogRing:
    """Log buffers of asynchronous bfs calls, allocated once per context and
    reused round robin: a pinned prefix row and a device log per slot (pinning
    or allocating per call costs milliseconds and can synchronise).  The
    device logs of calls up to the default loop cap share one slab allocated
    on first use: per-slot allocations came from the caching allocator's small
    pool, whose every eighth request mapped a new 2 MB segment with a
    synchronising cudaMalloc -- that drained the queue of asynchronous calls."""

    SLOTS = 256
    STRIDE = 1 + 3 * 10_000   # Descriptor().max_niter

    def __init__(self, device):
        self.pin = torch.empty((self.SLOTS, 1 + 3 * _LOG_PREFIX), dtype=torch.int64,
                               pin_memory=True)
        self.slab = None
        # device logs of larger caps are sized per slot, on first use
        self.dev = [None] * self.SLOTS
        self.device = device
        self.owner = [None] * self.SLOTS
        self.events = [None] * self.SLOTS  # completion event per slot (reused)
        self.next = 0

    def _settle(self, i):
        prev = self.owner[i]() if self.owner[i] is not None else None
        if prev is not None:
            prev.settle()
        self.owner[i] = None

    def take(self, pending, cap):
        need = 1 + 3 * cap
        i = self.next
        self.next = (i + 1) % self.SLOTS
        self._settle(i)  # the slot's previous call has finished with both buffers
        if need <= self.STRIDE:
            if self.slab is None:
                self.slab = torch.empty((self.SLOTS, self.STRIDE), dtype=torch.int64,
                                        device=self.device)
            dev = self.slab[i]
        else:
            if self.dev[i] is None or self.dev[i].numel() < need:
                self.dev[i] = torch.empty(need, dtype=torch.int64, device=self.device)
            dev = self.dev[i]
        self.owner[i] = weakref.ref(pending)
        if self.events[i] is None:
            self.events[i] = _lib.DeviceEvent(pending.ctx)
        pending.event = self.events[i]
        pending.row = self.pin[i]
        pending.dev = dev
        return self.pin[i], dev

    def release(self):
        """Settle every outstanding call and drop the device logs (ctx.trim())."""
        for i in range(self.SLOTS):
            self._settle(i)
        self.slab = None
        self.dev = [None] * self.SLOTS


_rings = {}


def _log_ring(ctx, device):
    ring = _rings.get(id(ctx))
    if ring is None:
        ring = _rings[id(ctx)] = _LogRing(device)
        ctx.on_trim(ring.release)
    return ring


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
    if desc.count_work:
        first = len(desc.direction_log)
        levels = _bfs_fused(A, source, desc)
        _bfs_count_work(A, source, desc, levels, desc.direction_log[first:])
        return levels
    return _bfs_fused(A, source, desc)


def _bfs_count_work(A, source, desc, levels, decisions):
    """desc.counters += the reference's tallies of this BFS (gb_bfs_counters:
    recomputed from the levels and the direction log); beyond its limits
    (valued matrices, > 64 levels, > 4 pull levels) the composition is
    replayed for the counts."""
    dirs = np.array([_lib.DIR_PULL if d.chosen == "pull" else _lib.DIR_PUSH for d in decisions],
                    np.int32)
    tot = np.zeros(3, np.int64)
    try:
        if not A.has_csc:
            raise NotImplementedError
        s, _k1 = A.orient(False).csr_struct()
        t, _k2 = A.orient(True).csr_struct()
        _lib.context().call("gb_bfs_counters", C.byref(s), C.byref(t), _lib.ptr(levels._vals),
                            int(dirs.size), dirs.ctypes.data_as(C.c_void_p),
                            1 if desc.early_exit else 0, tot.ctypes.data_as(C.c_void_p))
    except NotImplementedError:
        d = Descriptor(direction=desc.direction, switch_ratio=desc.switch_ratio,
                       max_niter=desc.max_niter, fused=False, early_exit=desc.early_exit)
        _bfs_composed(A, source, d)
        tot[:] = (d.counters.matrix_entries_read, d.counters.semiring_multiplies,
                  d.counters.semiring_adds)
    desc.counters.matrix_entries_read += int(tot[0])
    desc.counters.semiring_multiplies += int(tot[1])
    desc.counters.semiring_adds += int(tot[2])


def _bfs_fused(A, source, desc):
    n = A.nrows
    iters = min(desc.max_niter, n + 1)
    if iters <= 0:
        # the reference loop runs zero times: an all-zero level vector, no log
        return Vector._wrap(n, None, full(n, 0, np.int64), 0, np.int64)
    levels = empty(n, np.int64)
    cap = max(iters, 1)
    dirs = np.zeros(cap, np.int32)
    nv = np.zeros(cap, np.int64)
    est = np.zeros(cap, np.int64)
    done = C.c_int64(0)
    trav = A.traversal() if _ORDERED_BFS else None
    if (trav is not None and _ASYNC_BFS and isinstance(desc.direction_log, DecisionLog)
            and cap < _ASYNC_CAP):
        # degree-ordered relabelling, enqueued without a host
        # synchronisation: the decision log is read when first used
        push_o, pull_o, rank = trav
        (push, _k1), (pull, _k2) = push_o.csr_struct(), pull_o.csr_struct()
        ctx = _lib.context()
        info = np.zeros(6, np.int64)
        pending = _PendingBfs(ctx, A, desc.switch_ratio, info)
        log_pin, log_dev = _log_ring(ctx, levels.device).take(pending, cap)
        ctx.call("gb_bfs_ordered_async", C.byref(push), C.byref(pull), _lib.ptr(pull_o.nonempty()),
                 _lib.ptr(rank), int(source), int(iters), float(desc.switch_ratio),
                 _POLICY[desc.direction], _lib.ptr(levels), _lib.ptr(log_dev),
                 C.c_void_p(log_pin.data_ptr()), info.ctypes.data_as(C.c_void_p))
        pending.event.record(ctx)
        desc.direction_log._defer(pending)
        return Vector._wrap(n, None, levels, 0, np.int64)
    if trav is not None:
        # degree-ordered relabelling: same levels and log
        push_o, pull_o, rank = trav
        (push, _k1), (pull, _k2) = push_o.csr_struct(), pull_o.csr_struct()
        _lib.context().call(
            "gb_bfs_ordered", C.byref(push), C.byref(pull), _lib.ptr(pull_o.nonempty()),
            _lib.ptr(rank), int(source), int(iters), float(desc.switch_ratio),
            _POLICY[desc.direction], _lib.ptr(levels), dirs.ctypes.data_as(C.c_void_p),
            nv.ctypes.data_as(C.c_void_p), est.ctypes.data_as(C.c_void_p), C.byref(done))
        _log_decisions(desc, A, dirs, nv, est, int(done.value))
        return Vector._wrap(n, None, levels, 0, np.int64)
    push, _k1 = A.orient(False).csr_struct()          # vxm push walks rows of A (CSR)
    pull_o = A.orient(True) if A.has_csc else None    # vxm pull walks rows of A^T (CSC)
    pull, _k2 = pull_o.csr_struct() if pull_o is not None else (None, None)
    _lib.context().call(
        "gb_bfs", C.byref(push), C.byref(pull) if pull is not None else None,
        _lib.ptr(pull_o.nonempty()) if pull_o is not None else None,
        int(source), int(iters), float(desc.switch_ratio), _POLICY[desc.direction],
        _lib.ptr(levels), dirs.ctypes.data_as(C.c_void_p), nv.ctypes.data_as(C.c_void_p),
        est.ctypes.data_as(C.c_void_p), C.byref(done))
    _log_decisions(desc, A, dirs, nv, est, int(done.value))
    return Vector._wrap(n, None, levels, 0, np.int64)


def bfs_parents(A: SparseMatrix, source: int, desc=None):
    """Extension beyond the reference (which returns levels only,
    algorithms.py:66-77; BASELINE.json north star "BFS levels/parents"):
    ``(levels, parents)`` where ``levels`` is exactly ``bfs(A, source)`` and
    ``parents`` a BFS tree derived from it on the device (gb_bfs_parents):
    parent[v] = the smallest u with (u, v) stored in A and level[u] =
    level[v] - 1, parent[source] = source, -1 when unreached."""
    levels = bfs(A, source, desc)
    n = A.nrows
    parents = empty(n, np.int64)
    s, _k = A.orient(True).csr_struct()   # in-edges: rows of A^T (FormatError without CSC)
    _lib.context().call("gb_bfs_parents", C.byref(s), _lib.ptr(levels._vals), int(source),
                        _lib.ptr(parents))
    return levels, Vector._wrap(n, None, parents, -1, np.int64)


def validate_bfs(A: SparseMatrix, source: int, levels, parents) -> dict:
    """Graph500-style validation of a BFS tree on the device
    (gb_bfs_validate): violation counts of the four checks; ``ok`` when all
    are zero.  ``levels``/``parents`` are Vectors from bfs_parents (or any
    int64 vectors of the same meaning)."""
    _require_square(A)
    s, _k1 = A.orient(False).csr_struct()
    t, _k2 = A.orient(True).csr_struct()
    lv = levels.to_dense(0)._vals if isinstance(levels, Vector) else levels
    pa = parents.to_dense(-1)._vals if isinstance(parents, Vector) else parents
    err = np.zeros(4, np.int64)
    _lib.context().call("gb_bfs_validate", C.byref(s), C.byref(t), int(source), _lib.ptr(lv),
                        _lib.ptr(pa), err.ctypes.data_as(C.c_void_p))
    names = ("source", "tree_edges", "unreached", "graph_edges")
    out = {k: int(v) for k, v in zip(names, err)}
    out["ok"] = not err.any()
    return out


def _replay_counts(desc, run):
    """count_work for SSSP / CC / TC: the reference's tallies come from
    replaying the operator composition (run(d) with a fused=False copy of the
    descriptor's settings); results still come from the fused driver."""
    d = Descriptor(direction=desc.direction, switch_ratio=desc.switch_ratio,
                   max_niter=desc.max_niter, fused=False)
    run(d)
    desc.counters.merge(d.counters)


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




# ---------------------------------------------------------------------------
# SSSP
# ---------------------------------------------------------------------------


def sssp(A: SparseMatrix, source: int, desc=None, on_iteration=None) -> Vector:
    """Single-source shortest distances by frontier-sparsified relaxation (algorithms.py:80-119)."""
    _require_square(A)
    if not 0 <= source < A.nrows:
        raise IndexError(f"source {source} out of range")
    wmin = _min_value(A) if A.nnz else 0.0
    if A.nnz and wmin <= 0:
        raise ValueError("edge weights must be positive")
    desc = desc if desc is not None else Descriptor()
    if not desc.fused:
        return _sssp_composed(A, source, desc, on_iteration)
    if desc.count_work:
        _replay_counts(desc, lambda d: _sssp_composed(A, source, d, None))
    n = A.nrows
    iters = min(desc.max_niter, n)
    dist = empty(n, np.float64)
    trav = A.traversal() if _ORDERED_SSSP and on_iteration is None else None
    if trav is not None:
        # relax on the degree-ordered layout, unpermute the distances once
        push_o, pull_o, rank = trav
        src_run = int(rank[source].item())
        work = empty(n, np.float64)
    else:
        push_o = A.orient(False)
        pull_o = A.orient(True) if A.has_csc else None
        src_run, work = source, dist
    push, _k1 = push_o.csr_struct()
    pull, _k2 = pull_o.csr_struct() if pull_o is not None else (None, None)
    cap = max(iters, 1)
    dirs, nv, est = np.zeros(cap, np.int32), np.zeros(cap, np.int64), np.zeros(cap, np.int64)
    done = C.c_int64(0)
    cb = _lib.ITER_CB()  # NULL function pointer
    if on_iteration is not None:
        def _hook(it, _user):
            on_iteration(int(it), Vector._wrap(n, None, dist.clone(), np.inf, np.float64))
        cb = _lib.ITER_CB(_hook)
    ctx = _lib.context()
    ctx.call(
        "gb_sssp", C.byref(push), C.byref(pull) if pull is not None else None, int(src_run),
        int(iters), float(desc.switch_ratio), _POLICY[desc.direction], float(wmin), _lib.ptr(work),
        dirs.ctypes.data_as(C.c_void_p), nv.ctypes.data_as(C.c_void_p),
        est.ctypes.data_as(C.c_void_p), C.byref(done), cb, None)
    if trav is not None:
        ctx.call("gb_gather", _lib.dtype_code(np.float64), n, _lib.ptr(A._rank64()), n,
                 _lib.ptr(work), _lib.ptr(dist))
    _log_decisions(desc, A, dirs, nv, est, int(done.value))
    return Vector._wrap(n, None, dist, np.inf, np.float64)


def _min_value(A):
    """Smallest stored value (sssp's positivity check and its pull bound).
    Cached on the orientation, keyed by the values tensor and its in-place
    version counter, so repeated calls on one matrix skip the reduction and
    its host synchronisation (s20: a 50 us pass over 31 M weights per call)."""
    o = A.orient(False)
    if o.values is None:
        return o.iso
    key = (o.values.data_ptr(), o.values._version, o.nnz)
    hit = getattr(o, "_min_cache", None)
    if hit is not None and hit[0] == key:
        return hit[1]
    lo, hi = C.c_double(), C.c_double()
    _lib.context().call("gb_values_minmax", o.nnz, _lib.ptr(o.values), _lib.dtype_code(o.dt),
                        C.byref(lo), C.byref(hi))
    o._min_cache = (key, lo.value)
    return lo.value


def _sssp_composed(A, source, desc, on_iteration):
    min_plus = builtin_semiring("MinPlus")
    minimum = builtin_monoid("Minimum")
    plus = builtin_monoid("Plus")
    n = A.nrows
    dist = Vector.filled(n, np.inf, dtype=np.float64)
    dist.zero = np.float64(np.inf)
    dist.set_element(source, 0.0)
    frontier = Vector.from_entries([source], [0.0], n, dtype=np.float64)
    ceiling = Vector.filled(n, np.finfo(np.float64).max)
    succ_last = -1.0
    for it in range(min(desc.max_niter, n)):
        candidates = vxm(min_plus, frontier, A, desc=desc)
        improved = ewise_mult(LESS, candidates, dist, desc=desc)
        dist = ewise_add(minimum, dist, candidates, desc=desc)
        frontier = apply(lambda x: x, candidates, mask=improved, desc=desc)
        if on_iteration is not None:
            on_iteration(it, dist.dup())
        reached = ewise_mult(builtin_semiring("PlusLess"), dist, ceiling, desc=desc)
        succ = float(reduce(plus, reached))
        if succ == succ_last and frontier.nvals == 0:
            break
        succ_last = succ
    return dist


# ---------------------------------------------------------------------------
# PageRank
# ---------------------------------------------------------------------------


def pagerank(A: SparseMatrix, alpha=0.85, eps=1e-7, max_iters=10_000, desc=None) -> Vector:
    """Damped rank scores; iterates until the L2 step delta is <= eps (algorithms.py:132-162).

    The fused driver multiplies with the pull kernel (the reference dispatch
    always pulls a PageRank iterate: every rank is >= (1-alpha)/n > 0, so the
    estimate is nnz > switch_ratio*nnz); FORCE_PUSH replays the composition."""
    _require_square(A)
    if not 0.0 < alpha < 1.0:
        raise ValueError(f"alpha must be in (0, 1), got {alpha}")
    if eps <= 0.0:
        raise ValueError(f"eps must be positive, got {eps}")
    desc = desc if desc is not None else Descriptor()
    if not desc.fused or desc.direction is Direction.FORCE_PUSH or A.nnz == 0:
        return _pagerank_composed(A, alpha, eps, max_iters, desc)
    first = len(desc.direction_log) if desc.count_work else 0
    out = _pagerank_fused(A, alpha, eps, max_iters, desc)
    if desc.count_work:
        log = desc.direction_log[first:]
        if all(d.chosen == "pull" and d.frontier_nvals == A.nrows for d in log):
            # every iterate positive (teleport > 0): each pull reads and
            # multiplies every stored entry, one segment per non-empty row
            # (kernels.py:153-191)
            nnz = A.nnz
            rows = int(A.orient(True).row_plan()[0].nrows_nz)
            desc.counters.matrix_entries_read += nnz * len(log)
            desc.counters.semiring_multiplies += nnz * len(log)
            desc.counters.semiring_adds += (nnz - rows) * len(log)
        else:
            d = Descriptor(direction=desc.direction, switch_ratio=desc.switch_ratio, fused=False)
            _pagerank_composed(A, alpha, eps, max_iters, d)
            desc.counters.merge(d.counters)
    return out


def _pagerank_fused(A, alpha, eps, max_iters, desc):
    n = A.nrows
    ranks = empty(n, np.float64)
    trav = A.traversal() if _ORDERED_PR else None
    if trav is not None:
        # iterate on the degree-ordered layout (hub ranks packed in L1/L2),
        # unpermute once at the end
        push_o, pull_o, rank = trav
        out_off = push_o.offsets
        work = empty(n, np.float64)
    else:
        pull_o, out_off, work = A.orient(True), A.orient(False).offsets, ranks
    pull, _k = pull_o.csr_struct()
    cap = max(max_iters, 1)
    dirs, nv, est = np.zeros(cap, np.int32), np.zeros(cap, np.int64), np.zeros(cap, np.int64)
    errs = np.zeros(cap, np.float64)
    done = C.c_int64(0)
    ctx = _lib.context()
    ctx.call(
        "gb_pagerank", C.byref(pull), _lib.ptr(out_off), float(alpha), float(eps),
        int(max_iters), float(desc.switch_ratio), _POLICY[desc.direction], _lib.ptr(work),
        dirs.ctypes.data_as(C.c_void_p), nv.ctypes.data_as(C.c_void_p),
        est.ctypes.data_as(C.c_void_p), errs.ctypes.data_as(C.c_void_p), C.byref(done))
    if trav is not None:
        ctx.call("gb_gather", _lib.dtype_code(np.float64), n, _lib.ptr(A._rank64()), n,
                 _lib.ptr(work), _lib.ptr(ranks))
    _log_decisions(desc, A, dirs, nv, est, int(done.value))
    return Vector._wrap(n, None, ranks, 0.0, np.float64)


def _scale_rows(A, alpha):
    """algorithms.py:122-129: Â(i, j) = alpha / outdegree(i), as a device matrix."""
    o = A.orient(False)
    vals = empty(o.nnz, np.float64)
    _lib.context().call("gb_scale_rows", A.nrows, _lib.ptr(o.offsets), float(alpha),
                        _lib.ptr(vals))
    return SparseMatrix.from_csr(A.nrows, A.ncols, o.offsets, o.indices, vals)


def _pagerank_composed(A, alpha, eps, max_iters, desc):
    plus_times = builtin_semiring("PlusMultiplies")
    plus = builtin_monoid("Plus")
    n = A.nrows
    scaled = _scale_rows(A, alpha)
    teleport = (1.0 - alpha) / n
    ranks = Vector.filled(n, 1.0 / n)
    for _ in range(max_iters):
        previous = ranks
        spread = vxm(plus_times, previous, scaled, desc=desc)
        ranks = ewise_add(plus_times, spread, teleport, desc=desc)
        delta = ewise_mult(MINUS, ranks, previous, desc=desc)
        squared = ewise_add(TIMES, delta, delta, desc=desc)
        error = math.sqrt(float(reduce(plus, squared)))
        if error <= eps:
            break
    return ranks


# ---------------------------------------------------------------------------
# Connected components (FastSV)
# ---------------------------------------------------------------------------


def connected_components(A: SparseMatrix, desc=None, sparsify=True) -> Vector:
    """Component labels = minimum vertex id per component (algorithms.py:165-203)."""
    _require_square(A)
    _require_symmetric(A)
    desc = desc if desc is not None else Descriptor()
    if not desc.fused:
        return _cc_composed(A, desc, sparsify)
    if desc.count_work:
        _replay_counts(desc, lambda d: _cc_composed(A, d, sparsify))
    n = A.nrows
    parent = empty(n, np.int64)
    rows, _k1 = A.orient(False).csr_struct()
    cols, _k2 = A.orient(True).csr_struct()
    cap = max(desc.max_niter, 1)
    dirs, nv, est = np.zeros(cap, np.int32), np.zeros(cap, np.int64), np.zeros(cap, np.int64)
    done = C.c_int64(0)
    if desc.max_niter <= 0:
        return Vector._wrap(n, None, iota(n, np.int64), 0,
                            np.int64)
    _lib.context().call(
        "gb_cc", C.byref(rows), C.byref(cols), int(desc.max_niter), float(desc.switch_ratio),
        _POLICY[desc.direction], 1 if sparsify else 0, _lib.ptr(parent),
        dirs.ctypes.data_as(C.c_void_p), nv.ctypes.data_as(C.c_void_p),
        est.ctypes.data_as(C.c_void_p), C.byref(done))
    _log_decisions(desc, A, dirs, nv, est, int(done.value))
    return Vector._wrap(n, None, parent, _INT_INF, np.int64)


def _cc_composed(A, desc, sparsify):
    min_second = builtin_semiring("MinimumSelectSecond")
    min_fold = builtin_monoid("Minimum")
    not_equal = builtin_semiring("MinimumNotEqualTo")
    plus = builtin_monoid("Plus")
    n = A.nrows
    parent = Vector.dense_of(np.arange(n, dtype=np.int64), 0)
    min_neighbor = parent.dup()
    grandparent = parent.dup()
    grandparent_prev = parent.dup()
    for _ in range(desc.max_niter):
        parent_prev = parent.dup()
        hooked = mxv(min_second, A, grandparent, desc=desc)
        min_neighbor = ewise_add(min_fold, min_neighbor, hooked, desc=desc)
        assign_scatter(parent, min_neighbor, parent_prev, desc=desc)
        parent = ewise_add(min_fold, parent, min_neighbor, desc=desc)
        parent = ewise_add(min_fold, parent, parent_prev, desc=desc)
        extract_gather(grandparent, parent, parent, desc=desc)
        changed = ewise_mult(not_equal, grandparent_prev, grandparent, desc=desc)
        if int(reduce(plus, changed)) == 0:
            break
        grandparent_prev = grandparent.dup()
        if sparsify:
            desc.toggle("mask")
            assign(grandparent, _INT_INF, mask=changed, desc=desc)
            desc.toggle("mask")
    return parent


# ---------------------------------------------------------------------------
# Triangle counting
# ---------------------------------------------------------------------------


def _has_diagonal(A):
    s, _k = A.orient(False).csr_struct()
    f = C.c_int32(0)
    _lib.context().call("gb_has_diagonal", C.byref(s), C.byref(f))
    return bool(f.value)


def triangle_count(A: SparseMatrix, desc=None) -> int:
    """Triangles of an undirected simple graph, each counted once (algorithms.py:221-240).

    Fused: one device pass ranks vertices by (degree, id), keeps each vertex's
    higher-ranked neighbours and counts sorted-list intersections -- the same
    integer the reference's masked product L.L^T.*L reduces to."""
    _require_square(A)
    _require_symmetric(A)
    if _has_diagonal(A):
        raise ValueError("adjacency matrix must have an empty diagonal")
    desc = desc if desc is not None else Descriptor()
    if not desc.fused:
        return _tc_composed(A, desc)
    if desc.count_work:
        _replay_counts(desc, lambda d: _tc_composed(A, d))
    o = A.orient(False)
    if o.values is not None or (o.iso is not None and o.iso != 1):
        # weighted entries: the product sums value products, not a count
        return _tc_composed(A, desc)
    s, _k = o.csr_struct()
    c = C.c_int64(0)
    _lib.context().call("gb_tc", C.byref(s), C.byref(c))
    return int(c.value)


def _degree_sorted_lower_triangle(A):
    """algorithms.py:206-218 on the device."""
    o = A.orient(False)
    s, _k = o.csr_struct()
    rows, cols = empty(max(o.nnz, 1), np.int64), empty(max(o.nnz, 1), np.int64)
    vals = empty(max(o.nnz, 1), o.dt)
    c = C.c_int64(0)
    _lib.context().call("gb_lower_by_rank", C.byref(s), _lib.ptr(rows), _lib.ptr(cols),
                        _lib.ptr(vals), C.byref(c))
    k = int(c.value)
    return SparseMatrix.from_tuples(rows[:k], cols[:k], vals[:k], A.nrows, A.ncols)


def _tc_composed(A, desc):
    plus_times = builtin_semiring("PlusMultiplies")
    plus = builtin_monoid("Plus")
    lower = _degree_sorted_lower_triangle(A)
    desc.toggle("inp1")
    closed = mxm_masked(plus_times, lower, lower, mask=lower, desc=desc)
    desc.toggle("inp1")
    return int(reduce_scalar_matrix(plus, closed))
