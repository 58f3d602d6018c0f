"""1D-partitioned multi-GPU BFS (north star: "the graph is 1D row-partitioned
across GPUs, and each iteration's frontier is exchanged with NCCL").

One process per GPU (torchrun), ``torch.distributed`` over NCCL for the
plumbing.  Rank p owns the contiguous vertex block [lo, hi); block boundaries
put ~nnz/P stored entries in every block -- the reference's nonzero split
(kernels.py:133-150) lifted from threads to GPUs -- and are multiples of
1024 so bitmap words (and the 32-word groups the kernels walk) never straddle
two ranks.  Each rank stores

* ``rowblock`` -- rows lo..hi-1 of A^T (in-edges of its vertices): the pull
  direction walks them against the replicated frontier bitmap;
* ``colblock`` -- all n rows of A restricted to columns in [lo, hi): the push
  direction expands the replicated frontier list over it, so only owned
  vertices are ever marked.

Per BFS level the new frontier is replicated by the exchange the north star
names (FrontierExchange): every rank lists its owned new vertices and the P
counts are allgathered (8 B per rank; their sum is the global frontier size
|f|, so no separate reduction or read-back is needed); then either a dense
ALLGATHER of the owned bitmap word slices (|f|*32 > n: n/8 bytes in total)
or an ALLGATHERV of the owned vertex ids (4 B per new vertex; NCCL has no
native allgatherv, so the lists are padded to the largest count).  Every
rank then applies the same global bitmap, so the frontier count, the
push/pull decision (the reference rule, kernels.py:108-126) and the level
vector are identical and replicated -- no all-to-all is needed.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .containers import Descriptor, Direction, SparseMatrix, Vector, _Orient
from .kernels import DirectionDecision, direction_rule

ALIGN = 1024


def partition_bounds(row_offsets, world: int, align: int = ALIGN):
    """Edge-balanced vertex blocks: world+1 boundaries, multiples of ``align``
    (except the last = n), non-decreasing."""
    off = np.asarray(row_offsets, dtype=np.int64)
    n = off.size - 1
    total = int(off[-1])
    targets = np.arange(world + 1, dtype=np.float64) * total / world
    b = np.searchsorted(off, targets, side="left").astype(np.int64)
    b = (b + align // 2) // align * align
    b = np.clip(b, 0, n // align * align)  # inner boundaries stay aligned
    b[0], b[-1] = 0, n
    return np.maximum.accumulate(b).tolist()


@dataclass
class BlockGraph:
    """One rank's share of a square matrix (device tensors)."""

    n: int
    nnz: int                    # global stored entries (the direction rule's nnz)
    lo: int
    hi: int
    bounds: list
    row_off: torch.Tensor       # [hi-lo+1], rebased
    row_idx: torch.Tensor       # global column ids
    row_nonempty: torch.Tensor  # ceil((hi-lo)/32) words
    col_off: torch.Tensor       # [n+1]
    col_idx: torch.Tensor       # global column ids in [lo, hi)
    values_iso: object = 1

    @classmethod
    def from_matrix(cls, A: SparseMatrix, rank: int, world: int, bounds=None):
        if A.nrows != A.ncols:
            raise ValueError("1D partitioning needs a square matrix")
        if A._csr.values is not None:
            raise NotImplementedError("distributed BFS takes a pattern (iso-valued) matrix")
        n = A.nrows
        csr = A.orient(False)
        csc = A.orient(True)
        if bounds is None:
            bounds = partition_bounds(csr.offsets.cpu().numpy(), world)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        ctx = _lib.context()
        # pull block: rows lo..hi-1 of the in-edge orientation
        a, b = int(csc.offsets[lo].item()), int(csc.offsets[hi].item())
        row_off = (csc.offsets[lo:hi + 1] - a).contiguous()
        row_idx = csc.indices[a:b].clone()
        W = max((hi - lo + 31) // 32, 1)
        ne = torch.zeros(W, dtype=torch.int32, device=row_off.device)
        if hi > lo:
            ctx.call("gb_nonempty_rows", hi - lo, _lib.ptr(row_off), _lib.ptr(ne))
        # push block: rows of A, columns in [lo, hi)
        s, _k = csr.csr_struct()
        col_off = torch.empty(n + 1, dtype=torch.int64, device=row_off.device)
        cnt = C.c_int64(0)
        ctx.call("gb_csr_column_block", C.byref(s), lo, hi, _lib.ptr(col_off), None, C.byref(cnt))
        col_idx = torch.empty(max(int(cnt.value), 1), dtype=torch.int32, device=row_off.device)
        ctx.call("gb_csr_column_block", C.byref(s), lo, hi, _lib.ptr(col_off), _lib.ptr(col_idx),
                 C.byref(cnt))
        return cls(n, A.nnz, lo, hi, list(bounds), row_off, row_idx, ne, col_off,
                   col_idx[:int(cnt.value)], csr.iso)

    def _orient(self, which):
        if which == "row":
            return _Orient(self.hi - self.lo, self.n, self.row_off, self.row_idx, None,
                           self.values_iso, np.int64)
        return _Orient(self.n, self.n, self.col_off, self.col_idx, None, self.values_iso, np.int64)


class NativeSteps:
    """The per-rank level steps, executed by libgraphblast_sm100a."""

    def __init__(self, g: BlockGraph):
        self.g = g
        self.ctx = _lib.context()
        self.rows, self._k1 = g._orient("row").csr_struct()
        self.cols, self._k2 = g._orient("col").csr_struct()
        n = g.n
        W = (n + 31) // 32
        dev = g.row_off.device
        self.levels = torch.empty(n, dtype=torch.int64, device=dev)
        self.vbm = torch.empty(W, dtype=torch.int32, device=dev)
        self.vprev = torch.empty(W, dtype=torch.int32, device=dev)
        self.fbm = torch.empty(W, dtype=torch.int32, device=dev)
        self.xbm = torch.empty(W, dtype=torch.int32, device=dev)
        self.F = torch.empty(n, dtype=torch.int32, device=dev)
        self.ids = torch.empty(max(g.hi - g.lo, 1), dtype=torch.int32, device=dev)
        self.count = torch.zeros(1, dtype=torch.int64, device=dev)
        # rows sorted by column (the degree-ordered layout guarantees it):
        # the device-resident push may skip the dense visited prefix
        self.prefix_cut = False

    def init(self, source):
        p = _lib.ptr
        self.ctx.call("gb_bfs_dist_init", self.g.n, int(source), p(self.levels), p(self.vbm),
                      p(self.vprev), p(self.fbm), p(self.F))

    def push(self, K):
        g, p = self.g, _lib.ptr
        self.ctx.call("gb_bfs_dist_push", C.byref(self.cols), int(K), p(self.F), p(self.vbm))
        self.ctx.call("gb_bfs_dist_collect", g.n, g.lo, g.hi, p(self.vbm), p(self.vprev), p(self.xbm))

    def pull(self, depth):
        g, p = self.g, _lib.ptr
        self.ctx.call("gb_bfs_dist_pull", C.byref(self.rows), g.lo, g.hi, p(g.row_nonempty), g.n,
                      int(depth), p(self.vbm), p(self.vprev), p(self.fbm), p(self.xbm),
                      p(self.levels))

    def apply(self, depth, K=None):
        """Stamp the replicated new frontier.  K known (from the exchange): no
        read-back; otherwise the count is read (synchronizes)."""
        p = _lib.ptr
        k = C.c_int64(0)
        self.ctx.call("gb_bfs_dist_apply", self.g.n, int(depth), p(self.xbm), p(self.vbm),
                      p(self.vprev), p(self.fbm), p(self.levels), p(self.F),
                      None if K is not None else C.byref(k))
        return int(K) if K is not None else int(k.value)

    # -- frontier exchange steps (gb_bfs_dist_owned / pack / unpack / set_ids)
    def owned(self):
        """Device int64[1]: this rank's new vertices (listed in self.ids)."""
        g = self.g
        self.ctx.call("gb_bfs_dist_owned", g.lo, g.hi, _lib.ptr(self.xbm), _lib.ptr(self.ids),
                      _lib.ptr(self.count))
        return self.count

    def pack_words(self, wmax):
        out = torch.empty(max(wmax, 1), dtype=torch.int32, device=self.xbm.device)
        self.ctx.call("gb_bfs_dist_pack_words", self.g.lo, self.g.hi, int(wmax),
                      _lib.ptr(self.xbm), _lib.ptr(out))
        return out[:wmax]

    def unpack_words(self, gathered, wmax, wb):
        self.ctx.call("gb_bfs_dist_unpack_words", int(wb.numel() - 1), int(wmax), _lib.ptr(wb),
                      _lib.ptr(gathered), _lib.ptr(self.xbm))

    def owned_ids(self, kmax):
        return self.ids[:kmax] if kmax <= self.ids.numel() else torch.cat(
            [self.ids, self.ids.new_zeros(kmax - self.ids.numel())])

    def set_ids(self, gathered, counts, kmax):
        self.ctx.call("gb_bfs_dist_set_ids", self.g.n, int(counts.numel()), int(kmax),
                      _lib.ptr(counts), _lib.ptr(gathered), _lib.ptr(self.xbm))

    def unstamp(self, K):
        self.ctx.call("gb_bfs_dist_unstamp", int(K), _lib.ptr(self.F), _lib.ptr(self.levels))

    # -- device-resident levels (gb_bfs_dist_dev_*): no scalar reaches the host
    STATE_DONE, STATE_ITERS = 6, 8   # DistBfsState fields read back (int64 slots)

    def dev_init(self, source, max_iters, switch_ratio, policy):
        g, p = self.g, _lib.ptr
        self.state = torch.zeros(24, dtype=torch.int64, device=self.levels.device)
        self.log = torch.zeros(1 + 3 * max(int(max_iters), 1), dtype=torch.int64,
                               device=self.levels.device)
        self.ctx.call("gb_bfs_dist_dev_init", p(self.state), p(self.log), g.n, g.nnz, int(source),
                      int(max_iters), float(switch_ratio), int(policy), p(self.levels), p(self.vbm),
                      p(self.vprev), p(self.fbm), p(self.F))

    def dev_level(self):
        g, p = self.g, _lib.ptr
        self.ctx.call("gb_bfs_dist_dev_level", p(self.state), p(self.log), C.byref(self.rows),
                      C.byref(self.cols), g.lo, g.hi, p(g.row_nonempty), g.n, p(self.vbm),
                      p(self.vprev), p(self.fbm), p(self.xbm), p(self.levels), p(self.F),
                      1 if self.prefix_cut else 0)

    def dev_apply(self):
        p = _lib.ptr
        self.ctx.call("gb_bfs_dist_dev_apply", p(self.state), self.g.n, p(self.xbm), p(self.vbm),
                      p(self.vprev), p(self.fbm), p(self.levels), p(self.F))


class FrontierExchange:
    """The per-level frontier exchange of the north star: allgather of the
    owned new-frontier counts, then a dense allgather of the owned bitmap
    word slices (|f|*32 > n) or an allgather(v) of the owned vertex ids.
    Returns the global frontier size; ``log`` records (mode, bytes sent per
    rank) per level."""

    def __init__(self, group=None):
        self.group = group
        self.log = []
        self._wb = None

    def _world(self):
        import torch.distributed as dist
        if dist.is_initialized():
            return dist.get_world_size(self.group)
        return 1

    def _allgather(self, t):
        """Equal-length 1-D tensors of every rank, concatenated in rank order."""
        import torch.distributed as dist
        P = dist.get_world_size(self.group)
        if dist.get_backend(self.group) == "nccl":
            out = torch.empty(P * t.numel(), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
            return out
        parts = [torch.empty_like(t) for _ in range(P)]
        dist.all_gather(parts, t.contiguous(), group=self.group)
        return torch.cat(parts)

    def word_bounds(self, g, device):
        if self._wb is None or self._wb[0] is not g:
            W = (g.n + 31) // 32
            wb = [min(b // 32, W) for b in g.bounds[:-1]] + [W]
            self._wb = (g, torch.tensor(wb, dtype=torch.int64, device=device),
                        max(b - a for a, b in zip(wb, wb[1:])))
        return self._wb[1], self._wb[2]

    def __call__(self, steps, g) -> int:
        count = steps.owned()
        P = self._world()
        if P == 1:
            total = int(count.item())
            self.log.append(("local", 0))
            return total
        counts = self._allgather(count)
        ch = counts.cpu().tolist()                      # the one host read per level
        total = int(sum(ch))
        if total * 32 > g.n:
            wb, wmax = self.word_bounds(g, count.device)
            gathered = self._allgather(steps.pack_words(wmax))
            steps.unpack_words(gathered, wmax, wb)
            self.log.append(("dense", 4 * wmax))
        else:
            kmax = max(ch)
            if kmax > 0:
                gathered = self._allgather(steps.owned_ids(kmax))
            else:
                gathered = count.new_zeros(0, dtype=torch.int32)
            steps.set_ids(gathered, counts, kmax)
            self.log.append(("sparse", 4 * kmax))
        return total


    def dense(self, steps, g):
        """The dense exchange alone (fixed size, nothing read back): the
        device-resident loop's per-level step."""
        if self._world() == 1:
            return
        wb, wmax = self.word_bounds(g, steps.xbm.device)
        gathered = self._allgather(steps.pack_words(wmax))
        steps.unpack_words(gathered, wmax, wb)
        self.log.append(("dense", 4 * wmax))


def bfs_partitioned_device(g: BlockGraph, source: int, desc=None, steps=None, exchange=None,
                           lookahead: int = 1):
    """bfs_partitioned with the level loop's scalars on the device
    (gb_bfs_dist_dev_*): the direction rule runs on the device, the push or
    pull kernel returns at once when the level took the other direction, and
    the frontier is exchanged as the dense allgather of owned word slices
    (2 MB over all ranks at s24 -- on NVSwitch a few microseconds, against a
    host round trip per level for the count-dependent sparse mode).  The host
    enqueues levels back to back and learns that the traversal ended from a
    pinned copy of the state's `done` flag, waiting only on the level
    `lookahead` behind (so every rank stops after the same number of
    collectives, `lookahead` no-op levels past the end).  Levels and the
    direction log equal bfs_partitioned's."""
    if not 0 <= source < g.n:
        raise IndexError(f"source {source} out of range")
    desc = desc if desc is not None else Descriptor()
    steps = steps if steps is not None else NativeSteps(g)
    exchange = exchange if exchange is not None else FrontierExchange()
    iters = min(desc.max_niter, g.n + 1)
    if iters <= 0:
        # the reference loop runs zero times: nothing is stamped, not even the source
        steps.init(source)
        steps.unstamp(1)
        return steps.levels
    policy = {Direction.AUTO: _lib.DIR_AUTO, Direction.FORCE_PUSH: _lib.DIR_PUSH,
              Direction.FORCE_PULL: _lib.DIR_PULL}[desc.direction]
    steps.dev_init(source, iters, desc.switch_ratio, policy)
    slots = max(lookahead, 1) + 1
    flags = torch.zeros((slots, 1), dtype=torch.int64, pin_memory=True)
    pending = []   # (slot, event) of enqueued levels, oldest first
    stream = torch.cuda.current_stream(steps.levels.device)
    for it in range(iters):
        steps.dev_level()
        exchange.dense(steps, g)
        steps.dev_apply()
        slot = it % slots
        flags[slot].copy_(steps.state[NativeSteps.STATE_DONE:NativeSteps.STATE_DONE + 1],
                          non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        pending.append((slot, ev))
        # deterministic: every rank waits on the same level, so all ranks stop
        # after the same number of collectives (an event query would let
        # them diverge)
        if len(pending) > lookahead:
            s0, e0 = pending.pop(0)
            e0.synchronize()
            if int(flags[s0, 0]):
                break
    torch.cuda.current_stream(steps.levels.device).synchronize()
    n_it = int(steps.state[NativeSteps.STATE_ITERS].item())
    raw = steps.log[:1 + 3 * n_it].cpu().numpy()
    for i in range(n_it):
        d, k, est = int(raw[1 + 3 * i]), int(raw[2 + 3 * i]), int(raw[3 + 3 * i])
        desc.direction_log.append(DirectionDecision("pull" if d == _lib.DIR_PULL else "push", k,
                                                    est, g.nnz, g.nnz * desc.switch_ratio))
    return steps.levels


def bfs_partitioned(g: BlockGraph, source: int, desc=None, steps=None, exchange=None):
    """algorithms.py:48-77 on a 1D-partitioned graph.  Returns (levels tensor,
    replicated on every rank, int64[n]) and appends the reference direction
    trace to ``desc.direction_log``."""
    if not 0 <= source < g.n:
        raise IndexError(f"source {source} out of range")
    desc = desc if desc is not None else Descriptor()
    steps = steps if steps is not None else NativeSteps(g)
    exchange = exchange if exchange is not None else FrontierExchange()
    iters = min(desc.max_niter, g.n + 1)
    steps.init(source)
    if iters <= 0:
        # the reference loop runs zero times: nothing is stamped, not even the source
        steps.unstamp(1)
        return steps.levels
    K, depth = 1, 1
    for it in range(iters):
        chosen, est, thr = direction_rule(g.nnz, g.n, K, desc.switch_ratio, desc.direction)
        desc.direction_log.append(DirectionDecision(chosen, K, est, g.nnz, thr))
        if chosen == "pull":
            steps.pull(depth + 1)
        else:
            steps.push(K)
        K = exchange(steps, g)
        steps.apply(depth + 1, K)
        if K == 0:
            break
        depth += 1
        if it + 1 == iters:
            steps.unstamp(K)  # the reference stamps a frontier at the next iteration
    return steps.levels


# ---------------------------------------------------------------------------
# connected components (FastSV, algorithms.py:165-203) on the 1D partition
# ---------------------------------------------------------------------------


class NativeCCSteps:
    """Per-rank FastSV steps (gb_cc_dist_*); int32 label vectors, replicated."""

    def __init__(self, g: BlockGraph):
        self.g = g
        self.ctx = _lib.context()
        self.rows, self._k1 = g._orient("row").csr_struct()
        self.cols, self._k2 = g._orient("col").csr_struct()
        dev = g.row_off.device

        def v():
            return torch.empty(g.n, dtype=torch.int32, device=dev)
        self.parent, self.mn, self.gp, self.gpp, self.pp, self.hook, self.prop = (
            v(), v(), v(), v(), v(), v(), v())

    def init(self):
        p = _lib.ptr
        self.ctx.call("gb_cc_dist_init", self.g.n, p(self.parent), p(self.mn), p(self.gp), p(self.gpp))

    def hook_and_propose(self, pull: bool):
        g, p = self.g, _lib.ptr
        self.ctx.call("gb_cc_dist_hook", 1 if pull else 0, C.byref(self.rows), C.byref(self.cols),
                      g.lo, g.hi, g.n, p(self.gp), p(self.parent), p(self.pp), p(self.hook))
        self.ctx.call("gb_cc_dist_propose", g.n, g.lo, g.hi, p(self.hook), p(self.mn), p(self.pp),
                      p(self.prop))

    def shortcut(self, sparsify: bool):
        p = _lib.ptr
        ch, lv = C.c_int64(0), C.c_int64(0)
        self.ctx.call("gb_cc_dist_shortcut", self.g.n, p(self.pp), p(self.prop), p(self.parent),
                      p(self.gp), p(self.gpp), 1 if sparsify else 0, C.byref(ch), C.byref(lv))
        return int(ch.value), int(lv.value)

    def result(self):
        out = torch.empty(self.g.n, dtype=torch.int64, device=self.parent.device)
        self.ctx.call("gb_widen_i32", self.g.n, _lib.ptr(self.parent), _lib.ptr(out))
        return out


class TorchMinExchange:
    """All-reduce MIN of the int32 parent proposals."""

    def __init__(self, group=None):
        self.group = group

    def allreduce_min(self, prop: torch.Tensor):
        import torch.distributed as dist
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(prop, op=dist.ReduceOp.MIN, group=self.group)


def cc_partitioned(g: BlockGraph, desc=None, sparsify=True, steps=None, exchange=None):
    """FastSV on a 1D-partitioned symmetric graph.  Per iteration: hook the
    owned vertices (pull over the row block / push over the column block, by
    the reference rule on the replicated live-grandparent count), propose
    parent minima, ONE all-reduce MIN of the proposals, then every rank applies
    them and shortcuts identically.  Returns the replicated int64 labels."""
    desc = desc if desc is not None else Descriptor()
    steps = steps if steps is not None else NativeCCSteps(g)
    exchange = exchange if exchange is not None else TorchMinExchange()
    steps.init()
    live = g.n
    for _ in range(desc.max_niter):
        chosen, est, thr = direction_rule(g.nnz, g.n, live, desc.switch_ratio, desc.direction)
        desc.direction_log.append(DirectionDecision(chosen, live, est, g.nnz, thr))
        steps.hook_and_propose(chosen == "pull")
        exchange.allreduce_min(steps.prop)
        changed, live = steps.shortcut(sparsify)
        if changed == 0:
            break
    return steps.result()


def connected_components(A_or_block, desc=None, sparsify=True, group=None):
    """Public entry: FastSV on this rank's block; returns the replicated label Vector."""
    g = A_or_block
    if isinstance(A_or_block, SparseMatrix):
        import torch.distributed as dist
        if not A_or_block.is_symmetric():
            raise ValueError("adjacency matrix must be symmetric (undirected graph)")
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        g = BlockGraph.from_matrix(A_or_block, rank, world)
    labels = cc_partitioned(g, desc, sparsify, exchange=TorchMinExchange(group))
    return Vector._wrap(g.n, None, labels, np.iinfo(np.int64).max, np.int64)


class OrderedPartitionedBfs:
    """The partitioned BFS over the degree-ordered layout of A (as the
    single-GPU bfs uses it): vertices renumbered by descending degree
    (SparseMatrix.traversal), edge-balanced blocks of NEW ids -- rank 0 owns
    the hubs, and every rank's probes fall in its own slice of the bitmap --
    the source mapped in, the replicated levels gathered back to the original
    ids at the end (gb_gather).  Levels and the direction log equal bfs(A)."""

    def __init__(self, A: SparseMatrix, rank: int, world: int, group=None, bounds=None,
                 loop: str = "device"):
        if loop not in ("device", "host"):
            raise ValueError("loop is 'device' (bfs_partitioned_device) or 'host' (bfs_partitioned)")
        self.loop = loop
        push_o, pull_o, self.rank_t = A.traversal()
        Ar = SparseMatrix._wrap(A.nrows, A.ncols, push_o, pull_o, A.dtype, A._sym)
        self.block = BlockGraph.from_matrix(Ar, rank, world, bounds)
        self.steps = NativeSteps(self.block)
        self.steps.prefix_cut = True   # traversal() relabels with sorted rows
        self.exchange = FrontierExchange(group)
        self.rank64 = A._rank64()
        self.out = torch.empty(A.nrows, dtype=torch.int64, device=push_o.offsets.device)

    def __call__(self, source: int, desc=None):
        if not 0 <= source < self.block.n:
            raise IndexError(f"source {source} out of range")
        src = int(self.rank_t[source].item())
        run = bfs_partitioned_device if self.loop == "device" else bfs_partitioned
        lv = run(self.block, src, desc, steps=self.steps, exchange=self.exchange)
        n = self.block.n
        _lib.context().call("gb_gather", _lib.dtype_code(np.int64), n, _lib.ptr(self.rank64), n,
                            _lib.ptr(lv), _lib.ptr(self.out))
        return self.out


def bfs(A_or_block, source, desc=None, group=None, ordered=True, loop="device"):
    """Public entry: bfs on this rank's block; returns the (replicated) level Vector.
    A SparseMatrix with a column orientation is partitioned over its
    degree-ordered layout unless ``ordered=False``.  ``loop="device"`` keeps
    the level loop's scalars on the device (dense exchange every level, no
    host read per level); ``loop="host"`` is the count-driven loop with the
    dense / sparse exchange."""
    g = A_or_block
    if isinstance(A_or_block, SparseMatrix):
        import torch.distributed as dist
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        if ordered and A_or_block.traversal() is not None:
            run = OrderedPartitionedBfs(A_or_block, rank, world, group, loop=loop)
            return Vector._wrap(A_or_block.nrows, None, run(source, desc).clone(), 0, np.int64)
        g = BlockGraph.from_matrix(A_or_block, rank, world)
    run = bfs_partitioned_device if loop == "device" else bfs_partitioned
    levels = run(g, source, desc, exchange=FrontierExchange(group))
    return Vector._wrap(g.n, None, levels, 0, np.int64)
