"""Multi-rank host logic of the 1D-partitioned BFS, on CPU with gloo.

The partition, the level loop, the reference direction rule on global
counts, the frontier exchange (allgather of the owned counts, then a dense
allgather of the owned bitmap words or an allgather(v) of the owned ids) and
the loop-cap handling are the product code (paper_1908_01407_b200.distributed).
The per-rank level steps -- CUDA kernels in the product -- are replaced here
by a numpy restatement with the same contract, so world_size-2 runs execute
on this CPU-only box.  Results must equal the single-process oracle BFS.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port
from paper_1908_01407_b200.distributed import (ALIGN, FrontierExchange, bfs_partitioned,
                                               partition_bounds)


def test_partition_bounds_properties():
    rng = np.random.default_rng(0)
    for _ in range(50):
        n = int(rng.integers(1, 20000))
        deg = rng.integers(0, 50, size=n)
        deg[:5] *= 100  # hubs at low ids, like R-MAT
        off = np.r_[0, np.cumsum(deg)]
        for P in (1, 2, 3, 4, 8):
            b = partition_bounds(off, P)
            assert b[0] == 0 and b[-1] == n and len(b) == P + 1
            assert all(x <= y for x, y in zip(b, b[1:]))
            assert all(x % ALIGN == 0 for x in b[:-1])
    # balance on a large uniform graph: every block within one alignment unit
    off = np.arange(0, 1 << 20, dtype=np.int64) * 16
    b = partition_bounds(off, 8)
    sizes = np.diff([off[x] for x in b])
    assert sizes.max() - sizes.min() <= 16 * ALIGN


class Block:
    """Numpy stand-in for BlockGraph (same fields the loop reads)."""

    def __init__(self, rp, ci, lo, hi, bounds=None):
        self.n = rp.size - 1
        self.nnz = int(rp[-1])
        self.lo, self.hi = lo, hi
        self.bounds = bounds
        self.rp, self.ci = rp, ci   # symmetric: in-edges == out-edges


class NumpySteps:
    """Same contract as NativeSteps (gb_bfs_dist_*), restated in numpy."""

    def __init__(self, g):
        self.g = g
        n = g.n
        W = (n + 31) // 32
        self.levels = np.zeros(n, np.int64)
        self.vbm = np.zeros(W, np.uint32)
        self.vprev = np.zeros(W, np.uint32)
        self.fbm = np.zeros(W, np.uint32)
        self.xbm = torch.zeros(W, dtype=torch.int32)
        self.F = np.zeros(0, np.int64)

    @staticmethod
    def _set(bm, v):
        bm[v >> 5] |= np.uint32(1) << np.uint32(v & 31)

    @staticmethod
    def _get(bm, v):
        return (int(bm[v >> 5]) >> (v & 31)) & 1

    def _x(self):
        return self.xbm.numpy().view(np.uint32)

    def init(self, s):
        self.levels[s] = 1
        for bm in (self.vbm, self.vprev, self.fbm):
            self._set(bm, s)
        self.F = np.array([s])

    def push(self, K):
        g = self.g
        for u in self.F[:K]:
            for v in g.ci[g.rp[u]:g.rp[u + 1]]:
                if g.lo <= v < g.hi and not self._get(self.vbm, v):
                    self._set(self.vbm, v)
        x = self._x()
        x[:] = 0
        wl, wh = g.lo // 32, (g.hi + 31) // 32
        x[wl:wh] = self.vbm[wl:wh] & ~self.vprev[wl:wh]

    def pull(self, depth):
        g = self.g
        x = self._x()
        x[:] = 0
        for v in range(g.lo, g.hi):
            if self._get(self.vbm, v):
                continue
            nb = g.ci[g.rp[v]:g.rp[v + 1]]
            if any(self._get(self.fbm, int(j)) for j in nb):
                for bm in (self.vbm, self.vprev, x):
                    self._set(bm, v)
                self.levels[v] = depth

    def apply(self, depth, K=None):
        x = self._x().copy()
        self.vbm |= x
        self.vprev |= x
        self.fbm[:] = x
        bits = np.unpackbits(x.view(np.uint8), bitorder="little")[: self.g.n]
        F = np.flatnonzero(bits)
        self.levels[F] = depth
        self.F = F
        assert K is None or K == F.size
        return int(F.size)

    # frontier exchange steps (gb_bfs_dist_owned / pack / unpack / set_ids)
    def owned(self):
        g = self.g
        x = self._x()
        wl, wh = g.lo // 32, (g.hi + 31) // 32
        bits = np.unpackbits(x[wl:wh].view(np.uint8), bitorder="little")
        self.ids = (np.flatnonzero(bits) + wl * 32).astype(np.int32)
        return torch.tensor([self.ids.size], dtype=torch.int64)

    def pack_words(self, wmax):
        g = self.g
        wl, wh = g.lo // 32, (g.hi + 31) // 32
        out = np.zeros(wmax, np.uint32)
        out[: wh - wl] = self._x()[wl:wh]
        return torch.from_numpy(out.view(np.int32))

    def unpack_words(self, gathered, wmax, wb):
        x = self._x()
        gw = gathered.numpy().view(np.uint32)
        wb = wb.numpy()
        for p in range(wb.size - 1):
            x[wb[p]:wb[p + 1]] = gw[p * wmax: p * wmax + wb[p + 1] - wb[p]]

    def owned_ids(self, kmax):
        out = np.zeros(kmax, np.int32)
        out[: self.ids.size] = self.ids
        return torch.from_numpy(out)

    def set_ids(self, gathered, counts, kmax):
        x = self._x()
        x[:] = 0
        g = gathered.numpy()
        for p, c in enumerate(counts.tolist()):
            for v in g[p * kmax: p * kmax + c]:
                self._set(x, int(v))

    def unstamp(self, K):
        self.levels[self.F[:K]] = 0


class NumpyCCSteps:
    """Same contract as NativeCCSteps (gb_cc_dist_*), restated in numpy."""

    MAX = np.iinfo(np.int32).max

    def __init__(self, g):
        self.g = g
        n = g.n
        self.parent = np.arange(n, dtype=np.int64)
        self.mn = self.parent.copy()
        self.gp = self.parent.copy()
        self.gpp = self.parent.copy()
        self.pp = self.parent.copy()
        self.prop = torch.full((n,), self.MAX, dtype=torch.int32)

    def init(self):
        pass

    def hook_and_propose(self, pull):
        g, M = self.g, self.MAX
        self.pp = self.parent.copy()
        hook = np.full(g.n, M, np.int64)
        if pull:
            for i in range(g.lo, g.hi):
                nb = self.gp[g.ci[g.rp[i]:g.rp[i + 1]]]
                nb = nb[nb != M]
                if nb.size:
                    hook[i] = nb.min()
        else:
            for j in np.flatnonzero(self.gp != M):
                for i in g.ci[g.rp[j]:g.rp[j + 1]]:
                    if g.lo <= i < g.hi:
                        hook[i] = min(hook[i], self.gp[j])
        prop = np.full(g.n, M, np.int64)
        for k in range(g.lo, g.hi):
            m = min(self.mn[k], hook[k])
            self.mn[k] = m
            prop[k] = min(prop[k], m)
            prop[self.pp[k]] = min(prop[self.pp[k]], m)
        self.prop[:] = torch.from_numpy(prop.astype(np.int32))

    def shortcut(self, sparsify):
        self.parent = np.minimum(self.pp, self.prop.numpy().astype(np.int64))
        g = self.parent[self.parent]
        changed = g != self.gpp
        self.gpp = g.copy()
        self.gp = np.where(changed | (not sparsify), g, self.MAX)
        return int(changed.sum()), int((self.gp != self.MAX).sum())

    def result(self):
        return self.parent.copy()


def _cc_worker(rank, world, port_, scale, sparsify, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1908_01407_b200.containers import Descriptor
    from paper_1908_01407_b200.distributed import TorchMinExchange, cc_partitioned
    rp, ci, n = port.rmat_csr(scale)
    bounds = partition_bounds(rp, world)
    g = Block(rp, ci, bounds[rank], bounds[rank + 1])
    desc = Descriptor()
    labels = cc_partitioned(g, desc, sparsify, steps=NumpyCCSteps(g), exchange=TorchMinExchange())
    results[rank] = (labels, [(d.chosen, d.frontier_nvals) for d in desc.direction_log])
    dist.destroy_process_group()


@pytest.mark.parametrize("scale,sparsify", [(10, True), (11, False)])
def test_partitioned_cc_world2_matches_oracle(scale, sparsify):
    ctx = mp.get_context("spawn")
    results = ctx.Manager().dict()
    port_ = _free_port()
    procs = [ctx.Process(target=_cc_worker, args=(r, 2, port_, scale, sparsify, results))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    rp, ci, n = port.rmat_csr(scale)
    P = port.mat_from_csr(rp, ci, np.ones(ci.size, np.int64), n)
    pd = port.Desc()
    want = port.connected_components(P, pd, sparsify=sparsify)
    for r in range(2):
        labels, trace = results[r]
        assert np.array_equal(labels, want.vals)
        assert trace == [(x[0], x[1]) for x in pd.log]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port_, scale, source, cap, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rp, ci, n = port.rmat_csr(scale)
    bounds = partition_bounds(rp, world)
    g = Block(rp, ci, bounds[rank], bounds[rank + 1], bounds)
    from paper_1908_01407_b200.containers import Descriptor
    desc = Descriptor(max_niter=cap)
    ex = FrontierExchange()
    levels = bfs_partitioned(g, source, desc, steps=NumpySteps(g), exchange=ex)
    results[rank] = (levels.copy(), [(d.chosen, d.frontier_nvals, d.estimated_frontier_edges)
                                     for d in desc.direction_log], list(ex.log))
    dist.destroy_process_group()


@pytest.mark.parametrize("scale,source,cap", [(10, 0, 10_000), (11, 5, 10_000), (10, 0, 2), (10, 0, 0)])
def test_partitioned_bfs_world2_matches_oracle(scale, source, cap):
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    results = manager.dict()
    port_ = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_, scale, source, cap, results))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    rp, ci, n = port.rmat_csr(scale)
    P = port.mat_from_csr(rp, ci, np.ones(ci.size, np.int64), n)
    pd = port.Desc(max_niter=cap)
    want = port.bfs(P, source, pd)
    for r in range(2):
        levels, trace, xlog = results[r]
        assert np.array_equal(levels, want.vals)
        assert [t[0] for t in trace] == [x[0] for x in pd.log]
        assert [t[1:] for t in trace] == [tuple(x[1:3]) for x in pd.log]
        # the exchange mode follows |f|*32 > n on the NEXT frontier size
        sizes = [x[1] for x in pd.log[1:]]
        assert [m for m, _b in xlog[:len(sizes)]] == ["dense" if k * 32 > n else "sparse"
                                                     for k in sizes]
    if cap > 2:
        assert {"dense", "sparse"} <= {m for m, _b in results[0][2]}
