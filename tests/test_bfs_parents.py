"""BFS parents (the north star's "levels/parents-validity" extension; the
reference returns levels only, algorithms.py:66-77).

CPU: the C oracle's min-id parent rule checked against a plain-Python
restatement of the Graph500 tree conditions.  GPU: bfs_parents equals the
oracle bit for bit (R-MAT s10-s20, uniform, directed) and validate_bfs
accepts it and counts every kind of corruption."""

import numpy as np
import pytest

from oracle import cgraph


def _py_parents(rp, ci, lv, source):
    n = rp.size - 1
    par = np.full(n, -1, np.int64)
    for v in range(n):
        if lv[v] == 0:
            continue
        if v == source:
            par[v] = source
            continue
        nb = ci[rp[v]:rp[v + 1]]
        cand = nb[lv[nb] == lv[v] - 1]
        par[v] = cand.min() if cand.size else -2
    return par


@pytest.mark.parametrize("scale", [8, 10])
def test_oracle_parents_match_python_rule(scale):
    rp, ci = cgraph.rmat_csr(scale)
    for src in (0, 5):
        lv, _ = cgraph.bfs(rp, ci, src)
        par = cgraph.bfs_parents(rp, ci, lv, src)
        assert np.array_equal(par, _py_parents(rp, ci, lv, src))
        reached = lv > 0
        assert (par[reached] >= 0).all() and (par[~reached] == -1).all()


def _digest(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, np.int64).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def gb():
    import paper_1908_01407_b200 as gb
    return gb


@pytest.mark.gpu
@pytest.mark.parametrize("scale,a", [(10, .57), (14, .57), (20, .57), (12, .25), (16, .25)])
def test_gpu_parents_equal_oracle_and_validate(gb, scale, a):
    b = c = .19 if a == .57 else .25
    d = 1 - a - b - c
    A = gb.io.rmat_matrix(scale, a=a, b=b, c=c, d=d)
    rp, ci = A._csr.offsets.cpu().numpy(), A._csr.indices.cpu().numpy()
    for src in (0, 3):
        lv, par = gb.bfs_parents(A, src)
        want_lv, _ = cgraph.bfs(rp, ci, src)
        assert np.array_equal(lv.values, want_lv)
        want = cgraph.bfs_parents(rp, ci, want_lv, src)
        assert _digest(par.values) == _digest(want)
        v = gb.validate_bfs(A, src, lv, par)
        assert v["ok"], v


@pytest.mark.gpu
def test_gpu_parents_directed(gb):
    rng = np.random.default_rng(4)
    n = 2000
    r = rng.integers(0, n, 12000)
    c = rng.integers(0, n, 12000)
    A = gb.SparseMatrix.from_tuples(r, c, np.ones(r.size, np.int64), n, n)
    lv, par = gb.bfs_parents(A, 7)
    rp, ci = A._csr.offsets.cpu().numpy(), A._csr.indices.cpu().numpy()
    cp, ri = A._csc.offsets.cpu().numpy(), A._csc.indices.cpu().numpy()
    want_lv, _ = cgraph.bfs(rp, ci, 7, cp=cp, ri=ri)
    assert np.array_equal(lv.values, want_lv)
    assert np.array_equal(par.values, cgraph.bfs_parents(rp, ci, want_lv, 7, cp=cp, ri=ri))
    assert gb.validate_bfs(A, 7, lv, par)["ok"]


@pytest.mark.gpu
def test_gpu_validator_counts_corruption(gb):
    import torch
    A = gb.io.rmat_matrix(12)
    lv, par = gb.bfs_parents(A, 0)
    L, P = lv._vals.clone(), par._vals.clone()
    reached = torch.nonzero(L >= 3).flatten()   # a level-2 vertex's only candidate is the source
    v = int(reached[5])
    # a non-adjacent parent one level up
    P2 = P.clone()
    lvl = int(L[v])
    others = torch.nonzero(L == lvl - 1).flatten()
    rp, ci = A._csr.offsets.cpu().numpy(), A._csr.indices.cpu().numpy()
    nb = set(ci[rp[v]:rp[v + 1]].tolist())
    bad = next(int(u) for u in others.tolist() if int(u) not in nb)
    P2[v] = bad
    assert gb.validate_bfs(A, 0, L, P2)["tree_edges"] == 1
    # a wrong level breaks the tree edge and the graph-edge layering
    L2 = L.clone()
    L2[v] += 2
    r = gb.validate_bfs(A, 0, L2, P)
    assert r["tree_edges"] >= 1 and r["graph_edges"] >= 1 and not r["ok"]
    # source and unreached conditions
    P3 = P.clone()
    P3[0] = 1
    unreached = torch.nonzero(L == 0).flatten()
    if unreached.numel():
        P3[int(unreached[0])] = 0
    r = gb.validate_bfs(A, 0, L, P3)
    assert r["source"] == 1 and r["unreached"] == (1 if unreached.numel() else 0)
