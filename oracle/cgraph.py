"""ctypes loader for oracle/cgraph.c (TEST ORACLE / CPU BASELINE ONLY).

Build: ``make -C oracle`` (or ``__graft_entry__.build()``) -> oracle/build/libcgraph.so.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "libcgraph.so")

_lib = None

vp, i64, i32, f64, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_uint64


def build():
    subprocess.check_call(["make", "-s", "-C", HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = C.CDLL(LIB)
        L.og_threads.restype = C.c_int
        L.og_set_threads.argtypes = [C.c_int]
        L.og_rmat_edges.argtypes = [C.c_int, i64, u64, f64, f64, f64, vp, vp]
        L.og_rmat_csr.restype = i64
        L.og_rmat_csr.argtypes = [C.c_int, i64, u64, f64, f64, f64, vp, vp]
        L.og_bfs.restype = i64
        L.og_bfs.argtypes = [i64, vp, vp, vp, vp, i64, i64, f64, C.c_int, vp, vp, vp, vp]
        L.og_sssp.restype = i64
        L.og_sssp.argtypes = [i64, vp, vp, vp, vp, vp, vp, i64, i64, f64, C.c_int, vp, vp, vp, vp]
        L.og_pagerank.restype = i64
        L.og_pagerank.argtypes = [i64, vp, vp, vp, f64, f64, i64, vp, vp]
        L.og_cc.restype = i64
        L.og_cc.argtypes = [i64, vp, vp, vp, vp, i64, f64, C.c_int, C.c_int, vp, vp, vp, vp]
        L.og_upper_weights.restype = i64
        L.og_upper_weights.argtypes = [i64, vp, vp, u64, i64, i64, vp]
        L.og_bfs_parents.restype = i64
        L.og_bfs_parents.argtypes = [i64, vp, vp, vp, i64, vp]
        L.og_tc.restype = i64
        L.og_tc.argtypes = [i64, vp, vp]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(vp)


def _csr(rp, ci):
    return np.ascontiguousarray(rp, np.int64), np.ascontiguousarray(ci, np.int32)


def set_threads(t):
    lib().og_set_threads(int(t))


def threads():
    return int(lib().og_threads())


def rmat_edges(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1):
    m = edge_factor << scale
    src = np.empty(m, np.int32)
    dst = np.empty(m, np.int32)
    tab = a + b
    lib().og_rmat_edges(scale, m, seed, a, tab, tab + c, _p(src), _p(dst))
    return src, dst


def rmat_csr(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1):
    """(row_offsets int64, col_indices int32) of the preprocessed R-MAT graph."""
    m = edge_factor << scale
    n = 1 << scale
    rp = np.empty(n + 1, np.int64)
    ci = np.empty(2 * m, np.int32)
    tab = a + b
    nnz = lib().og_rmat_csr(scale, m, seed, a, tab, tab + c, _p(rp), _p(ci))
    return rp, ci[:nnz].copy()


def upper_weights(rp, ci, seed=1, low=1, high=64):
    """io.py:252-272 on a symmetric sorted CSR: float64 weights per stored entry."""
    rp, ci = _csr(rp, ci)
    w = np.empty(ci.size, np.float64)
    if lib().og_upper_weights(rp.size - 1, _p(rp), _p(ci), seed, low, high, _p(w)) != 0:
        raise ValueError("CSR is not symmetric / has self loops")
    return w


def _log(cap):
    return np.zeros(cap, np.int32), np.zeros(cap, np.int64), np.zeros(cap, np.int64)


def _trace(d, nv, est, k):
    return [("pull" if d[i] == 2 else "push", int(nv[i]), int(est[i])) for i in range(k)]


def bfs(rp, ci, source=0, cp=None, ri=None, max_iters=None, ratio=0.1, policy=0):
    """(levels int64[n], trace) -- symmetric graphs may omit cp/ri (CSC = CSR)."""
    rp, ci = _csr(rp, ci)
    cp, ri = (rp, ci) if cp is None else _csr(cp, ri)
    n = rp.size - 1
    iters = min(n + 1, 10_000) if max_iters is None else max_iters
    lv = np.empty(n, np.int64)
    d, nv, est = _log(iters)
    k = lib().og_bfs(n, _p(rp), _p(ci), _p(cp), _p(ri), source, iters, ratio, policy, _p(lv),
                     _p(d), _p(nv), _p(est))
    return lv, _trace(d, nv, est, k)


def bfs_parents(rp, ci, levels, source=0, cp=None, ri=None):
    """Min-id BFS parents derived from a level vector (og_bfs_parents)."""
    rp, ci = _csr(rp, ci)
    cp, ri = (rp, ci) if cp is None else _csr(cp, ri)
    lv = np.ascontiguousarray(levels, np.int64)
    par = np.empty(lv.size, np.int64)
    bad = lib().og_bfs_parents(lv.size, _p(cp), _p(ri), _p(lv), int(source), _p(par))
    assert bad == 0, "level vector is not a BFS layering"
    return par


def sssp(rp, ci, w, source=0, cp=None, ri=None, wt=None, ratio=0.1, policy=0):
    rp, ci = _csr(rp, ci)
    w = np.ascontiguousarray(w, np.float64)
    if cp is None:
        cp, ri, wt = rp, ci, w
    else:
        cp, ri = _csr(cp, ri)
        wt = np.ascontiguousarray(wt, np.float64)
    n = rp.size - 1
    iters = min(n, 10_000)
    dist = np.empty(n, np.float64)
    d, nv, est = _log(iters)
    k = lib().og_sssp(n, _p(rp), _p(ci), _p(w), _p(cp), _p(ri), _p(wt), source, iters, ratio,
                      policy, _p(dist), _p(d), _p(nv), _p(est))
    return dist, _trace(d, nv, est, k)


def pagerank(rp, ci, alpha=0.85, eps=1e-7, max_iters=10_000, cp=None, ri=None):
    rp, ci = _csr(rp, ci)
    cp, ri = (rp, ci) if cp is None else _csr(cp, ri)
    n = rp.size - 1
    r = np.empty(n, np.float64)
    errs = np.zeros(max(max_iters, 1), np.float64)
    k = lib().og_pagerank(n, _p(rp), _p(cp), _p(ri), alpha, eps, max_iters, _p(r), _p(errs))
    return r, errs[:k]


def cc(rp, ci, cp=None, ri=None, sparsify=True, ratio=0.1, policy=0, max_iters=10_000):
    rp, ci = _csr(rp, ci)
    cp, ri = (rp, ci) if cp is None else _csr(cp, ri)
    n = rp.size - 1
    parent = np.empty(n, np.int64)
    d, nv, est = _log(max_iters)
    k = lib().og_cc(n, _p(rp), _p(ci), _p(cp), _p(ri), max_iters, ratio, policy,
                    1 if sparsify else 0, _p(parent), _p(d), _p(nv), _p(est))
    return parent, _trace(d, nv, est, k)


def tc(rp, ci):
    rp, ci = _csr(rp, ci)
    return int(lib().og_tc(rp.size - 1, _p(rp), _p(ci)))
