"""Pin the C oracle (oracle/cgraph.c) to the reference's own outputs at the
BASELINE scales.  CPU only.

cgraph is the checker for every GPU comparison at s16 and above (C2, C3, C5,
the uniform row) and the timing arm of ``bench.py --impl reference``, so it
must reproduce what the reference package computed on the same inputs:

* ``algorithms.json`` / ``algorithms_big.json`` -- BFS (two sources, s8-s20),
  SSSP / CC / TC / PageRank (s8-s20) digests, traces and counts, written by
  ``tests/golden/make_golden.py`` running graphalg itself;
* ``pins.json`` -- reference weight digests at s16/s18/s20 (io.py:252-272),
  the non-integral SSSP variant (sqrt of the weights) at s16/s20, every one of
  the 20 PageRank iterates at s16/s20 (sum, sum of squares, L2 step error and
  256 sampled ranks), and the uniform family at s14/s16;
* SURVEY.md §8(c) digests of the reference at s22 (BFS, CC, PageRank Σp),
  measured with the reference's algorithms on its own CSR.
"""

import hashlib

import numpy as np
import pytest

from golden_io import load_json
from oracle import cgraph

UNIFORM = dict(a=0.25, b=0.25, c=0.25)

# SURVEY.md §8(c) "What is not pinned by the reference tests" (reference run at s22)
S22_BFS = "2ee717d6a34a1fef9477299ae5cea7e52f4ed4e701305bd4042c3c86875df934"
S22_CC = "337b66f151ed772991d59671f7841f648ec258867d4b38eeb22e8d7120a8e75d"
S22_PR_SUM = 0.635613537
INT_INF = np.iinfo(np.int64).max  # the Minimum identity: CC labels are stored dense with this zero


def digest_dense(values, zero):
    """cli.py:148-156 on a dense vector (extract_tuples drops entries == zero)."""
    values = np.asarray(values)
    idx = np.flatnonzero(values != zero).astype(np.int64)
    h = hashlib.sha256()
    h.update(idx.tobytes())
    h.update(np.ascontiguousarray(np.round(values[idx].astype(np.float64), 9)).tobytes())
    return h.hexdigest()


def wdigest(w):
    return hashlib.sha256(np.ascontiguousarray(w, np.float64).tobytes()).hexdigest()


def same_trace(tr, gold):
    return [list(t[:3]) for t in tr] == [g[:3] for g in gold]


_GRAPHS = {}


def graph(s, uniform=False):
    key = (s, uniform)
    if key not in _GRAPHS:
        _GRAPHS.clear()
        _GRAPHS[key] = cgraph.rmat_csr(s, **(UNIFORM if uniform else {}))
    return _GRAPHS[key]


def gold(name, key):
    return load_json(name)[key]


BFS_KEYS = [(s, k) for s in (8, 10, 12, 14, 16, 18, 20)
            for k in load_json("algorithms_big.json") if k == f"bfs_s{s}" or k.startswith(f"bfs_s{s}_src")]


@pytest.mark.parametrize("s,key", BFS_KEYS)
def test_cgraph_bfs_matches_reference(s, key):
    g = gold("algorithms_big.json", key)
    rp, ci = graph(s)
    lv, tr = cgraph.bfs(rp, ci, g.get("source", 0))
    assert digest_dense(lv, 0) == g["digest"]
    assert same_trace(tr, g["trace"])


@pytest.mark.parametrize("s", [8, 10, 12, 14, 16, 20])
def test_cgraph_sssp_cc_tc_pr_match_reference(s):
    big = gold("algorithms_big.json", f"sssp_s{s}")
    rp, ci = graph(s)
    w = cgraph.upper_weights(rp, ci)
    dist, tr = cgraph.sssp(rp, ci, w, 0)
    assert digest_dense(dist, np.inf) == big["digest"]
    assert same_trace(tr, big["trace"])
    assert int(np.isfinite(dist).sum()) == big["finite"]
    par, tr = cgraph.cc(rp, ci)
    g = gold("algorithms_big.json", f"cc_s{s}")
    assert digest_dense(par, INT_INF) == g["digest"]
    assert same_trace(tr, g["trace"])
    assert np.unique(par).size == g["components"]
    assert cgraph.tc(rp, ci) == gold("algorithms_big.json", f"tc_s{s}")["count"]
    ranks, _ = cgraph.pagerank(rp, ci, eps=1e-300, max_iters=20)
    g = gold("algorithms_big.json", f"pr_s{s}")
    assert abs(ranks.sum() - g["sum"]) <= 1e-12
    assert digest_dense(ranks, 0.0) == g["digest9"]
    rd, _ = cgraph.pagerank(rp, ci)
    assert abs(rd.sum() - g["sum_default"]) <= 1e-12


@pytest.mark.parametrize("s", [16, 18, 20])
def test_cgraph_weights_match_reference(s):
    g = gold("pins.json", f"weights_rmat_s{s}")
    rp, ci = graph(s)
    w = cgraph.upper_weights(rp, ci)
    assert w.size == g["nnz"]
    assert wdigest(w) == g["digest"]


@pytest.mark.parametrize("s", [16, 20])
def test_cgraph_sssp_non_integral_weights(s):
    """C2's non-integral variant: the same CSR with sqrt weights on both sides."""
    g = gold("pins.json", f"sssp_sqrt_s{s}")
    rp, ci = graph(s)
    w = np.sqrt(cgraph.upper_weights(rp, ci))
    dist, tr = cgraph.sssp(rp, ci, w, 0)
    fin = np.isfinite(dist)
    assert int(fin.sum()) == g["finite"]
    assert abs(dist[fin].sum() - g["sum_finite"]) <= 1e-9 * g["sum_finite"]
    ids = np.asarray(g["sample_ids"])
    want = np.array([np.inf if x is None else x for x in g["samples"]])
    assert np.array_equal(np.isinf(dist[ids]), np.isinf(want))
    f = ~np.isinf(want)
    assert np.allclose(dist[ids][f], want[f], rtol=1e-12, atol=0)
    assert same_trace(tr, g["trace"])
    assert digest_dense(dist, np.inf) == g["digest"]


@pytest.mark.parametrize("s", [16, 20])
def test_cgraph_pagerank_every_iteration(s):
    """C3's gate restated at the pinned scales: each of the 20 iterates."""
    g = gold("pins.json", f"pr_iter_s{s}")
    rp, ci = graph(s)
    ids = np.asarray(g["sample_ids"])
    for k, rec in enumerate(g["iterations"], start=1):
        r, errs = cgraph.pagerank(rp, ci, eps=1e-300, max_iters=k)
        assert errs.size == k
        assert abs(r.sum() - rec["sum"]) <= 1e-12, k
        assert abs(np.dot(r, r) - rec["sumsq"]) <= 1e-12 * rec["sumsq"], k
        assert abs(errs[-1] - rec["error"]) <= 1e-9 * rec["error"], k
        assert np.allclose(r[ids], rec["samples"], rtol=1e-12, atol=0), k
        assert digest_dense(r, 0.0) == rec["digest9"], k


@pytest.mark.parametrize("s", [14, 16])
def test_cgraph_uniform_family(s):
    g = gold("pins.json", f"uniform_s{s}")
    rp, ci = graph(s, uniform=True)
    assert ci.size == g["nnz"]
    h = hashlib.sha256()
    h.update(rp.astype(np.int64).tobytes())
    h.update(ci.astype(np.int64).tobytes())
    assert h.hexdigest() == g["csr"]
    w = cgraph.upper_weights(rp, ci)
    assert wdigest(w) == g["weights"]
    lv, tr = cgraph.bfs(rp, ci, 0)
    assert digest_dense(lv, 0) == g["bfs"]["digest"]
    assert same_trace(tr, g["bfs"]["trace"])
    par, tr = cgraph.cc(rp, ci)
    assert digest_dense(par, INT_INF) == g["cc"]["digest"]
    assert same_trace(tr, g["cc"]["trace"])
    dist, _ = cgraph.sssp(rp, ci, w, 0)
    assert digest_dense(dist, np.inf) == g["sssp"]["digest"]
    assert cgraph.tc(rp, ci) == g["tc"]


def test_cgraph_s22_against_survey_digests():
    rp, ci = graph(22)
    lv, _ = cgraph.bfs(rp, ci, 0)
    assert digest_dense(lv, 0) == S22_BFS
    par, _ = cgraph.cc(rp, ci)
    assert digest_dense(par, INT_INF) == S22_CC
    r, _ = cgraph.pagerank(rp, ci, eps=1e-300, max_iters=20)
    assert abs(r.sum() - S22_PR_SUM) <= 5e-10
