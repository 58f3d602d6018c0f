"""Descriptor(count_work=True): the fused algorithms fill desc.counters with
exactly the reference's tallies -- equal to the operator composition
(fused=False), whose counters are pinned to the reference's kernel cases in
test_gpu_kernels.py.  BFS counts are recomputed on the device from the
levels and the direction log (gb_bfs_counters), PageRank's from the log."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gb():
    import paper_1908_01407_b200 as gb
    return gb


def _counts(d):
    c = d.counters
    return (c.matrix_entries_read, c.semiring_multiplies, c.semiring_adds)


def _pair(gb, fn, **kw):
    fused = gb.Descriptor(count_work=True, **kw)
    composed = gb.Descriptor(fused=False, **kw)
    a = fn(fused)
    b = fn(composed)
    return a, b, _counts(fused), _counts(composed), fused, composed


@pytest.mark.parametrize("scale,a", [(10, .57), (14, .57), (16, .57), (12, .25)])
@pytest.mark.parametrize("src", [0, 3])
@pytest.mark.parametrize("early", [True, False])
def test_bfs_counters_equal_composition(gb, scale, a, src, early):
    b = c = .19 if a == .57 else .25
    A = gb.io.rmat_matrix(scale, a=a, b=b, c=c, d=1 - a - b - c)
    x, y, cf, cc, df, dc = _pair(gb, lambda d: gb.bfs(A, src, desc=d, early_exit=early))
    assert np.array_equal(x.values, y.values)
    assert cf == cc and cf[1] > 0
    assert [(q.chosen, q.frontier_nvals) for q in df.direction_log] == \
        [(q.chosen, q.frontier_nvals) for q in dc.direction_log]


@pytest.mark.parametrize("policy", ["FORCE_PUSH", "FORCE_PULL"])
def test_bfs_counters_forced_directions(gb, policy):
    A = gb.io.rmat_matrix(12)
    direction = getattr(gb.Direction, policy)
    x, y, cf, cc, _, _ = _pair(gb, lambda d: gb.bfs(A, 0, desc=d), direction=direction)
    assert np.array_equal(x.values, y.values) and cf == cc


def test_bfs_counters_capped_and_directed(gb):
    A = gb.io.rmat_matrix(12)
    _x, _y, cf, cc, _, _ = _pair(gb, lambda d: gb.bfs(A, 0, desc=d), max_niter=2)
    assert cf == cc
    rng = np.random.default_rng(3)
    n = 3000
    r, c = rng.integers(0, n, 20000), rng.integers(0, n, 20000)
    D = gb.SparseMatrix.from_tuples(r, c, np.ones(r.size, np.int64), n, n)
    x, y, cf, cc, _, _ = _pair(gb, lambda d: gb.bfs(D, 1, desc=d))
    assert np.array_equal(x.values, y.values) and cf == cc


def test_pagerank_sssp_cc_tc_counters(gb):
    A = gb.io.rmat_matrix(11)
    W = gb.io.rmat_matrix(11, weighted=True)
    _x, _y, cf, cc, _, _ = _pair(gb, lambda d: gb.pagerank(A, eps=1e-300, max_iters=7, desc=d))
    assert cf == cc and cf[0] > 0
    for fn in (lambda d: gb.sssp(W, 0, desc=d), lambda d: gb.connected_components(A, desc=d),
               lambda d: gb.triangle_count(A, desc=d)):
        _x, _y, cf, cc, _, _ = _pair(gb, fn)
        assert cf == cc and cf[1] > 0
    # without count_work the fused drivers leave the counters untouched
    d = gb.Descriptor()
    gb.bfs(A, 0, desc=d)
    assert _counts(d) == (0, 0, 0)
