"""The device-resident SSSP / PageRank / CC loops (one CUDA-graph launch per
call: WHILE node, device-side direction rule and exit test, SWITCH pull |
push) against the host-driven loop of the same kernels (gb_loop_engine(1)),
itself pinned to the reference goldens and the C oracle elsewhere: identical
results, direction logs, iteration counts and PageRank errors, over R-MAT,
uniform and directed graphs, loop caps 0 / 1 / 2 / default, early exits and
both CC sparsify settings."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gb():
    import paper_1908_01407_b200 as gb
    return gb


def _engine(gb, e):
    return gb._lib.load().gb_loop_engine(e)


def _both(gb, fn):
    out = []
    for e in (1, 0):   # host loop first, then the device loop
        prev = _engine(gb, e)
        try:
            d = gb.Descriptor()
            r = fn(d)
            out.append((r, [(x.chosen, x.frontier_nvals, x.estimated_frontier_edges)
                            for x in d.direction_log]))
        finally:
            _engine(gb, prev)
    return out


GRAPHS = [("rmat", 12, .57), ("rmat", 16, .57), ("uniform", 14, .25)]


def _graph(gb, kind, scale, a, weighted=False):
    b = c = .19 if a == .57 else .25
    return gb.io.rmat_matrix(scale, a=a, b=b, c=c, d=1 - a - b - c, weighted=weighted)


@pytest.mark.parametrize("kind,scale,a", GRAPHS)
@pytest.mark.parametrize("cap", [None, 0, 1, 2])
def test_sssp_graph_loop_equals_host_loop(gb, kind, scale, a, cap):
    W = _graph(gb, kind, scale, a, weighted=True)

    def run(d):
        if cap is not None:
            d.max_niter = cap
        return gb.sssp(W, 0, desc=d).values
    (h, hl), (g, gl) = _both(gb, run)
    assert np.array_equal(h, g) and hl == gl


@pytest.mark.parametrize("kind,scale,a", GRAPHS)
@pytest.mark.parametrize("eps,iters", [(1e-300, 20), (1e-7, 10_000), (1e-300, 1), (1e-300, 0)])
def test_pagerank_graph_loop_equals_host_loop(gb, kind, scale, a, eps, iters):
    A = _graph(gb, kind, scale, a)
    (h, hl), (g, gl) = _both(gb, lambda d: gb.pagerank(A, eps=eps, max_iters=iters, desc=d).values)
    assert hl == gl
    # same kernels; hub rows fold across tiles with float atomics, so the sums
    # may differ in the last bit between any two runs
    assert np.abs(h - g).sum() <= 1e-12


@pytest.mark.parametrize("kind,scale,a", GRAPHS)
@pytest.mark.parametrize("sparsify", [True, False])
def test_cc_graph_loop_equals_host_loop(gb, kind, scale, a, sparsify):
    A = _graph(gb, kind, scale, a)
    (h, hl), (g, gl) = _both(gb, lambda d: gb.connected_components(A, desc=d,
                                                                    sparsify=sparsify).values)
    assert np.array_equal(h, g) and hl == gl


def test_cc_push_branch_and_long_rows(gb):
    """Force push every iteration (hub rows > 4096 entries take the grid-wide
    pass) and compare with the host loop."""
    A = gb.io.rmat_matrix(16)
    (h, hl), (g, gl) = _both(gb, lambda d: gb.connected_components(
        A, desc=_force(gb, d, gb.Direction.FORCE_PUSH)).values)
    assert np.array_equal(h, g) and hl == gl
    assert {x[0] for x in gl} == {"push"}


def test_sssp_push_only_directed(gb):
    rng = np.random.default_rng(8)
    n = 5000
    r = rng.integers(0, n, 60000)
    c = (r + rng.integers(1, 300, r.size)) % n
    w = rng.random(r.size) + 0.1
    A = gb.SparseMatrix.from_tuples(r, c, w, n, n, dedup=gb.builtin_monoid("Minimum"))
    (h, hl), (g, gl) = _both(gb, lambda d: gb.sssp(A, 0, desc=_force(
        gb, d, gb.Direction.FORCE_PUSH)).values)
    assert np.array_equal(h, g) and hl == gl


def _force(gb, d, direction):
    d.direction = direction
    return d


def test_cc_unsorted_rows(gb):
    """Rows that do not start at their smallest column (from_csr wraps them
    as given): the first pull falls back to the streaming row minimum and the
    labels, logs and iteration counts equal the sorted matrix's."""
    A = gb.io.rmat_matrix(12)
    o = A.orient(False)
    off = o.offsets.cpu().numpy()
    idx = o.indices.cpu().numpy().copy()
    for r in range(A.nrows):          # reverse every row: the minimum moves last
        idx[off[r]:off[r + 1]] = idx[off[r]:off[r + 1]][::-1].copy()
    U = gb.SparseMatrix.from_csr(A.nrows, A.ncols, off, idx, np.ones(idx.size, np.int64),
                                 symmetric=True)
    want = _both(gb, lambda d: gb.connected_components(A, desc=d).values)
    got = _both(gb, lambda d: gb.connected_components(U, desc=d).values)
    for (w, wl), (g, gl) in zip(want, got):
        assert np.array_equal(w, g) and wl == gl
