"""GPU parity: R-MAT generator and fused BFS against the reference goldens and the C oracle."""

import hashlib

import numpy as np
import pytest

from golden_io import load_json

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gb():
    import paper_1908_01407_b200 as gb
    return gb


def csr_digest(rp, ci):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(rp, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(ci, dtype=np.int64).tobytes())
    return h.hexdigest()


def digest(vec):
    idx, vals = vec.extract_tuples()
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(idx).tobytes())
    h.update(np.ascontiguousarray(np.round(np.asarray(vals, dtype=np.float64), 9)).tobytes())
    return h.hexdigest()


def trace(desc):
    return [[d.chosen, d.frontier_nvals, d.estimated_frontier_edges, d.threshold_edges]
            for d in desc.direction_log]


@pytest.mark.parametrize("key", ["rmat_s8", "rmat_s10", "rmat_s12", "rmat_s14", "rmat_s16",
                                 "uniform_s8", "uniform_s10", "uniform_s12", "uniform_s14"])
def test_generator_matches_reference(gb, key):
    g = load_json("rmat_graphs.json")["graphs"][key]
    kw = dict(a=0.25, b=0.25, c=0.25, d=0.25) if key.startswith("uniform") else {}
    A = gb.io.rmat_matrix(g["scale"], **kw)
    assert A.nnz == g["nnz"]
    assert csr_digest(A.row_offsets, A.col_indices) == g["csr"]
    assert A.is_symmetric()
    if g["weights"] is not None:
        W = gb.io.rmat_matrix(g["scale"], weighted=True, **kw)
        assert hashlib.sha256(W.csr_values.tobytes()).hexdigest() == g["weights"]


@pytest.mark.parametrize("s", [8, 10, 12, 14, 16])
def test_bfs_golden(gb, s):
    gold = load_json("algorithms.json")
    A = gb.io.rmat_matrix(s)
    desc = gb.Descriptor()
    lv = gb.bfs(A, 0, desc=desc)
    assert digest(lv) == gold[f"bfs_s{s}"]["digest"]
    assert trace(desc) == gold[f"bfs_s{s}"]["trace"]
    if "values" in gold[f"bfs_s{s}"]:
        assert lv.values.tolist() == gold[f"bfs_s{s}"]["values"]
    other = [k for k in gold if k.startswith(f"bfs_s{s}_src")][0]
    src = gold[other]["source"]
    desc = gb.Descriptor()
    lv = gb.bfs(A, src, desc=desc)
    assert digest(lv) == gold[other]["digest"]
    assert trace(desc) == gold[other]["trace"]


@pytest.mark.parametrize("s", [10, 12])
def test_bfs_uniform_golden(gb, s):
    gold = load_json("algorithms.json")[f"uniform_bfs_s{s}"]
    A = gb.io.rmat_matrix(s, a=0.25, b=0.25, c=0.25, d=0.25)
    desc = gb.Descriptor()
    assert digest(gb.bfs(A, 0, desc=desc)) == gold["digest"]
    assert trace(desc) == gold["trace"]


@pytest.mark.parametrize("s", [18, 20])
def test_bfs_matches_c_oracle(gb, s):
    from oracle import cgraph
    A = gb.io.rmat_matrix(s)
    rp, ci = cgraph.rmat_csr(s)
    assert np.array_equal(A.row_offsets, rp) and np.array_equal(A.col_indices, ci)
    for src in (0, 1, int(np.argmax(np.diff(rp) == 1))):
        desc = gb.Descriptor()
        lv = gb.bfs(A, src, desc=desc)
        want, tr = cgraph.bfs(rp, ci, src)
        assert np.array_equal(lv.values, want)
        assert [(d.chosen, d.frontier_nvals, d.estimated_frontier_edges) for d in desc.direction_log] == tr


def test_bfs_s24_properties(gb):
    """Size-independent checks at the benchmark scale (SURVEY §8 input table)."""
    from oracle import cgraph
    import torch
    A = gb.io.rmat_matrix(24)
    assert A.nnz == 520_756_042
    deg = torch.diff(A._csr.offsets)
    assert int(deg.max()) == 405_970 and int(deg.argmax()) == 0
    assert int((deg == 0).sum()) == 7_906_093
    desc = gb.Descriptor()
    lv = gb.bfs(A, 0, desc=desc)
    vals = lv.values
    assert int(np.count_nonzero(vals)) == 8_865_184
    assert [d.chosen for d in desc.direction_log] == ["push", "push", "pull", "push", "push", "push"]
    assert [d.frontier_nvals for d in desc.direction_log] == [1, 405_970, 7_612_546, 843_624, 3_034, 9]
    rp = A._csr.offsets.cpu().numpy()
    ci = A._csr.indices.cpu().numpy()
    want, _ = cgraph.bfs(rp, ci, 0)
    assert np.array_equal(vals, want)


# ---------------------------------------------------------------------------
# device-driven loop (one CUDA graph) vs the host-driven loop
# ---------------------------------------------------------------------------


def _run_both(gb, A, src, **kw):
    from paper_1908_01407_b200 import _lib
    ctx = _lib.context()
    d1 = gb.Descriptor(**kw)
    g = gb.bfs(A, src, desc=d1).values            # graph path
    ctx.profiling(True)                            # per-kernel events force the host loop
    try:
        d2 = gb.Descriptor(**kw)
        h = gb.bfs(A, src, desc=d2).values
    finally:
        ctx.profiling(False)
        ctx.prof_read()
    t1 = [(d.chosen, d.frontier_nvals, d.estimated_frontier_edges) for d in d1.direction_log]
    t2 = [(d.chosen, d.frontier_nvals, d.estimated_frontier_edges) for d in d2.direction_log]
    return g, h, t1, t2


@pytest.mark.parametrize("s", [6, 12, 16, 20])
def test_bfs_graph_loop_equals_host_loop(gb, s):
    A = gb.io.rmat_matrix(s)
    for src in (0, 5, A.nrows - 1):
        for kw in ({}, {"max_niter": 1}, {"max_niter": 2}, {"max_niter": 3},
                   {"direction": gb.Direction.FORCE_PUSH}, {"direction": gb.Direction.FORCE_PULL},
                   {"switch_ratio": 0.0}, {"switch_ratio": 1.0}):
            g, h, t1, t2 = _run_both(gb, A, src, **kw)
            assert np.array_equal(g, h), (src, kw)
            assert t1 == t2, (src, kw)


def test_bfs_graph_cache_follows_the_matrix(gb):
    """The cached graph is keyed by the matrix: alternating matrices and
    sources gives each one's own answer."""
    from oracle import cgraph
    mats = [gb.io.rmat_matrix(10), gb.io.rmat_matrix(11), gb.io.rmat_matrix(10, a=0.25, b=0.25, c=0.25, d=0.25)]
    for _ in range(2):
        for A in mats:
            rp = A._csr.offsets.cpu().numpy()
            ci = A._csr.indices.cpu().numpy()
            for src in (0, 9):
                want, _ = cgraph.bfs(rp, ci, src)
                assert np.array_equal(gb.bfs(A, src).values, want)


def test_bfs_graph_long_path(gb):
    """A path graph runs one level per vertex: many WHILE iterations, both
    halves of the unrolled body, and more than 21 logged decisions."""
    n = 300
    r = np.r_[np.arange(n - 1), np.arange(1, n)]
    c = np.r_[np.arange(1, n), np.arange(n - 1)]
    A = gb.SparseMatrix.from_tuples(r, c, np.ones(r.size, np.int64), n, n)
    g, h, t1, t2 = _run_both(gb, A, 0)
    assert g.tolist() == list(range(1, n + 1))
    assert np.array_equal(g, h) and t1 == t2 and len(t1) == n
    for cap in (20, 21, 22, 23, 150):
        g, h, t1, t2 = _run_both(gb, A, 0, max_niter=cap)
        assert np.array_equal(g, h) and t1 == t2 and len(t1) == cap


def test_bfs_deep_levels_past_narrow_range(gb):
    """Relabelled runs keep 16-bit levels and redo runs of >= 65,000 levels
    with int32 levels: both engines, around the switch and the saturation."""
    n = 65600
    r = np.r_[np.arange(n - 1), np.arange(1, n)]
    c = np.r_[np.arange(1, n), np.arange(n - 1)]
    A = gb.SparseMatrix.from_tuples(r, c, np.ones(r.size, np.int64), n, n)
    for cap in (70000, 65001):
        g, h, t1, t2 = _run_both(gb, A, 0, max_niter=cap)
        want = np.arange(1, n + 1)
        want[cap:] = 0
        assert np.array_equal(g, want), cap
        assert np.array_equal(g, h) and t1 == t2, cap


def test_bfs_deep_levels_with_a_shortcut(gb):
    from oracle import port
    n = 700
    r = np.r_[np.arange(n - 1), np.arange(1, n), [0, 5]]
    c = np.r_[np.arange(1, n), np.arange(n - 1), [5, 0]]
    A = gb.SparseMatrix.from_tuples(r, c, np.ones(r.size, np.int64), n, n)
    P = port.mat_from_tuples(r, c, np.ones(r.size, np.int64), n, n)
    for src, cap in ((0, None), (350, None), (0, 249), (0, 256), (0, 400)):
        kw = {} if cap is None else {"max_niter": cap}
        g, h, t1, t2 = _run_both(gb, A, src, **kw)
        want = port.bfs(P, src, port.Desc(**kw)).vals
        assert np.array_equal(g, want), (src, cap)
        assert np.array_equal(g, h) and t1 == t2, (src, cap)


# ---------------------------------------------------------------------------
# edge cases the reference semantics define
# ---------------------------------------------------------------------------


def test_bfs_isolated_source(gb):
    A = gb.matrix_build([(1, 2, 1), (2, 1, 1)], 4, 4)
    desc = gb.Descriptor()
    lv = gb.bfs(A, 0, desc=desc)
    assert lv.values.tolist() == [1, 0, 0, 0]
    assert [d.chosen for d in desc.direction_log] == ["push"]


def test_bfs_path_graph_spec_example(gb):
    # SPEC example: path 0-1-2 from 0 gives [1, 2, 3]
    A = gb.matrix_build([(0, 1, 1), (1, 0, 1), (1, 2, 1), (2, 1, 1)], 3, 3)
    assert gb.bfs(A, 0).values.tolist() == [1, 2, 3]


def test_bfs_directed_graph_uses_both_orientations(gb):
    from oracle import port
    rng = np.random.default_rng(5)
    n = 300
    r = rng.integers(0, n, 3000)
    c = rng.integers(0, n, 3000)
    A = gb.SparseMatrix.from_tuples(r, c, np.ones(r.size, np.int64), n, n)
    assert not A.is_symmetric()
    P = port.mat_from_tuples(r, c, np.ones(r.size, np.int64), n, n)
    for policy in (gb.Direction.AUTO, gb.Direction.FORCE_PUSH, gb.Direction.FORCE_PULL):
        desc = gb.Descriptor(direction=policy)
        got = gb.bfs(A, 3, desc=desc)
        pd = port.Desc(direction=policy.value)
        want = port.bfs(P, 3, pd)
        assert np.array_equal(got.values, want.vals)
        assert [d.chosen for d in desc.direction_log] == [x[0] for x in pd.log]


def test_bfs_max_niter_cap(gb):
    from oracle import port
    A = gb.io.rmat_matrix(10)
    rp, ci, n = port.rmat_csr(10)
    P = port.mat_from_csr(rp, ci, np.ones(ci.size, np.int64), n)
    for cap in (1, 2, 3):
        desc = gb.Descriptor(max_niter=cap)
        got = gb.bfs(A, 0, desc=desc)
        pd = port.Desc(max_niter=cap)
        want = port.bfs(P, 0, pd)
        assert np.array_equal(got.values, want.vals)
        assert len(desc.direction_log) == len(pd.log)


def test_bfs_zero_valued_edges_do_not_propagate(gb):
    # LogicalAnd(0, 1) is false: a stored 0 is not an edge for traversal
    A = gb.matrix_build([(0, 1, 0), (1, 0, 0), (0, 2, 1), (2, 0, 1), (2, 3, 5), (3, 2, 5)], 4, 4)
    assert gb.bfs(A, 0).values.tolist() == [1, 0, 2, 3]
    for policy in (gb.Direction.FORCE_PUSH, gb.Direction.FORCE_PULL):
        assert gb.bfs(A, 0, gb.Descriptor(direction=policy)).values.tolist() == [1, 0, 2, 3]


def test_bfs_bad_source(gb):
    A = gb.io.rmat_matrix(6)
    with pytest.raises(IndexError):
        gb.bfs(A, 64)
    with pytest.raises(gb.ShapeError):
        gb.bfs(gb.matrix_build([(0, 1, 1)], 2, 3), 0)


# ---------------------------------------------------------------------------
# degree-ordered traversal layout (SparseMatrix.traversal, gb_bfs_ordered)
# ---------------------------------------------------------------------------


def _orient_tuples(o):
    rp = o.offsets.cpu().numpy()
    ci = o.indices.cpu().numpy().astype(np.int64)
    rows = np.repeat(np.arange(o.nrows), np.diff(rp))
    vals = o.dense_values().cpu().numpy()
    return rp, rows, ci, vals


def test_degree_order_and_relabel_are_an_isomorphism(gb):
    rng = np.random.default_rng(11)
    n = 700
    r = rng.integers(0, n, 6000)
    c = rng.integers(0, n, 6000)
    v = rng.integers(0, 3, 6000)  # stored zeros included
    A = gb.SparseMatrix.from_tuples(r, c, v, n, n)
    assert not A.is_symmetric()
    push, pull, rank = A.traversal()
    rank = rank.cpu().numpy().astype(np.int64)
    assert np.array_equal(np.sort(rank), np.arange(n))
    indeg = np.diff(A._csc.offsets.cpu().numpy())
    order = np.argsort(rank)
    assert np.array_equal(order, np.lexsort((np.arange(n), -indeg)))  # degree desc, ties by id
    # push = P A P^T, pull = P A^T P^T, every row sorted
    ar, ac, av = A.extract_tuples()
    for o, (i, j) in ((push, (ar, ac)), (pull, (ac, ar))):
        rp, rows, ci, vals = _orient_tuples(o)
        got = sorted(zip(rows.tolist(), ci.tolist(), vals.tolist()))
        want = sorted(zip(rank[i].tolist(), rank[j].tolist(), av.tolist()))
        assert got == want
        for k in range(n):
            seg = ci[rp[k]:rp[k + 1]]
            assert np.all(np.diff(seg) > 0)
    assert A.traversal()[0] is push  # cached


def _bfs_both_layouts(gb, A, src, monkeypatch, **kw):
    from paper_1908_01407_b200 import algorithms
    out = []
    for ordered in (True, False):
        monkeypatch.setattr(algorithms, "_ORDERED_BFS", ordered)
        g, h, t1, t2 = _run_both(gb, A, src, **kw)
        assert np.array_equal(g, h) and t1 == t2, (ordered, src, kw)
        out.append((g, t1))
    monkeypatch.setattr(algorithms, "_ORDERED_BFS", True)
    (g1, t1), (g2, t2) = out
    assert np.array_equal(g1, g2), (src, kw)
    assert t1 == t2, (src, kw)


@pytest.mark.parametrize("s", [8, 14, 18])
def test_bfs_ordered_equals_original_labels(gb, s, monkeypatch):
    A = gb.io.rmat_matrix(s)
    for src in (0, 3, A.nrows - 1):
        for kw in ({}, {"max_niter": 2}, {"direction": gb.Direction.FORCE_PUSH},
                   {"direction": gb.Direction.FORCE_PULL}):
            _bfs_both_layouts(gb, A, src, monkeypatch, **kw)


def test_bfs_ordered_directed_valued(gb, monkeypatch):
    rng = np.random.default_rng(7)
    n = 2000
    r = rng.integers(0, n, 30000)
    c = (r + rng.integers(1, 40, 30000)) % n
    v = rng.integers(0, 4, 30000)
    A = gb.SparseMatrix.from_tuples(r, c, v, n, n)
    for src in (0, 17, 1999):
        for kw in ({}, {"direction": gb.Direction.FORCE_PUSH}, {"direction": gb.Direction.FORCE_PULL},
                   {"switch_ratio": 0.0}, {"max_niter": 3}):
            _bfs_both_layouts(gb, A, src, monkeypatch, **kw)


def test_bfs_ordered_smem_prefix_large_frontier(gb, monkeypatch):
    """Uniform graph whose push levels are large enough to take the
    shared-memory prefix path, with n above the 1.57 M-vertex prefix."""
    A = gb.io.rmat_matrix(21, a=0.25, b=0.25, c=0.25, d=0.25)
    from oracle import cgraph
    rp = A._csr.offsets.cpu().numpy()
    ci = A._csr.indices.cpu().numpy()
    for src in (0, 123457):
        for kw in ({}, {"direction": gb.Direction.FORCE_PUSH}):
            desc = gb.Descriptor(**kw)
            lv = gb.bfs(A, src, desc=desc).values
            want, tr = cgraph.bfs(rp, ci, src) if not kw else (None, None)
            if want is not None:
                assert np.array_equal(lv, want)
            _bfs_both_layouts(gb, A, src, monkeypatch, **kw)


# ---------------------------------------------------------------------------
# engines: the CUDA graph (default) vs the host-driven loop, both layouts
# ---------------------------------------------------------------------------


def _engines(gb, A, src, **kw):
    from paper_1908_01407_b200 import _lib
    lib = _lib.load()
    out = []
    prev = lib.gb_bfs_engine(-1)
    try:
        for eng in (0, 1):
            lib.gb_bfs_engine(eng)
            d = gb.Descriptor(**kw)
            lv = gb.bfs(A, src, desc=d).values
            out.append((lv, [(x.chosen, x.frontier_nvals, x.estimated_frontier_edges)
                             for x in d.direction_log]))
    finally:
        lib.gb_bfs_engine(prev)
    return out


@pytest.mark.parametrize("s", [6, 12, 18, 22])
def test_bfs_engines_agree(gb, s, monkeypatch):
    from paper_1908_01407_b200 import algorithms
    A = gb.io.rmat_matrix(s)
    for ordered in (True, False):
        monkeypatch.setattr(algorithms, "_ORDERED_BFS", ordered)
        for src in (0, 7, A.nrows - 1):
            for kw in ({}, {"max_niter": 1}, {"max_niter": 3}, {"direction": gb.Direction.FORCE_PUSH},
                       {"direction": gb.Direction.FORCE_PULL}, {"switch_ratio": 0.0}):
                (g, tg), (h, th) = _engines(gb, A, src, **kw)
                assert np.array_equal(g, h), (ordered, src, kw)
                assert tg == th, (ordered, src, kw)


def test_bfs_engines_long_path_and_values(gb):
    n = 300
    r = np.r_[np.arange(n - 1), np.arange(1, n)]
    c = np.r_[np.arange(1, n), np.arange(n - 1)]
    A = gb.SparseMatrix.from_tuples(r, c, np.ones(r.size, np.int64), n, n)
    for kw in ({}, {"max_niter": 21}, {"max_niter": 150}):
        (g, tg), (h, th) = _engines(gb, A, 0, **kw)
        assert np.array_equal(g, h) and tg == th
    # stored zeros are not edges; a directed graph uses both orientations
    rng = np.random.default_rng(3)
    n = 3000
    r = rng.integers(0, n, 40000)
    c = (r + rng.integers(1, 50, 40000)) % n
    v = rng.integers(0, 3, 40000)
    A = gb.SparseMatrix.from_tuples(r, c, v, n, n)
    for kw in ({}, {"direction": gb.Direction.FORCE_PULL}):
        (g, tg), (h, th) = _engines(gb, A, 5, **kw)
        assert np.array_equal(g, h) and tg == th


def test_bfs_async_logs_survive_the_ring(gb, monkeypatch):
    """bfs() returns before the device finishes; 300 calls (more than the 256
    ring slots) keep their own levels and decision logs, equal to the
    synchronous entry's, whatever order the logs are read in."""
    from paper_1908_01407_b200 import algorithms
    A = gb.io.rmat_matrix(12)
    n = A.nrows
    srcs = [(7 * i) % n for i in range(300)]
    pending = [(s, gb.Descriptor()) for s in srcs]
    outs = [gb.bfs(A, s, desc=d) for s, d in pending]
    monkeypatch.setattr(algorithms, "_ASYNC_BFS", False)
    for k in list(range(299, -1, -37)) + list(range(300)):
        s, d = pending[k]
        d2 = gb.Descriptor()
        want = gb.bfs(A, s, desc=d2).values
        assert np.array_equal(outs[k].values, want), k
        assert list(d.direction_log) == list(d2.direction_log), k


@pytest.mark.parametrize("src", [0, 5])
def test_bfs_async_launch_accounting_matches_sync(gb, src, monkeypatch):
    """The launches an asynchronous bfs books when its log is read equal the
    synchronous graph entry's count for the same run (bench gpu_launches)."""
    from paper_1908_01407_b200 import _lib, algorithms
    ctx = _lib.context()
    A = gb.io.rmat_matrix(14)
    gb.bfs(A, src).values  # build the graph and the log ring
    monkeypatch.setattr(algorithms, "_ASYNC_BFS", False)
    l0 = ctx.launches()
    d1 = gb.Descriptor()
    gb.bfs(A, src, desc=d1).values
    sync_n = ctx.launches() - l0
    monkeypatch.setattr(algorithms, "_ASYNC_BFS", True)
    l0 = ctx.launches()
    d2 = gb.Descriptor()
    gb.bfs(A, src, desc=d2).values
    assert len(d2.direction_log) == len(d1.direction_log)
    assert ctx.launches() - l0 == sync_n > 0


@pytest.mark.parametrize("scale,src,cap", [(10, 0, 10_000), (13, 3, 10_000), (12, 0, 2),
                                           (12, 0, 1)])
def test_cooperative_small_graph_bfs_equals_graph_loop(gb, scale, src, cap):
    """The one-kernel cooperative BFS (gb_bfs_coop.cu, the default for small
    graphs) against the device-graph loop: levels, trace and loop caps."""
    lib = gb._lib.load()
    A = gb.io.rmat_matrix(scale)
    out = {}
    for name, lim in (("coop", 1 << 30), ("graph", 0)):
        prev = lib.gb_bfs_coop_max_n(lim)
        try:
            d = gb.Descriptor(max_niter=cap)
            out[name] = (gb.bfs(A, src, desc=d).values,
                         [(x.chosen, x.frontier_nvals, x.estimated_frontier_edges)
                          for x in d.direction_log])
        finally:
            lib.gb_bfs_coop_max_n(prev)
    assert np.array_equal(out["coop"][0], out["graph"][0])
    assert out["coop"][1] == out["graph"][1]
