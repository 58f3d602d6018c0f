"""GPU parity of the fused SSSP / PageRank / CC / TC drivers.

Small scales: against the reference goldens (digests, traces, full vectors).
Larger scales: against the C oracle on the same CSR.  Each fused driver is
also cross-checked against the reference's literal operator composition run
through the unfused kernels (Descriptor(fused=False)).
"""

import hashlib

import numpy as np
import pytest

from golden_io import GOLDEN, load_json

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gb():
    import paper_1908_01407_b200 as gb
    return gb


def digest(vec):
    idx, vals = vec.extract_tuples()
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(idx).tobytes())
    h.update(np.ascontiguousarray(np.round(np.asarray(vals, dtype=np.float64), 9)).tobytes())
    return h.hexdigest()


def trace(desc):
    return [[d.chosen, d.frontier_nvals, d.estimated_frontier_edges, d.threshold_edges]
            for d in desc.direction_log]


@pytest.mark.parametrize("s", [8, 10, 12, 14])
def test_sssp_golden(gb, s):
    gold = load_json("algorithms.json")[f"sssp_s{s}"]
    W = gb.io.rmat_matrix(s, weighted=True)
    seen = []
    desc = gb.Descriptor()
    dist = gb.sssp(W, 0, desc=desc, on_iteration=lambda it, d: seen.append(it))
    assert digest(dist) == gold["digest"]
    assert trace(desc) == gold["trace"]
    assert len(seen) == gold["iterations"]
    if "values" in gold:
        assert np.array_equal(dist.values, np.asarray(gold["values"]))


@pytest.mark.parametrize("s", [8, 10, 12, 14])
def test_cc_golden(gb, s):
    gold = load_json("algorithms.json")[f"cc_s{s}"]
    A = gb.io.rmat_matrix(s)
    desc = gb.Descriptor()
    cc = gb.connected_components(A, desc=desc)
    assert digest(cc) == gold["digest"]
    assert trace(desc) == gold["trace"]
    if "values" in gold:
        assert cc.values.tolist() == gold["values"]


@pytest.mark.parametrize("s", [8, 10, 12, 14])
def test_pagerank_golden(gb, s):
    A = gb.io.rmat_matrix(s)
    want = np.load(f"{GOLDEN}/pr_s{s}.npy")
    got = gb.pagerank(A, alpha=0.85, eps=1e-300, max_iters=20).values
    assert np.abs(got - want).sum() <= 1e-6
    assert np.abs(got - want).max() <= 1e-12
    want_d = np.load(f"{GOLDEN}/pr_default_s{s}.npy")
    got_d = gb.pagerank(A).values
    assert np.abs(got_d - want_d).sum() <= 1e-6


@pytest.mark.parametrize("s", [8, 10, 12, 14])
def test_tc_golden(gb, s):
    gold = load_json("algorithms.json")[f"tc_s{s}"]
    assert gb.triangle_count(gb.io.rmat_matrix(s)) == gold["count"]


@pytest.mark.parametrize("s", [10, 12])
def test_uniform_family_goldens(gb, s):
    gold = load_json("algorithms.json")
    A = gb.io.rmat_matrix(s, a=0.25, b=0.25, c=0.25, d=0.25)
    assert digest(gb.connected_components(A)) == gold[f"uniform_cc_s{s}"]["digest"]
    assert gb.triangle_count(A) == gold[f"uniform_tc_s{s}"]["count"]


def test_fused_equals_composed(gb):
    """Fused drivers == the reference's literal composition on the unfused kernels."""
    A = gb.io.rmat_matrix(10)
    W = gb.io.rmat_matrix(10, weighted=True)
    for algo in ("bfs", "sssp", "cc", "pr", "tc"):
        df, dc = gb.Descriptor(), gb.Descriptor(fused=False)
        if algo == "bfs":
            a, b = gb.bfs(A, 0, desc=df), gb.bfs(A, 0, desc=dc)
        elif algo == "sssp":
            a, b = gb.sssp(W, 0, desc=df), gb.sssp(W, 0, desc=dc)
        elif algo == "cc":
            a, b = gb.connected_components(A, desc=df), gb.connected_components(A, desc=dc)
        elif algo == "pr":
            a = gb.pagerank(A, eps=1e-300, max_iters=20, desc=df)
            b = gb.pagerank(A, eps=1e-300, max_iters=20, desc=dc)
            assert np.abs(a.values - b.values).sum() <= 1e-12
            continue
        else:
            assert gb.triangle_count(A, desc=df) == gb.triangle_count(A, desc=dc)
            continue
        ai, av = a.extract_tuples()
        bi, bv = b.extract_tuples()
        assert np.array_equal(ai, bi) and np.array_equal(av, bv), algo
        assert [(x.chosen, x.frontier_nvals) for x in df.direction_log] == \
            [(x.chosen, x.frontier_nvals) for x in dc.direction_log], algo


@pytest.mark.parametrize("s", [16, 18])
def test_algorithms_match_c_oracle(gb, s):
    from oracle import cgraph, port
    A = gb.io.rmat_matrix(s)
    rp, ci = A._csr.offsets.cpu().numpy(), A._csr.indices.cpu().numpy()
    par, tr = cgraph.cc(rp, ci)
    desc = gb.Descriptor()
    assert np.array_equal(gb.connected_components(A, desc=desc).values, par)
    assert [(d.chosen, d.frontier_nvals) for d in desc.direction_log] == [t[:2] for t in tr]
    ranks, errs = cgraph.pagerank(rp, ci, eps=1e-300, max_iters=20)
    got = gb.pagerank(A, eps=1e-300, max_iters=20).values
    assert np.abs(got - ranks).sum() <= 1e-6
    assert gb.triangle_count(A) == cgraph.tc(rp, ci)
    W = gb.io.rmat_matrix(s, weighted=True)
    w = W._csr.values.cpu().numpy()
    dist, tr = cgraph.sssp(rp, ci, w, 0)
    desc = gb.Descriptor()
    got = gb.sssp(W, 0, desc=desc).values
    assert np.array_equal(np.isinf(got), np.isinf(dist))
    fin = ~np.isinf(dist)
    assert np.allclose(got[fin], dist[fin], rtol=1e-5, atol=0)
    assert np.array_equal(got, dist)  # integral weights: exact
    assert [(d.chosen, d.frontier_nvals) for d in desc.direction_log] == [t[:2] for t in tr]


def test_spec_examples(gb):
    K4 = gb.matrix_build([(i, j, 1) for i in range(4) for j in range(4) if i != j], 4, 4)
    assert gb.triangle_count(K4) == 4
    T = gb.matrix_build([(0, 1, 4.0), (1, 0, 4.0), (0, 2, 2.0), (2, 0, 2.0), (1, 2, 5.0), (2, 1, 5.0)], 3, 3)
    assert gb.sssp(T, 0).values.tolist() == [0.0, 4.0, 2.0]
    two = gb.matrix_build([(0, 1, 1), (1, 0, 1), (2, 3, 1), (3, 2, 1)], 5, 5)
    assert gb.connected_components(two).values.tolist() == [0, 0, 2, 2, 4]


def test_algorithm_input_errors(gb):
    neg = gb.matrix_build([(0, 1, -1.0), (1, 0, -1.0)], 2, 2)
    with pytest.raises(ValueError):
        gb.sssp(neg, 0)
    directed = gb.matrix_build([(0, 1, 1)], 2, 2)
    with pytest.raises(ValueError):
        gb.connected_components(directed)
    with pytest.raises(ValueError):
        gb.triangle_count(directed)
    loop = gb.matrix_build([(0, 0, 1), (0, 1, 1), (1, 0, 1)], 2, 2)
    with pytest.raises(ValueError):
        gb.triangle_count(loop)
    A = gb.io.rmat_matrix(6)
    with pytest.raises(ValueError):
        gb.pagerank(A, alpha=1.5)
    with pytest.raises(ValueError):
        gb.pagerank(A, eps=0.0)
    with pytest.raises(gb.ShapeError):
        gb.sssp(gb.matrix_build([(0, 1, 1.0)], 2, 3), 0)


def test_cc_without_sparsify_and_max_niter(gb):
    from oracle import port
    A = gb.io.rmat_matrix(10)
    rp, ci, n = port.rmat_csr(10)
    P = port.mat_from_csr(rp, ci, np.ones(ci.size, np.int64), n)
    for sp in (True, False):
        for cap in (1, 2, 50):
            d = gb.Descriptor(max_niter=cap)
            got = gb.connected_components(A, desc=d, sparsify=sp)
            pd = port.Desc(max_niter=cap)
            want = port.connected_components(P, pd, sparsify=sp)
            assert np.array_equal(got.values, want.vals), (sp, cap)
            assert [x.chosen for x in d.direction_log] == [x[0] for x in pd.log]
