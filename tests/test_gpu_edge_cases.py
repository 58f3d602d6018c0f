"""Edge cases of this round's device paths: edgeless and single-vertex
graphs, an isolated source, zero loop caps, empty masks, masks that allow
nothing -- through the row bins, column stripes, device loops, BFS parents /
validation and the fused counters, each against the reference composition
(fused=False) or the obvious answer."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gb():
    import paper_1908_01407_b200 as gb
    return gb


def _edgeless(gb, n, weighted=False):
    e = np.zeros(0, np.int64)
    vals = np.zeros(0, np.float64 if weighted else np.int64)
    return gb.SparseMatrix.from_tuples(e, e, vals, n, n)


@pytest.mark.parametrize("n", [1, 7])
def test_algorithms_on_edgeless_graphs(gb, n):
    A = _edgeless(gb, n)
    W = _edgeless(gb, n, weighted=True)
    for fused in (True, False):
        d = gb.Descriptor(fused=fused)
        lv = gb.bfs(A, 0, desc=d).values
        assert lv.tolist() == [1] + [0] * (n - 1)
        assert gb.sssp(W, 0, desc=gb.Descriptor(fused=fused)).to_dense(np.inf).values.tolist() == \
            [0.0] + [np.inf] * (n - 1)
        cc = gb.connected_components(A, desc=gb.Descriptor(fused=fused)).values
        assert cc.tolist() == list(range(n))
        assert gb.triangle_count(A, desc=gb.Descriptor(fused=fused)) == 0
    lv, par = gb.bfs_parents(A, 0)
    assert par.values.tolist() == [0] + [-1] * (n - 1)
    assert gb.validate_bfs(A, 0, lv, par)["ok"]
    d = gb.Descriptor(count_work=True)
    gb.bfs(A, 0, desc=d)
    c = gb.Descriptor(fused=False)
    gb.bfs(A, 0, desc=c)
    assert (d.counters.matrix_entries_read, d.counters.semiring_multiplies) == \
        (c.counters.matrix_entries_read, c.counters.semiring_multiplies)


def test_pagerank_edgeless_and_single_vertex(gb):
    # nnz == 0 takes the composed path; the result is the teleport fixpoint
    for n in (1, 5):
        A = _edgeless(gb, n)
        want = gb.pagerank(A, desc=gb.Descriptor(fused=False)).values
        got = gb.pagerank(A).values
        np.testing.assert_allclose(got, want, rtol=1e-12)


def test_isolated_source_and_zero_caps(gb):
    A = gb.io.rmat_matrix(10)
    deg = np.diff(A.row_offsets)
    iso = int(np.flatnonzero(deg == 0)[0])
    lv = gb.bfs(A, iso).values
    assert lv[iso] == 1 and lv.sum() == 1
    lvp, par = gb.bfs_parents(A, iso)
    assert par.values[iso] == iso and (par.values >= 0).sum() == 1
    W = gb.io.rmat_matrix(10, weighted=True)
    for cap in (0, 1):
        for fused in (True, False):
            d = gb.Descriptor(max_niter=cap, fused=fused)
            got = gb.sssp(W, 0, desc=d).to_dense(np.inf).values
            ref = gb.sssp(W, 0, desc=gb.Descriptor(max_niter=cap, fused=False)).to_dense(np.inf).values
            assert np.array_equal(got, ref)
        got = gb.connected_components(A, desc=gb.Descriptor(max_niter=cap)).values
        ref = gb.connected_components(A, desc=gb.Descriptor(max_niter=cap, fused=False)).values
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("impl", ["bins", "stripes"])
def test_masks_allowing_nothing_or_everything(gb, monkeypatch, impl):
    from paper_1908_01407_b200 import kernels
    monkeypatch.setattr(kernels, "_MV_BINS", "1")
    monkeypatch.setattr(kernels, "_MV_STRIPE_BYTES", 4096 if impl == "stripes" else 0)
    monkeypatch.setattr(kernels, "_MV_STRIPE_SKEW", 1.0)
    A = gb.io.rmat_matrix(11)
    n = A.nrows
    x = gb.Vector.dense_of(np.arange(n, dtype=np.float64) + 1, 0.0)
    sr = gb.builtin_semiring("PlusMultiplies")
    none = gb.Vector.dense_of(np.zeros(n, np.int64), 0)
    d = gb.Descriptor(direction=gb.Direction.FORCE_PULL)
    w = gb.mxv(sr, A, x, mask=none, desc=d).to_dense(0.0).values
    assert not w.any() and d.counters.matrix_entries_read == 0
    everything = gb.Vector.dense_of(np.ones(n, np.int64), 0)
    d1 = gb.Descriptor(direction=gb.Direction.FORCE_PULL)
    w1 = gb.mxv(sr, A, x, mask=everything, desc=d1).to_dense(0.0).values
    monkeypatch.setattr(kernels, "_MV_BINS", "0")
    d2 = gb.Descriptor(direction=gb.Direction.FORCE_PULL)
    w2 = gb.mxv(sr, A, x, desc=d2).to_dense(0.0).values
    np.testing.assert_allclose(w1, w2, rtol=1e-12, atol=0)
    assert (d1.counters.matrix_entries_read, d1.counters.semiring_multiplies,
            d1.counters.semiring_adds) == (d2.counters.matrix_entries_read,
                                           d2.counters.semiring_multiplies,
                                           d2.counters.semiring_adds)
