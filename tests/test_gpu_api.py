"""The reference's API-level test strategy run against the device backend.

Same behaviours the reference suite pins (pkg/tests/test_kernels.py,
test_containers.py), written against this package: dense-loop oracle on the
Table-4 semirings x mask modes, push == pull, exact work counters on the
paper's 8-vertex example, the direction rule, mask rules, masked SpGEMM,
element-wise ops, assign/scatter/gather, partition invariance, containers.
Seeds are fixed (the reference's hash()-seeded cases vary per process).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

EIGHT_EDGES = [(1, 0), (1, 2), (1, 3), (0, 2), (0, 4), (2, 1), (2, 4), (2, 7), (3, 0), (3, 1),
               (3, 7), (4, 5), (4, 6), (4, 2), (7, 5), (7, 6), (7, 1), (5, 6), (6, 3), (6, 7)]
TABLE = ["PlusMultiplies", "LogicalOrAnd", "MinPlus", "MaxPlus", "MinMultiplies"]


@pytest.fixture(scope="module")
def gb():
    import paper_1908_01407_b200 as gb
    return gb


def eight(gb):
    r, c = zip(*EIGHT_EDGES)
    return gb.SparseMatrix.from_tuples(r, c, np.ones(len(r), np.int64), 8, 8)


def rand_matrix(gb, rng, nr, nc, density, dtype=np.int64, low=1, high=9, symmetric=False):
    stored = rng.random((nr, nc)) < density
    if symmetric:
        stored |= stored.T
        np.fill_diagonal(stored, False)
    r, c = np.nonzero(stored)
    if np.dtype(dtype).kind == "i":
        v = rng.integers(low, high + 1, size=r.size).astype(dtype)
    else:
        v = (rng.random(r.size) * (high - low) + low).astype(dtype)
    if symmetric:
        lo, hi = np.minimum(r, c), np.maximum(r, c)
        key = lo * nc + hi
        _, first, inv = np.unique(key, return_index=True, return_inverse=True)
        v = v[first][inv]
    return gb.SparseMatrix.from_tuples(r, c, v, nr, nc)


def rand_vector(gb, rng, n, k, dtype=np.int64, low=1, high=9):
    k = min(k, n)
    idx = np.sort(rng.choice(n, size=k, replace=False))
    if np.dtype(dtype).kind == "i":
        vals = rng.integers(low, high + 1, size=k).astype(dtype)
    else:
        vals = (rng.random(k) * (high - low) + low).astype(dtype)
    return gb.Vector.from_entries(idx, vals, n, dtype=dtype)


def rand_mask(gb, rng, n, dense=False):
    if dense:
        return gb.Vector.dense_of((rng.random(n) < 0.5).astype(np.int64), 0)
    idx = np.flatnonzero(rng.random(n) < 0.5)
    return gb.Vector.from_entries(idx, (rng.random(idx.size) < 0.8).astype(np.int64), n)


def allowed(mask, n, complement):
    if mask is None:
        a = np.ones(n, bool)
    elif mask.is_sparse:
        a = np.zeros(n, bool)
        a[mask.indices[mask.values != 0]] = True
    else:
        a = mask.values != 0
    return ~a if complement else a


def dense_oracle(sr, A, u, mask=None, complement=False):
    """Two-loop semiring product with the scalar fn (independent of the kernels)."""
    d = np.zeros((A.nrows, A.ncols), dtype=A.dtype)
    st = np.zeros((A.nrows, A.ncols), bool)
    r, c, v = A.extract_tuples()
    d[r, c] = v
    st[r, c] = True
    dtype = np.result_type(A.dtype, u.dtype)
    ident = sr.add.identity_for(dtype)
    ud = np.full(A.ncols, ident, dtype=dtype)
    if u.is_sparse:
        ud[u.indices] = u.values
    else:
        ud[:] = u.values
    ok = allowed(mask, A.nrows, complement)
    oi, ov = [], []
    for i in range(A.nrows):
        if not ok[i]:
            continue
        acc = None
        for j in range(A.ncols):
            if st[i, j] and ud[j] != ident:
                p = sr.multiply.fn(d[i, j], ud[j])
                acc = p if acc is None else sr.add.op.fn(acc, p)
        if acc is not None and acc != ident:
            oi.append(i)
            ov.append(acc)
    return np.asarray(oi, np.int64), np.asarray(ov, dtype=dtype)


def same(got, idx, vals):
    gi, gv = got.extract_tuples()
    assert np.array_equal(gi, idx)
    if gv.dtype.kind == "f":
        assert np.allclose(gv, vals, rtol=1e-10, atol=0)
    else:
        assert np.array_equal(gv, vals)


@pytest.mark.parametrize("name", TABLE)
def test_mxv_dense_oracle(gb, name):
    rng = np.random.default_rng(sum(map(ord, name)))
    sr = gb.builtin_semiring(name)
    for _ in range(8):
        lo, hi = (0, 1) if name == "LogicalOrAnd" else (1, 9)
        A = rand_matrix(gb, rng, 16, 16, 0.3, low=lo, high=hi)
        u = rand_vector(gb, rng, 16, int(rng.integers(0, 17)), low=1, high=1 if lo == 0 else 9)
        for mode in ("none", "normal", "complement"):
            mask = None if mode == "none" else rand_mask(gb, rng, 16)
            d = gb.Descriptor()
            if mode == "complement":
                d.toggle("mask")
            same(gb.mxv(sr, A, u, mask=mask, desc=d), *dense_oracle(sr, A, u, mask, mode == "complement"))


def test_running_example_step(gb):
    A = eight(gb)
    d = gb.Descriptor()
    d.toggle("mask")
    w = gb.vxm(gb.builtin_semiring("LogicalOrAnd"), gb.vector_build([0, 2, 3], [1, 1, 1], 8), A,
               mask=gb.vector_build([0, 1, 2, 3], [1, 1, 1, 1], 8), desc=d)
    idx, vals = w.extract_tuples()
    assert idx.tolist() == [4, 7] and vals.tolist() == [1, 1]


def test_empty_input_and_shape_errors(gb):
    A = eight(gb)
    B = gb.builtin_semiring("LogicalOrAnd")
    assert gb.mxv(B, A, gb.Vector.empty(8)).nvals == 0
    with pytest.raises(gb.ShapeError):
        gb.mxv(B, A, gb.vector_build([0], [1], 5))
    with pytest.raises(gb.ShapeError):
        gb.mxv(B, A, gb.vector_build([0], [1], 8), mask=gb.vector_fill(5, 1))


def test_vxm_equals_mxv_of_transpose(gb):
    rng = np.random.default_rng(3)
    sr = gb.builtin_semiring("PlusMultiplies")
    for _ in range(6):
        A = rand_matrix(gb, rng, 12, 12, 0.4)
        u = rand_vector(gb, rng, 12, int(rng.integers(0, 13)))
        a, b = gb.vxm(sr, u, A), gb.mxv(sr, gb.transpose(A), u)
        ai, av = a.extract_tuples()
        bi, bv = b.extract_tuples()
        assert np.array_equal(ai, bi) and np.array_equal(av, bv)
        d = gb.Descriptor()
        d.toggle("inp1")
        same(gb.vxm(sr, u, A, desc=d), *gb.mxv(sr, A, u).extract_tuples())


@pytest.mark.parametrize("name", TABLE)
def test_push_equals_pull(gb, name):
    rng = np.random.default_rng(100 + sum(map(ord, name)))
    sr = gb.builtin_semiring(name)
    for _ in range(6):
        lo, hi = (0, 1) if name == "LogicalOrAnd" else (1, 9)
        A = rand_matrix(gb, rng, 16, 16, 0.3, low=lo, high=hi)
        u = rand_vector(gb, rng, 16, int(rng.integers(0, 17)), low=1, high=1 if lo == 0 else 9)
        for mode in ("none", "normal", "complement"):
            mask = None if mode == "none" else rand_mask(gb, rng, 16)
            d = gb.Descriptor()
            if mode == "complement":
                d.toggle("mask")
            ident = sr.add.identity_for(np.result_type(A.dtype, u.dtype))
            pull = gb.spmv_pull(sr, A, u.to_dense(ident), mask=mask, desc=d)
            push = gb.spmspv_push(sr, A, u, mask=mask, desc=d)
            pi, pv = pull.extract_tuples()
            qi, qv = push.extract_tuples()
            assert np.array_equal(pi, qi)
            assert np.allclose(pv, qv, rtol=1e-10, atol=0)


def test_work_counters_eight_vertex(gb):
    A = eight(gb)
    B = gb.builtin_semiring("LogicalOrAnd")
    ones = gb.vector_fill(8, 1, dtype=np.int64)
    d = gb.Descriptor()
    gb.spmv_pull(B, A, ones, desc=d)
    assert d.counters.matrix_entries_read == 20
    d = gb.Descriptor()
    gb.spmv_pull(B, A, ones, mask=gb.vector_build([4, 6, 7], [1, 1, 1], 8), desc=d)
    lens = np.diff(A.row_offsets)
    assert d.counters.matrix_entries_read == lens[4] + lens[6] + lens[7]
    d = gb.Descriptor()
    out = gb.spmv_pull(B, A, ones, mask=gb.vector_fill(8, 0, dtype=np.int64), desc=d)
    assert d.counters.matrix_entries_read == 0 and out.nvals == 0
    d = gb.Descriptor()
    d.toggle("inp0")
    gb.spmspv_push(B, A, gb.vector_build([0, 2, 3], [1, 1, 1], 8), desc=d)
    assert d.counters.semiring_multiplies == 8
    w = gb.spmspv_push(B, A, gb.vector_build([2], [1], 8))
    assert w.extract_tuples()[0].tolist() == A.row_indices[A.col_offsets[2]:A.col_offsets[3]].tolist()


def test_early_exit_reads_fewer(gb):
    rng = np.random.default_rng(23)
    A = rand_matrix(gb, rng, 24, 24, 0.4, low=1, high=1)
    u = rand_vector(gb, rng, 24, 20, low=1, high=1)
    B = gb.builtin_semiring("LogicalOrAnd")
    exact, eager = gb.Descriptor(), gb.Descriptor()
    eager.early_exit = True
    w1 = gb.spmv_pull(B, A, u.to_dense(0), desc=exact)
    w2 = gb.spmv_pull(B, A, u.to_dense(0), desc=eager)
    assert np.array_equal(w1.values, w2.values)
    assert eager.counters.matrix_entries_read <= exact.counters.matrix_entries_read == A.nnz


def test_format_contracts(gb):
    A = eight(gb)
    B = gb.builtin_semiring("LogicalOrAnd")
    with pytest.raises(gb.FormatError):
        gb.spmv_pull(B, A, gb.vector_build([0], [1], 8))
    with pytest.raises(gb.FormatError):
        gb.spmspv_push(B, A, gb.vector_fill(8, 1, dtype=np.int64))
    with pytest.raises(gb.FormatError):
        gb.spmspv_push(B, gb.matrix_build([(0, 1, 1)], 2, 2, build_csc=False), gb.vector_build([0], [1], 2))


def test_mask_rules(gb):
    A = gb.matrix_build([(0, 1, 1), (1, 0, 1), (1, 2, 1), (2, 1, 1)], 3, 3)
    w = gb.mxv(gb.builtin_semiring("LogicalOrAnd"), A, gb.vector_fill(3, 1, dtype=np.int64),
               mask=gb.vector_build([0, 1], [1, 0], 3))
    assert w.extract_tuples()[0].tolist() == [0]  # a stored 0 blocks
    rng = np.random.default_rng(32)
    sr = gb.builtin_semiring("MinPlus")
    for _ in range(6):
        A = rand_matrix(gb, rng, 14, 14, 0.4)
        u = rand_vector(gb, rng, 14, int(rng.integers(0, 15)))
        mask = rand_mask(gb, rng, 14, dense=True)
        d = gb.Descriptor()
        d.toggle("mask")
        neg = gb.Vector.dense_of((mask.values == 0).astype(np.int64), 0)
        same(gb.mxv(sr, A, u, mask=mask, desc=d), *gb.mxv(sr, A, u, mask=neg).extract_tuples())


def test_decide_direction_cases(gb):
    def graph(nnz, nrows):
        rows = np.repeat(np.arange(nrows), nnz // nrows)
        cols = np.arange(nnz) % nrows
        return gb.SparseMatrix.from_tuples(rows, cols, np.ones(nnz, np.int64), nrows, nrows)
    A = graph(1000, 100)
    assert A.nnz == 1000
    rng = np.random.default_rng(1)
    for k, est, ch in [(5, 50, "push"), (11, 110, "pull"), (10, 100, "push")]:
        d = gb.decide_direction(rand_vector(gb, rng, 100, k), A)
        assert d.estimated_frontier_edges == est and d.chosen == ch
    assert gb.decide_direction(gb.Vector.empty(100), A).chosen == "push"
    assert gb.decide_direction(gb.vector_fill(4, 1, dtype=np.int64), gb.matrix_build([], 4, 4)).chosen == "push"


def test_mxm_masked_behaviours(gb):
    PT = gb.builtin_semiring("PlusMultiplies")
    K3 = gb.matrix_build([(1, 0, 1), (2, 0, 1), (2, 1, 1)], 3, 3)
    d = gb.Descriptor()
    d.toggle("inp1")
    C = gb.mxm_masked(PT, K3, K3, mask=K3, desc=d)
    assert C.nnz == 1 and C.extract_tuples()[2].tolist() == [1]
    A = gb.matrix_build([(i, j, 1) for i in range(4) for j in range(4) if i != j], 4, 4)
    assert gb.mxm_masked(PT, A, A, mask=gb.matrix_build([], 4, 4)).nnz == 0
    rng = np.random.default_rng(43)
    for _ in range(5):
        A = rand_matrix(gb, rng, 16, 16, 0.5)
        M = rand_matrix(gb, rng, 16, 16, 0.2, low=1, high=1)
        assert gb.mxm_masked(PT, A, A, mask=M).nnz <= M.nnz
    with pytest.raises(gb.ShapeError):
        gb.mxm_masked(PT, rand_matrix(gb, rng, 4, 4, 0.5), rand_matrix(gb, rng, 5, 5, 0.5),
                      mask=rand_matrix(gb, rng, 4, 4, 0.5))
    d = gb.Descriptor()
    d.toggle("mask")
    with pytest.raises(ValueError):
        gb.mxm_masked(PT, A, A, mask=M, desc=d)


def test_elementwise_behaviours(gb):
    P = gb.builtin_monoid("Plus")
    w = gb.ewise_add(P, gb.vector_build([0], [1], 4), gb.vector_build([1], [2], 4))
    assert [a.tolist() for a in w.extract_tuples()] == [[0, 1], [1, 2]]
    w = gb.ewise_add(gb.builtin_monoid("Minimum"), gb.vector_build([0], [1], 4), gb.vector_build([0], [3], 4))
    assert w.extract_tuples()[1].tolist() == [1]
    w = gb.ewise_add(gb.builtin_semiring("PlusMultiplies"), gb.vector_fill(2, 0.5), (1.0 - 0.85) / 2)
    assert np.allclose(w.values, [0.575, 0.575])
    w = gb.ewise_mult(gb.builtin_monoid("Multiplies"), gb.vector_build([0, 1], [2, 3], 4), gb.vector_build([1, 2], [5, 7], 4))
    assert [a.tolist() for a in w.extract_tuples()] == [[1], [15]]
    v = gb.Vector.dense_of(np.array([0.0, 4.0, np.inf]), np.inf)
    flags = gb.ewise_mult(gb.builtin_semiring("PlusLess"), v, gb.vector_fill(3, np.finfo(np.float64).max))
    assert float(gb.reduce(P, flags)) == 2.0
    with pytest.raises(gb.ShapeError):
        gb.ewise_add(P, gb.vector_fill(3, 1), gb.vector_fill(4, 1))


def test_assign_scatter_gather(gb):
    v = gb.vector_fill(8, 0, dtype=np.int64)
    gb.assign(v, 2, mask=gb.vector_build([0, 2, 3], [1, 1, 1], 8))
    assert v.values.tolist() == [2, 0, 2, 2, 0, 0, 0, 0]
    v = gb.vector_fill(4, 7, dtype=np.int64)
    gb.assign(v, 9, mask=gb.Vector.empty(4))
    assert v.values.tolist() == [7, 7, 7, 7]
    v = gb.vector_fill(4, 0, dtype=np.int64)
    d = gb.Descriptor()
    d.toggle("mask")
    gb.assign(v, 5, mask=gb.vector_build([1], [1], 4), desc=d)
    assert v.values.tolist() == [5, 0, 5, 5]
    w = gb.vector_fill(3, 100, dtype=np.int64)
    gb.assign_scatter(w, values=gb.Vector.dense_of(np.array([7, 4, 9]), -1),
                      indices=gb.Vector.dense_of(np.array([1, 1, 1]), -1))
    assert w.values.tolist() == [100, 4, 100]
    with pytest.raises(IndexError):
        gb.assign_scatter(gb.vector_fill(3, 0, dtype=np.int64), values=gb.vector_build([0], [1], 3),
                          indices=gb.vector_build([0], [5], 3))
    w = gb.Vector.empty(3)
    gb.extract_gather(w, gb.Vector.dense_of(np.array([1, 0, 0]), -1), gb.Vector.dense_of(np.array([1, 0, 0]), -1))
    assert w.values.tolist() == [0, 1, 1]
    with pytest.raises(IndexError):
        gb.extract_gather(gb.Vector.empty(3), gb.Vector.dense_of(np.arange(3), -1),
                          gb.Vector.dense_of(np.array([0, 1, 7]), -1))


def test_apply_reduce_transpose(gb):
    u = gb.Vector.dense_of(np.array([1.0, 2.0, 3.0]), 0.0)
    w = gb.apply(lambda x: x * 10, u, mask=gb.vector_build([0, 2], [1, 1], 3))
    assert [a.tolist() for a in w.extract_tuples()] == [[0, 2], [10.0, 30.0]]
    P = gb.builtin_monoid("Plus")
    assert int(gb.reduce(P, gb.vector_build([0, 3, 5], [1, 2, 3], 8))) == 6
    assert int(gb.reduce(P, gb.Vector.empty(8))) == 0
    path = gb.matrix_build([(0, 1, 1), (1, 0, 1), (1, 2, 1), (2, 1, 1)], 3, 3)
    assert gb.reduce_rows(P, path).values.tolist() == [1, 2, 1]
    A = eight(gb)
    r, c, v = gb.transpose(A).extract_tuples()
    er, ec, ev = A.extract_tuples()
    o = np.lexsort((er, ec))
    assert np.array_equal(r, ec[o]) and np.array_equal(c, er[o]) and np.array_equal(v, ev[o])


@pytest.mark.parametrize("part", ["nonzero", "row"])
def test_partition_invariance(gb, part):
    rng = np.random.default_rng(61)
    A = rand_matrix(gb, rng, 50, 50, 0.2)
    u = rand_vector(gb, rng, 50, 30).to_dense(0)
    PT = gb.builtin_semiring("PlusMultiplies")
    base = gb.spmv_pull(PT, A, u)
    for workers in (1, 2, 4, 7):
        d = gb.Descriptor(num_workers=workers, partition=gb.Partition(part))
        assert np.array_equal(base.values, gb.spmv_pull(PT, A, u, desc=d).values)


def test_containers(gb):
    A = gb.matrix_build([(0, 1, 1), (1, 0, 1), (1, 2, 1), (2, 1, 1)], 3, 3)
    assert A.nnz == 4 and list(zip(*A.extract_tuples())) == [(0, 1, 1), (1, 0, 1), (1, 2, 1), (2, 1, 1)]
    B = gb.matrix_build([(0, 0, 2), (0, 0, 3)], 1, 1, dedup=gb.builtin_monoid("Plus"))
    assert B.nnz == 1 and B.extract_element(0, 0) == 5
    B = gb.matrix_build([(0, 0, 2), (0, 0, 3)], 1, 1, dedup=gb.builtin_monoid("Minimum"))
    assert B.extract_element(0, 0) == 2
    assert gb.matrix_build([], 2, 2).row_offsets.tolist() == [0, 0, 0]
    with pytest.raises(IndexError):
        gb.matrix_build([(0, 5, 1)], 3, 3)
    with pytest.raises(IndexError):
        gb.matrix_build([(-1, 0, 1)], 3, 3)
    M = gb.matrix_build([(0, 1, 7)], 2, 2)
    assert M.extract_element(0, 1) == 7 and M.extract_element(1, 0) is None
    M.set_element(1, 0, 4)
    M.set_element(0, 1, 9)
    assert M.extract_element(1, 0) == 4 and M.extract_element(0, 1) == 9 and M.nnz == 2
    D = M.dup()
    D.set_element(0, 1, 1)
    assert M.extract_element(0, 1) == 9
    M.clear()
    assert M.nnz == 0
    rng = np.random.default_rng(12)
    for _ in range(10):
        n = int(rng.integers(1, 25))
        k = int(rng.integers(0, 3 * n))
        A = gb.SparseMatrix.from_tuples(rng.integers(0, n, k), rng.integers(0, n, k), rng.integers(1, 9, k), n, n)
        rr, cr, vr = A.extract_tuples()
        cc = np.repeat(np.arange(n), np.diff(A.col_offsets))
        o = np.lexsort((cc, A.row_indices))
        assert np.array_equal(A.row_indices[o], rr) and np.array_equal(cc[o], cr)
        assert np.array_equal(A.csc_values[o], vr)
    # build oracle with duplicates folded by Plus
    rows, cols, vals = rng.integers(0, 64, 10000), rng.integers(0, 64, 10000), rng.integers(1, 100, 10000)
    A = gb.SparseMatrix.from_tuples(rows, cols, vals, 64, 64)
    expect = {}
    for r, c, v in zip(rows, cols, vals):
        expect[(r, c)] = expect.get((r, c), 0) + v
    gr, gc, gv = A.extract_tuples()
    assert sorted(expect) == list(zip(gr, gc))
    assert all(expect[(r, c)] == v for r, c, v in zip(gr, gc, gv))


def test_vector_surface(gb):
    f = gb.vector_build([1], [1], 8)
    assert f.is_sparse and f.nvals == 1 and f.extract_element(1) == 1
    v = gb.vector_fill(4, 0)
    assert not v.is_sparse and v.nvals == 0 and v.values.tolist() == [0, 0, 0, 0]
    with pytest.raises(ValueError):
        gb.vector_build([1, 1], [1, 2], 4)
    with pytest.raises(IndexError):
        gb.vector_build([4], [1], 4)
    v = gb.vector_build([3, 0, 2], [30, 0, 20], 5)
    assert v.indices.tolist() == [0, 2, 3] and v.values.tolist() == [0, 20, 30]
    assert gb.vector_fill(4, 0).extract_element(2) is None
    w = gb.vector_build([1], [5], 3)
    x = w.dup()
    x.set_element(1, 9)
    assert w.extract_element(1) == 5
    w.clear()
    assert w.nvals == 0
    v = gb.vector_build([1, 5], [1, 5], 8)
    v.set_element(3, 3)
    assert v.indices.tolist() == [1, 3, 5]
    v.set_element(5, 50)
    assert v.values.tolist() == [1, 3, 50]
    assert gb.vector_convert(gb.vector_build([1], [5], 3), "dense", 0).values.tolist() == [0, 5, 0]
    s = gb.vector_convert(gb.Vector.dense_of(np.array([0, 5, 0]), 0), "sparse", 0)
    assert s.indices.tolist() == [1] and s.values.tolist() == [5]
    assert gb.vector_convert(gb.Vector.dense_of(np.array([7, 7]), 0), "sparse", 7).nvals == 0
    rng = np.random.default_rng(5)
    for _ in range(20):
        n = int(rng.integers(1, 40))
        k = int(rng.integers(0, n + 1))
        idx = np.sort(rng.choice(n, size=k, replace=False))
        v = gb.vector_build(idx, rng.integers(1, 50, size=k), n)
        back = v.to_dense(0).to_sparse(0)
        assert np.array_equal(back.indices, v.indices) and np.array_equal(back.values, v.values)


def test_user_defined_semiring_runs_on_device(gb):
    op_max = gb.BinaryOp("umax", max, np.maximum)
    op_mul = gb.BinaryOp("utimes", lambda a, b: a * b, np.multiply)
    sr = gb.Semiring(gb.Monoid(op_max, -np.inf), op_mul, "custom")
    rng = np.random.default_rng(9)
    A = rand_matrix(gb, rng, 12, 12, 0.4, dtype=np.float64)
    u = rand_vector(gb, rng, 12, 8, dtype=np.float64)
    same(gb.mxv(sr, A, u), *dense_oracle(sr, A, u))
