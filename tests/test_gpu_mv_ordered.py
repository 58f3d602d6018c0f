"""The alternative pull SpMV kernels -- the row-binned pull (gb_mxv_pull_binned,
the default for masked pulls and Partition.ROW_SPLIT) and the pull on the
degree-ordered layout (gb_mxv_pull_ordered) -- against the same call through
the edge-balanced row tiles (gb_mxv_pull, itself pinned to the reference's
kernel cases in test_gpu_kernels.py): identical outputs for
order-independent folds, equal within 1e-12 for float sums, identical work
counters (kernels.py:153-229), over every builtin semiring, mxv and vxm,
no / normal / complemented masks, symmetric and directed matrices."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SEMIRINGS = ["PlusMultiplies", "LogicalOrAnd", "MinPlus", "MaxPlus", "MinMultiplies",
             "MinimumSelectSecond", "PlusLess", "MinimumNotEqualTo"]


@pytest.fixture(scope="module")
def gb():
    import paper_1908_01407_b200 as gb
    return gb


@pytest.fixture(scope="module")
def graphs(gb):
    sym = gb.io.rmat_matrix(14, weighted=True)
    rng = np.random.default_rng(11)
    n = 3000
    r = rng.integers(0, n, 40000)
    c = (r * 7 + rng.integers(0, 50, r.size) ** 2) % n   # skewed, directed
    v = rng.integers(1, 9, r.size).astype(np.float64)
    directed = gb.SparseMatrix.from_tuples(r, c, v, n, n)
    pattern = gb.io.rmat_matrix(13)
    return {"sym_f64": sym, "directed_f64": directed, "pattern_i64": pattern}


# (GB_MV_ORDERED, GB_MV_BINS, GB_MV_STRIPE_BYTES): "stripes" cuts a
# structure-only matrix into 8 KB-of-vector column stripes (many stripes)
IMPLS = {"tiles": ("0", "0", 0), "ordered": ("1", "0", 0), "bins": ("0", "1", 0),
         "stripes": ("0", "1", 8192)}


def _use(monkeypatch, impl):
    from paper_1908_01407_b200 import kernels
    ordered, bins, stripe = IMPLS[impl]
    monkeypatch.setattr(kernels, "_MV_ORDERED", ordered)
    monkeypatch.setattr(kernels, "_MV_BINS", bins)
    monkeypatch.setattr(kernels, "_MV_STRIPE_BYTES", stripe)
    monkeypatch.setattr(kernels, "_MV_STRIPE_SKEW", 1.0)   # stripe skewed graphs too


def _run(gb, monkeypatch, impl, sr, A, u, mask, desc_kw, vxm):
    _use(monkeypatch, impl)
    d = gb.Descriptor(direction=gb.Direction.FORCE_PULL, **desc_kw)
    w = gb.vxm(sr, u, A, mask=mask, desc=d) if vxm else gb.mxv(sr, A, u, mask=mask, desc=d)
    c = d.counters
    return (w.to_dense(w.zero).values, (c.matrix_entries_read, c.semiring_multiplies,
                                        c.semiring_adds))


@pytest.mark.parametrize("name", SEMIRINGS)
@pytest.mark.parametrize("gname", ["sym_f64", "directed_f64", "pattern_i64"])
@pytest.mark.parametrize("vxm", [False, True])
@pytest.mark.parametrize("impl", ["ordered", "bins", "stripes"])
def test_pull_variants_equal_row_tiles(gb, graphs, monkeypatch, name, gname, vxm, impl):
    A = graphs[gname]
    n = A.nrows
    rng = np.random.default_rng(5)
    dt = np.int64 if gname.endswith("i64") else np.float64
    x = rng.integers(-3, 9, n).astype(dt)
    x[rng.random(n) < 0.2] = 0
    u = gb.Vector.dense_of(x, 0)
    m = gb.Vector.dense_of((rng.random(n) < 0.5).astype(np.int64), 0)
    sr = gb.builtin_semiring(name)
    for mask, kw in ((None, {}), (m, {}), (m, {"mask_mode": gb.MaskMode.COMPLEMENT})):
        want, wc = _run(gb, monkeypatch, "tiles", sr, A, u, mask, kw, vxm)
        got, gc = _run(gb, monkeypatch, impl, sr, A, u, mask, kw, vxm)
        assert gc == wc
        if dt == np.float64 and name.startswith("Plus"):
            np.testing.assert_allclose(got, want, rtol=1e-12, atol=0)
        else:
            assert np.array_equal(got, want)


@pytest.mark.parametrize("impl", ["ordered", "bins", "stripes"])
def test_pull_variants_s20_against_torch(gb, monkeypatch, impl):
    """Size-independent check at s20: torch index_add reference and exact
    counters."""
    from paper_1908_01407_b200.containers import Vector
    _use(monkeypatch, impl)
    if impl == "stripes":
        from paper_1908_01407_b200 import kernels
        monkeypatch.setattr(kernels, "_MV_STRIPE_BYTES", 2 << 20)   # 4 stripes at s20
    A = gb.io.rmat_matrix(20)
    assert A.nnz >= 1 << 24
    n = A.nrows
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 0.25
    mb = (torch.rand(n, device="cuda", generator=g) < 0.5).to(torch.int64)
    d = gb.Descriptor(mask_mode=gb.MaskMode.COMPLEMENT, direction=gb.Direction.FORCE_PULL)
    w = gb.mxv(gb.builtin_semiring("PlusMultiplies"), A, Vector._wrap(n, None, x, 0.0, np.float64),
               mask=Vector._wrap(n, None, mb, 0, np.int64), desc=d)
    if impl == "ordered":
        assert A._csr._mv_ordered, "the s20 call did not take the ordered layout"
    elif impl == "stripes":
        assert A._csr._stripes is not None and A._csr._stripes[0] == 4
    else:
        assert A._csr._bins is not None, "the s20 call did not take the row bins"
    deg = torch.diff(A._csr.offsets)
    rows = torch.repeat_interleave(torch.arange(n, device="cuda"), deg)
    allowed = mb == 0
    keep = allowed[rows]
    ref = torch.zeros(n, dtype=torch.float64, device="cuda")
    ref.index_add_(0, rows[keep], x[A._csr.indices.long()[keep]])
    got = w.to_dense(0.0)._vals
    assert float(((got - ref).abs() / ref.abs().clamp_min(1e-300)).max()) <= 1e-12
    reads = int(deg[allowed].sum())
    assert d.counters.matrix_entries_read == reads
    assert d.counters.semiring_adds == reads - int(((deg > 0) & allowed).sum())


@pytest.mark.parametrize("impl", ["tiles", "bins"])
def test_row_split_partition_and_ragged_rows(gb, monkeypatch, impl):
    """Partition.ROW_SPLIT takes the row bins; rows of every bin length
    (empty, 1..16, 17..512, > 512 spanning partial and full 512-entry tiles)
    against a float64 numpy reference."""
    from paper_1908_01407_b200 import kernels
    monkeypatch.setattr(kernels, "_MV_BINS", "0" if impl == "tiles" else "")
    rng = np.random.default_rng(2)
    n = 4096
    lens = np.concatenate([np.zeros(50, int), rng.integers(1, 17, 800), rng.integers(17, 513, 300),
                           [513, 1024, 1500, 2999, 4096, 700, 4000]])
    lens = np.concatenate([lens, np.zeros(n - lens.size, int)])
    rng.shuffle(lens)
    rows = np.repeat(np.arange(n), lens)
    cols = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens if k])
    vals = rng.integers(1, 5, rows.size).astype(np.float64)
    A = gb.SparseMatrix.from_tuples(rows, cols, vals, n, n)
    x = rng.random(n)
    m = (rng.random(n) < 0.3).astype(np.int64)
    d = gb.Descriptor(direction=gb.Direction.FORCE_PULL, partition=gb.Partition.ROW_SPLIT,
                      mask_mode=gb.MaskMode.COMPLEMENT)
    w = gb.mxv(gb.builtin_semiring("PlusMultiplies"), A, gb.Vector.dense_of(x, 0.0),
               mask=gb.Vector.dense_of(m, 0), desc=d).to_dense(0.0).values
    ref = np.zeros(n)
    keep = m[rows] == 0
    np.add.at(ref, rows[keep], vals[keep] * x[cols[keep]])
    np.testing.assert_allclose(w, ref, rtol=1e-12, atol=1e-300)
    assert d.counters.matrix_entries_read == int(keep.sum())
    assert d.counters.semiring_adds == int(keep.sum()) - int(((lens > 0) & (m == 0)).sum())
    if impl == "bins":
        assert A._csr._bins is not None


def test_stripes_chosen_for_regular_graphs_only(gb, monkeypatch):
    """The default dispatch stripes a uniform graph whose vector exceeds the
    stripe budget and leaves a skewed R-MAT graph unstriped."""
    from paper_1908_01407_b200 import kernels
    monkeypatch.setattr(kernels, "_MV_STRIPE_BYTES", 64 << 10)   # 8 K entries per stripe
    U = gb.io.rmat_matrix(14, a=.25, b=.25, c=.25, d=.25)
    R = gb.io.rmat_matrix(14)
    assert kernels._stripe_count(U._csr) == 2 and kernels._stripe_count(R._csr) == 1
    n = U.nrows
    x = np.random.default_rng(1).random(n)
    m = gb.Vector.dense_of((np.arange(n) % 3 == 0).astype(np.int64), 0)
    d = gb.Descriptor(direction=gb.Direction.FORCE_PULL, mask_mode=gb.MaskMode.COMPLEMENT)
    w = gb.mxv(gb.builtin_semiring("PlusMultiplies"), U, gb.Vector.dense_of(x, 0.0), mask=m, desc=d)
    assert U._csr._stripes is not None
    rp, ci = U.row_offsets, U.col_indices
    rows = np.repeat(np.arange(n), np.diff(rp))
    keep = (np.arange(n) % 3 != 0)[rows]
    ref = np.zeros(n)
    np.add.at(ref, rows[keep], x[ci[keep]])
    np.testing.assert_allclose(w.to_dense(0.0).values, ref, rtol=1e-12, atol=0)
