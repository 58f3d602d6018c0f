"""The push SpMSpV's dense-accumulator path (order-independent folds: integer
plus / times, min, max, logical or / and; f64 min, max, or, and) against the
stable sort-and-fold path it replaces (GB_PUSH_SORTED=1, the reference's
argsort(kind="stable") + reduceat order): identical entries, values and work
counters, with and without masks, over skewed and uniform graphs."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SEMIRINGS = ["PlusMultiplies", "LogicalOrAnd", "MinPlus", "MaxPlus", "MinMultiplies",
             "MinimumSelectSecond", "MinimumNotEqualTo", "PlusLess"]


@pytest.fixture(scope="module")
def gb():
    import paper_1908_01407_b200 as gb
    return gb


def _push(gb, sr, A, u, mask, sorted_path):
    d = gb.Descriptor(direction=gb.Direction.FORCE_PUSH)
    if mask is not None:
        d.mask_mode = gb.MaskMode.COMPLEMENT
    if sorted_path:
        os.environ["GB_PUSH_SORTED"] = "1"
    try:
        w = gb.vxm(gb.builtin_semiring(sr), u, A, mask=mask, desc=d)
    finally:
        os.environ.pop("GB_PUSH_SORTED", None)
    idx, vals = w.extract_tuples()
    return np.asarray(idx), np.asarray(vals), d.counters


@pytest.mark.parametrize("sr", SEMIRINGS)
@pytest.mark.parametrize("dtype", [np.int64, np.float64])
@pytest.mark.parametrize("graph", ["rmat", "uniform"])
def test_accumulator_push_equals_sorted(gb, sr, dtype, graph):
    rng = np.random.default_rng(len(sr) * 7 + (dtype == np.float64))
    a = .57 if graph == "rmat" else .25
    b = .19 if graph == "rmat" else .25
    A = gb.io.rmat_matrix(12, a=a, b=b, c=b, d=1 - a - 2 * b)
    n = A.nrows
    if dtype == np.float64:
        r, c = A.orient(False).offsets.cpu().numpy(), A.orient(False).indices.cpu().numpy()
        rows = np.repeat(np.arange(n), np.diff(r))
        vals = rng.integers(-3, 9, rows.size).astype(np.float64)
        A = gb.SparseMatrix.from_tuples(rows, c, vals, n, n)
    k = 600
    ids = np.sort(rng.choice(n, k, replace=False))
    uv = rng.integers(-4, 6, k).astype(dtype)
    u = gb.Vector.from_entries(ids, uv, n)
    mask = gb.Vector.from_entries(np.sort(rng.choice(n, n // 3, replace=False)),
                                  np.ones(n // 3, np.int64), n)
    for m in (None, mask):
        i1, v1, c1 = _push(gb, sr, A, u, m, False)
        i2, v2, c2 = _push(gb, sr, A, u, m, True)
        assert np.array_equal(i1, i2)
        assert np.array_equal(v1, v2)
        assert (c1.matrix_entries_read, c1.semiring_multiplies, c1.semiring_adds) == \
            (c2.matrix_entries_read, c2.semiring_multiplies, c2.semiring_adds)
