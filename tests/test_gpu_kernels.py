"""GPU parity of the unfused operator layer against the reference goldens.

Every case in tests/golden/kernel_cases.json was produced by the real
reference (make_golden.py): inputs, outputs, work counters and the direction
log.  The device kernels must reproduce all of them (floats to 1e-10 rel).
"""

import numpy as np
import pytest

from golden_io import canonical, kernel_cases, mat_arrays, same_values, vec_arrays

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gb():
    import paper_1908_01407_b200 as gb
    return gb


def to_vec(gb, j):
    if j is None:
        return None
    size, idx, vals, zero = vec_arrays(j)
    return gb.Vector(size, idx, vals, zero)


def to_mat(gb, j):
    r, c, v, nr, nc, csc = mat_arrays(j)
    return gb.SparseMatrix.from_tuples(r, c, v, nr, nc, build_csc=csc, dtype=v.dtype)


def check_vec(got, want_json):
    size, idx, vals, zero = vec_arrays(want_json)
    wi, wv = canonical(size, idx, vals, zero)
    gi, gv = got.extract_tuples()
    assert np.array_equal(gi, wi), (gi, wi)
    assert gv.dtype == wv.dtype, (gv.dtype, wv.dtype)
    assert same_values(gv, wv), (gv, wv)
    assert got.is_sparse == want_json["sparse"]


def make_desc(gb, case, tattr=None):
    d = gb.Descriptor()
    if case.get("mask_mode") == "complement":
        d.toggle("mask")
    if tattr and case.get("transpose"):
        d.toggle(tattr)
    d.direction = gb.Direction(case.get("direction", "auto"))
    d.early_exit = case.get("early_exit", False)
    return d


MV = kernel_cases("mv")


@pytest.mark.parametrize("chunk", range(16))
def test_mv_cases(gb, chunk):
    for c in MV[chunk::16]:
        sr = gb.builtin_semiring(c["semiring"])
        A, u, mask = to_mat(gb, c["A"]), to_vec(gb, c["u"]), to_vec(gb, c["mask"])
        op = c["op"]
        d = make_desc(gb, c, "inp1" if op == "vxm" else "inp0")
        try:
            if op == "mxv":
                w = gb.mxv(sr, A, u, mask=mask, desc=d)
            elif op == "vxm":
                w = gb.vxm(sr, u, A, mask=mask, desc=d)
            elif op == "pull":
                w = gb.spmv_pull(sr, A, u, mask=mask, desc=d)
            else:
                w = gb.spmspv_push(sr, A, u, mask=mask, desc=d)
            err = None
        except gb.ShapeError:
            err = "ShapeError"
        except gb.FormatError:
            err = "FormatError"
        assert err == c["error"], c
        if err is None:
            check_vec(w, c["out"])
            ct = d.counters
            assert [ct.matrix_entries_read, ct.semiring_multiplies, ct.semiring_adds] == c["counters"], c
            log = [[x.chosen, x.frontier_nvals, x.estimated_frontier_edges, x.threshold_edges]
                   for x in d.direction_log]
            assert log == c["log"]


def test_mxm_cases(gb):
    for c in kernel_cases("mxm"):
        sr = gb.builtin_semiring(c["semiring"])
        A, B, M = to_mat(gb, c["A"]), to_mat(gb, c["B"]), to_mat(gb, c["M"])
        d = gb.Descriptor()
        if c["transpose_b"]:
            d.toggle("inp1")
        C = gb.mxm_masked(sr, A, B, mask=M, desc=d)
        r, cc, v, *_ = mat_arrays(c["out"])
        gr, gc, gv = C.extract_tuples()
        assert np.array_equal(gr, r) and np.array_equal(gc, cc)
        assert same_values(gv, v.astype(gv.dtype))
        ct = d.counters
        assert [ct.matrix_entries_read, ct.semiring_multiplies, ct.semiring_adds] == c["counters"]


def resolve_op(gb, c):
    ops = {"Plus": gb.algebra.PLUS, "Minus": gb.algebra.MINUS, "Multiplies": gb.algebra.TIMES,
           "Minimum": gb.algebra.MIN, "Maximum": gb.algebra.MAX, "Less": gb.algebra.LESS,
           "NotEqualTo": gb.algebra.NOT_EQUAL, "LogicalOr": gb.algebra.LOGICAL_OR,
           "LogicalAnd": gb.algebra.LOGICAL_AND, "SelectSecond": gb.algebra.SECOND}
    if c["opkind"] == "semiring":
        return gb.builtin_semiring(c["op"])
    if c["opkind"] == "monoid":
        return gb.builtin_monoid(c["op"])
    return ops[c["op"]]


def test_ewise_cases(gb):
    for c in kernel_cases("ewise"):
        u, v, mask = to_vec(gb, c["u"]), to_vec(gb, c["v"]), to_vec(gb, c["mask"])
        d = gb.Descriptor()
        if c["mask_mode"] == "complement":
            d.toggle("mask")
        op = resolve_op(gb, c)
        try:
            if c["which"] == "add":
                w = gb.ewise_add(op, u, v, mask=mask, desc=d)
            elif c["which"] == "mult":
                w = gb.ewise_mult(op, u, v, mask=mask, desc=d)
            else:
                scalar = np.float64(c["scalar"]) if u.dtype.kind == "f" else np.int64(c["scalar"])
                w = gb.ewise_add(op, u, scalar, mask=mask, desc=d)
            err = None
        except TypeError:
            err = "TypeError"
        assert err == c["error"], c
        if err is None:
            check_vec(w, c["out"])


def test_assign_family_cases(gb):
    for c in kernel_cases("assign"):
        w, mask = to_vec(gb, c["w"]), to_vec(gb, c["mask"])
        d = gb.Descriptor()
        if c["mask_mode"] == "complement":
            d.toggle("mask")
        v = c["variant"]
        if v == "assign":
            out = gb.assign(w, c["value"], mask=mask, desc=d, indices=c["indices"])
        elif v == "scatter":
            out = gb.assign_scatter(w, to_vec(gb, c["values"]), to_vec(gb, c["targets"]),
                                    mask=mask, desc=d)
        elif v == "gather":
            out = gb.extract_gather(w, to_vec(gb, c["src"]), to_vec(gb, c["idx"]), mask=mask,
                                    desc=d)
        else:
            out = gb.apply(lambda x: x * c["scale"] + c["shift"], w, mask=mask, desc=d)
        check_vec(out, c["out"])


def test_reduce_cases(gb):
    for c in kernel_cases("reduce"):
        m = gb.builtin_monoid(c["monoid"])
        u = to_vec(gb, c["u"])
        r = gb.reduce(m, u)
        assert same_values(np.asarray(r), np.asarray(c["out"], dtype=np.asarray(r).dtype)), c
        A = to_mat(gb, c["A"])
        check_vec(gb.reduce_rows(m, A), c["rows"])
        s = gb.reduce_scalar_matrix(m, A)
        assert same_values(np.asarray(s), np.asarray(c["scalar"], dtype=np.asarray(s).dtype))
