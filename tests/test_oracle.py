"""Pin the numpy oracle (oracle/port.py) to the reference goldens.

CPU only.  The goldens were produced by the real reference package
(tests/golden/make_golden.py); the port must reproduce every one of them
before any GPU result is compared against it.  The C oracle (oracle/cgraph.c,
the checker at s16 and above) is pinned by tests/test_oracle_pins.py.
"""

import hashlib

import numpy as np
import pytest

from golden_io import canonical, kernel_cases, load_json, mat_arrays, same_values, vec_arrays
from oracle import port

MONOID_OPS = ["Plus", "Multiplies", "Minimum", "Maximum", "LogicalOr", "LogicalAnd"]


def to_vec(j):
    if j is None:
        return None
    size, idx, vals, zero = vec_arrays(j)
    return port.Vec(size, idx, vals, zero)


def to_mat(j):
    r, c, v, nr, nc, csc = mat_arrays(j)
    return port.mat_from_tuples(r, c, v, nr, nc, csc=csc, dtype=v.dtype)


def check_vec(got, want_json):
    size, idx, vals, zero = vec_arrays(want_json)
    wi, wv = canonical(size, idx, vals, zero)
    gi, gv = got.tuples()
    assert np.array_equal(gi, wi)
    assert gv.dtype == wv.dtype
    assert same_values(gv, wv)
    assert got.sparse == want_json["sparse"]


def desc_of(case, tattr=None):
    d = port.Desc()
    d.complement = case.get("mask_mode") == "complement"
    if tattr == "inp0":
        d.transpose0 = case["transpose"]
    elif tattr == "inp1":
        d.transpose1 = case["transpose"]
    d.direction = case.get("direction", "auto")
    d.early_exit = case.get("early_exit", False)
    return d


MV = kernel_cases("mv")


@pytest.mark.parametrize("k", range(0, len(MV), 1))
def test_mv_cases(k):
    c = MV[k]
    A, u, mask = to_mat(c["A"]), to_vec(c["u"]), to_vec(c["mask"])
    op = c["op"]
    d = desc_of(c, "inp1" if op == "vxm" else "inp0")
    try:
        if op == "mxv":
            w = port.mxv(c["semiring"], A, u, mask, d)
        elif op == "vxm":
            w = port.vxm(c["semiring"], u, A, mask, d)
        elif op == "pull":
            w = port.pull(c["semiring"], A, u, mask, d, d.transpose0)
        else:
            w = port.push(c["semiring"], A, u, mask, d, d.transpose0)
        err = None
    except ValueError:
        err = "ShapeError"
    except RuntimeError:
        err = "FormatError"
    assert err == c["error"]
    if err is None:
        check_vec(w, c["out"])
        assert d.counters.as_list() == c["counters"]
        assert [x[:3] for x in d.log] == [x[:3] for x in c["log"]]
        assert [x[3] for x in d.log] == [x[3] for x in c["log"]]


def test_mxm_cases():
    for c in kernel_cases("mxm"):
        A, B, M = to_mat(c["A"]), to_mat(c["B"]), to_mat(c["M"])
        d = port.Desc(transpose1=c["transpose_b"])
        C = port.mxm_masked(c["semiring"], A, B, M, d)
        r, cc, v, *_ = mat_arrays(c["out"])
        gr, gc, gv = C.tuples()
        assert np.array_equal(gr, r) and np.array_equal(gc, cc)
        assert same_values(gv, v.astype(gv.dtype))
        assert d.counters.as_list() == c["counters"]


OPNAMES = {"Plus", "Minus", "Multiplies", "Minimum", "Maximum", "Less", "NotEqualTo",
           "LogicalOr", "LogicalAnd", "SelectSecond"}


def resolve_op(c, which):
    """(op name, identity monoid or None) for ewise_add / ewise_mult."""
    if c["opkind"] == "semiring":
        add, mul = port.SEMIRINGS[c["op"]]
        return (add, add) if which != "mult" else (mul, None)
    if c["opkind"] == "monoid":
        return c["op"], c["op"]
    return c["op"], None


def test_ewise_cases():
    for c in kernel_cases("ewise"):
        u, v, mask = to_vec(c["u"]), to_vec(c["v"]), to_vec(c["mask"])
        d = port.Desc(complement=c["mask_mode"] == "complement")
        op, ident = resolve_op(c, c["which"])
        try:
            if c["which"] == "add":
                w = port.ewise_add(op, u, v, mask, d, identity=ident)
            elif c["which"] == "mult":
                w = port.ewise_mult(op, u, v, mask, d)
            else:
                scalar = np.float64(c["scalar"]) if u.vals.dtype.kind == "f" else np.int64(c["scalar"])
                w = port.ewise_add(op, u, scalar, mask, d, identity=ident)
            err = None
        except TypeError:
            err = "TypeError"
        assert err == c["error"], c
        if err is None:
            check_vec(w, c["out"])


def test_assign_family_cases():
    for c in kernel_cases("assign"):
        w, mask = to_vec(c["w"]), to_vec(c["mask"])
        d = port.Desc(complement=c["mask_mode"] == "complement")
        v = c["variant"]
        if v == "assign":
            out = port.assign(w, c["value"], mask, d, c["indices"])
        elif v == "scatter":
            out = port.assign_scatter(w, to_vec(c["values"]), to_vec(c["targets"]), mask, d)
        elif v == "gather":
            out = port.extract_gather(w, to_vec(c["src"]), to_vec(c["idx"]), mask, d)
        else:
            out = port.apply(lambda x: x * c["scale"] + c["shift"], w, mask, d)
        assert c["error"] is None
        check_vec(out, c["out"])


def test_reduce_cases():
    for c in kernel_cases("reduce"):
        u = to_vec(c["u"])
        r = port.reduce(c["monoid"], u)
        assert same_values(np.asarray(r), np.asarray(c["out"], dtype=r.dtype))
        A = to_mat(c["A"])
        check_vec(port.reduce_rows(c["monoid"], A), c["rows"])
        s = port.reduce_scalar_matrix(c["monoid"], A)
        assert same_values(np.asarray(s), np.asarray(c["scalar"], dtype=s.dtype))


# ---------------------------------------------------------------------------
# input pipeline and algorithms
# ---------------------------------------------------------------------------


def csr_digest(rp, ci):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(rp, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(ci, dtype=np.int64).tobytes())
    return h.hexdigest()


def digest_vec(idx, vals):
    """cli.py:148-156."""
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(idx).tobytes())
    h.update(np.ascontiguousarray(np.round(np.asarray(vals, dtype=np.float64), 9)).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("key", ["rmat_s8", "rmat_s10", "rmat_s12", "uniform_s10"])
def test_port_generator_bit_exact(key):
    g = load_json("rmat_graphs.json")["graphs"][key]
    kw = dict(a=0.25, b=0.25, c=0.25, d=0.25) if key.startswith("uniform") else {}
    rp, ci, n = port.rmat_csr(g["scale"], **kw)
    assert ci.size == g["nnz"]
    assert csr_digest(rp, ci) == g["csr"]
    if g["weights"] is not None:
        w = port.upper_weights(rp, ci, seed=1)
        assert hashlib.sha256(w.tobytes()).hexdigest() == g["weights"]


def test_port_generator_matches_s10_arrays():
    z = np.load(f"{__import__('golden_io').GOLDEN}/rmat_s10.npz")
    rp, ci, n = port.rmat_csr(10)
    assert np.array_equal(rp, z["row_offsets"]) and np.array_equal(ci, z["col_indices"])
    assert np.array_equal(port.upper_weights(rp, ci), z["weights"])


def graph(scale, weighted=False):
    rp, ci, n = port.rmat_csr(scale)
    vals = port.upper_weights(rp, ci) if weighted else np.ones(ci.size, np.int64)
    return port.mat_from_csr(rp, ci, vals, n)


@pytest.mark.parametrize("s", [8, 10, 12])
def test_port_bfs(s):
    g = load_json("algorithms.json")[f"bfs_s{s}"]
    d = port.Desc()
    lv = port.bfs(graph(s), 0, d)
    assert digest_vec(*lv.tuples()) == g["digest"]
    assert [x[0] for x in d.log] == [x[0] for x in g["trace"]]
    assert [x[1:3] for x in d.log] == [x[1:3] for x in g["trace"]]


@pytest.mark.parametrize("s", [8, 10])
def test_port_sssp_cc_tc(s):
    gold = load_json("algorithms.json")
    W = graph(s, weighted=True)
    dist = port.sssp(W, 0)
    assert digest_vec(*dist.tuples()) == gold[f"sssp_s{s}"]["digest"]
    A = graph(s)
    cc = port.connected_components(A)
    assert digest_vec(*cc.tuples()) == gold[f"cc_s{s}"]["digest"]
    assert port.triangle_count_fast(A) == gold[f"tc_s{s}"]["count"]


def test_port_pagerank_s10():
    import os
    from golden_io import GOLDEN
    want = np.load(os.path.join(GOLDEN, "pr_s10.npy"))
    got = port.pagerank(graph(10), eps=1e-300, max_iters=20).vals
    assert np.abs(got - want).sum() <= 1e-12
