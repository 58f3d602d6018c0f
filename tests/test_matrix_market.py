"""Matrix Market reader / writer (io.py:114-213) against the reference's own
reader on the same files (tests/golden/mm_cases.json, made by
tests/golden/make_mm_golden.py): identical edge lists, identical ParseError
messages and line numbers; writer round trips; a file read end to end into
a matrix and a BFS."""

import os

import numpy as np
import pytest

from golden_io import load_json

pytestmark = pytest.mark.gpu
CASES = load_json("mm_cases.json")


@pytest.fixture(scope="module")
def gb():
    import paper_1908_01407_b200 as gb
    return gb


@pytest.mark.parametrize("name", sorted(CASES))
def test_reader_matches_reference(gb, tmp_path, name):
    case = CASES[name]
    p = tmp_path / f"{name}.mtx"
    p.write_text(case["text"], encoding="ascii")
    if "error" in case:
        with pytest.raises(gb.ParseError) as ei:
            gb.read_matrix_market(str(p))
        assert str(ei.value) == case["error"]
        assert ei.value.line == case["line"]
        assert isinstance(ei.value, ValueError)   # errors.py: ParseError(GraphAlgError, ValueError)
        return
    e = gb.read_matrix_market(str(p))
    assert e.n == case["n"]
    assert e.src.tolist() == case["src"] and e.dst.tolist() == case["dst"]
    assert e.src.dtype == np.int64 and e.dst.dtype == np.int64
    if case["weight"] is None:
        assert e.weight is None
    else:
        assert e.weight.tolist() == case["weight"]


@pytest.mark.parametrize("weighted", [False, True])
def test_writer_round_trip(gb, tmp_path, weighted):
    rng = np.random.default_rng(1)
    n = 300
    src, dst = rng.integers(0, n, 1000), rng.integers(0, n, 1000)
    w = np.round(rng.random(1000) * 10, 3) if weighted else None
    e = gb.EdgeList(src, dst, n, w)
    p = str(tmp_path / "g.mtx")
    gb.write_matrix_market(p, e, comment="round trip")
    text = open(p).read().splitlines()
    assert text[0] == ("%%MatrixMarket matrix coordinate "
                       f"{'real' if weighted else 'pattern'} general")
    assert text[1] == "%round trip" and text[2] == f"{n} {n} 1000"
    back = gb.read_matrix_market(p)
    assert back.n == n and np.array_equal(back.src, src) and np.array_equal(back.dst, dst)
    if weighted:
        assert np.array_equal(back.weight, w)   # %g keeps 3 decimals of these values
    else:
        assert back.weight is None


def test_file_to_bfs(gb, tmp_path):
    """R-MAT s10 written as Matrix Market, read back, preprocessed: the same
    CSR and BFS levels as the generator's matrix."""
    A = gb.io.rmat_matrix(10)
    e = gb.generate_rmat(gb.RmatParams(scale=10))
    p = str(tmp_path / "r.mtx")
    gb.write_matrix_market(p, e)
    B = gb.edges_to_matrix(gb.preprocess(gb.read_matrix_market(p), make_undirected=True))
    assert np.array_equal(A.row_offsets, B.row_offsets)
    assert np.array_equal(A.col_indices, B.col_indices)
    assert np.array_equal(gb.bfs(A, 0).values, gb.bfs(B, 0).values)
