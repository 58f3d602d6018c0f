"""The command-line harness (cli.py:40-277 restated on the GPU): reports carry
the reference's result digest and direction trace for the same inputs."""

import contextlib
import hashlib
import io
import json

import pytest

from golden_io import load_json

pytestmark = pytest.mark.gpu


def run_cli(*argv):
    from paper_1908_01407_b200 import cli
    out = io.StringIO()
    with contextlib.redirect_stdout(out):
        rc = cli.main(list(argv))
    return rc, out.getvalue()


@pytest.mark.parametrize("algo,scale", [("bfs", 16), ("bfs", 12), ("sssp", 12), ("cc", 12)])
def test_cli_digest_and_trace_match_reference(algo, scale):
    gold = load_json("algorithms.json")[f"{algo}_s{scale}"]
    rc, out = run_cli(algo, "--rmat-scale", str(scale), "--runs", "2", "--json", "--verify")
    assert rc == 0
    rep = json.loads(out)
    assert rep["result_digest"] == gold["digest"]
    assert rep["verified"] is True
    trace = [[r["direction"], r["frontier_nvals"], r["estimated_frontier_edges"], r["threshold_edges"]]
             for r in rep["trace"]]
    assert trace == gold["trace"]
    assert rep["runs"] == 2 and rep["mteps"] > 0 and rep["nnz"] > 0


def test_cli_triangle_count_and_pagerank():
    gold = load_json("algorithms.json")["tc_s12"]["count"]
    rc, out = run_cli("tc", "--rmat-scale", "12", "--runs", "1", "--json", "--verify")
    rep = json.loads(out)
    assert rc == 0 and rep["verified"] is True
    assert rep["result_digest"] == hashlib.sha256(str(int(gold)).encode()).hexdigest()
    rc, out = run_cli("pr", "--rmat-scale", "10", "--runs", "1", "--verify")
    assert rc == 0 and "verification: ok" in out


def test_cli_text_report_and_trace_table():
    rc, out = run_cli("bfs", "--rmat-scale", "10", "--runs", "1", "--trace")
    assert rc == 0
    assert out.startswith("bfs on rmat-s10-e16: 1 runs")
    assert "iter  frontier  est_edges  threshold  direction" in out


def test_cli_bad_source():
    from paper_1908_01407_b200 import cli
    with pytest.raises(SystemExit):
        cli.main(["bfs", "--rmat-scale", "6", "--source", "64"])


def test_binary_csr_cache_round_trip(tmp_path):
    import numpy as np
    import paper_1908_01407_b200 as gb
    from paper_1908_01407_b200.io import load_matrix, save_matrix
    for weighted in (False, True):
        A = gb.io.rmat_matrix(12, weighted=weighted)
        p = str(tmp_path / f"g{int(weighted)}.npz")
        save_matrix(p, A)
        B = load_matrix(p)
        assert B.nnz == A.nnz and B.is_symmetric()
        assert np.array_equal(B.row_offsets, A.row_offsets)
        assert np.array_equal(B.col_indices, A.col_indices)
        assert np.array_equal(B.csr_values, A.csr_values)
    gold = load_json("algorithms.json")["bfs_s12"]
    save_matrix(str(tmp_path / "s12.npz"), gb.io.rmat_matrix(12))
    rc, out = run_cli("bfs", "--graph", str(tmp_path / "s12.npz"), "--runs", "1", "--json")
    assert rc == 0 and json.loads(out)["result_digest"] == gold["digest"]


def test_cli_certificates_reject_corrupted_results():
    """--verify's SSSP / CC certificates (gb_sssp_certify, gb_cc_certify) fail
    on a perturbed result and pass on the computed one."""
    import numpy as np
    import paper_1908_01407_b200 as gb
    from paper_1908_01407_b200 import cli
    from paper_1908_01407_b200.containers import Vector
    args = cli.build_parser().parse_args(["sssp", "--rmat-scale", "10"])
    h = cli.Harness(args)
    W = gb.io.rmat_matrix(10, weighted=True)
    d = gb.sssp(W, 0)
    assert h._certify_sssp(W, d)
    bad = d.to_dense(np.inf)._vals.clone()
    v = int(np.flatnonzero(np.isfinite(d.values) & (d.values > 0))[3])
    bad[v] += 1.0
    assert not h._certify_sssp(W, Vector._wrap(W.nrows, None, bad, np.inf, np.float64))
    bad = d.to_dense(np.inf)._vals.clone()
    bad[v] -= 0.5
    assert not h._certify_sssp(W, Vector._wrap(W.nrows, None, bad, np.inf, np.float64))
    A = gb.io.rmat_matrix(10)
    lab = gb.connected_components(A)
    args = cli.build_parser().parse_args(["cc", "--rmat-scale", "10"])
    h = cli.Harness(args)
    assert h._certify_cc(A, lab)
    t = lab.to_dense(0)._vals.clone()
    t[5] = 5 if int(t[5]) != 5 else 4     # a label that is not the class minimum
    assert not h._certify_cc(A, Vector._wrap(A.nrows, None, t, 0, np.int64))
