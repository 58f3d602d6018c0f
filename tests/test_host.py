"""CPU-only checks: the C ABI loads and exports every declared symbol, and the
host-side logic (direction rule, algebra encoding, descriptor) matches the
reference."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "graphblast.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1908_01407_b200 import _lib
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and every symbol the binding declares is in the header
    assert set(_lib.SIGNATURES) <= set(syms)
    # and every header function has a typed binding (ctypes cannot pass a
    # double without one)
    unbound = [s for s in syms if s not in _lib.SIGNATURES]
    assert not unbound, unbound
    assert lib.gb_abi_version() == _lib.ABI_VERSION == 2


def test_native_direction_rule_matches_reference_cases():
    # kernels.py:108-126 with the reference test's numbers (test_kernels.py:308-341)
    from paper_1908_01407_b200 import _lib
    lib = _lib.load()
    est = ctypes.c_int64()
    assert lib.gb_decide_direction(1000, 100, 5, 0.1, 0, ctypes.byref(est)) == _lib.DIR_PUSH
    assert est.value == 50
    assert lib.gb_decide_direction(1000, 100, 11, 0.1, 0, ctypes.byref(est)) == _lib.DIR_PULL
    assert est.value == 110
    assert lib.gb_decide_direction(1000, 100, 10, 0.1, 0, ctypes.byref(est)) == _lib.DIR_PUSH  # tie
    assert lib.gb_decide_direction(0, 4, 4, 0.1, 0, ctypes.byref(est)) == _lib.DIR_PUSH
    assert lib.gb_decide_direction(1000, 100, 50, 0.1, 1, None) == _lib.DIR_PUSH
    assert lib.gb_decide_direction(1000, 100, 0, 0.1, 2, None) == _lib.DIR_PULL


def test_native_rule_rounds_half_even_like_python():
    from paper_1908_01407_b200 import _lib
    from paper_1908_01407_b200.kernels import direction_rule
    from paper_1908_01407_b200.containers import Direction
    lib = _lib.load()
    rng = np.random.default_rng(3)
    cases = [(5, 2, 1), (15, 2, 1), (25, 10, 1), (7, 2, 3), (520_756_042, 16_777_216, 405_970),
             (128_310_252, 4_194_304, 163_043)]
    cases += [(int(rng.integers(0, 10**9)), int(rng.integers(1, 10**7)), int(rng.integers(0, 10**7)))
              for _ in range(2000)]
    for nnz, nrows, k in cases:
        est = ctypes.c_int64()
        d = lib.gb_decide_direction(nnz, nrows, k, 0.1, 0, ctypes.byref(est))
        chosen, e, thr = direction_rule(nnz, nrows, k, 0.1, Direction.AUTO)
        assert est.value == e, (nnz, nrows, k)
        assert (d == _lib.DIR_PULL) == (chosen == "pull")


def test_s24_trace_from_survey_numbers():
    # SURVEY §8 level profile at s24: estimates and directions
    from paper_1908_01407_b200.kernels import direction_rule
    from paper_1908_01407_b200.containers import Direction
    nnz, n = 520_756_042, 16_777_216
    f = [1, 405_970, 7_612_546, 843_624, 3_034, 9]
    est = [31, 12_601_097, 236_289_461, 26_185_649, 94_174, 279]
    want = ["push", "push", "pull", "push", "push", "push"]
    for k, e, w in zip(f, est, want):
        chosen, got, thr = direction_rule(nnz, n, k, 0.1, Direction.AUTO)
        assert got == e and chosen == w


def test_algebra_encoding():
    from paper_1908_01407_b200 import _lib
    from paper_1908_01407_b200.algebra import (
        BinaryOp, Monoid, Semiring, builtin_semiring, fold_op_id, pair_op_id, PLUS, SECOND, LESS)
    assert pair_op_id(PLUS) == _lib.OP_PLUS          # saturating pairwise
    assert fold_op_id(PLUS) == _lib.OP_PLUS          # wrapping fold
    assert pair_op_id(SECOND) == _lib.OP_SECOND
    with pytest.raises(TypeError):
        fold_op_id(LESS)                             # numpy has no reduce loop for less
    user = BinaryOp("umax", max, np.maximum)
    assert pair_op_id(user) == _lib.OP_MAX
    assert pair_op_id(BinaryOp("addw", lambda a, b: a + b, np.add)) == _lib.OP_PLUS_WRAP
    with pytest.raises(NotImplementedError):
        pair_op_id(BinaryOp("gcdish", lambda a, b: a + b))
    sr = Semiring(Monoid(user, -np.inf), BinaryOp("utimes", lambda a, b: a * b, np.multiply))
    assert sr.add.identity_for(np.float64) == -np.inf
    assert builtin_semiring("MinPlus").add.identity_for(np.int64) == np.iinfo(np.int64).max


def test_host_algebra_utilities_match_reference_tests():
    # test_algebra.py:84-124 behaviours on host arrays
    from paper_1908_01407_b200.algebra import PLUS, BinaryOp, Monoid, builtin_monoid
    imax, imin = np.iinfo(np.int64).max, np.iinfo(np.int64).min
    out = PLUS.pairwise(np.array([imax, imax - 3, 10]), np.array([5, 10, 20]))
    assert out.tolist() == [imax, imax, 30]
    out = PLUS.pairwise(np.array([imin, imin + 2]), np.array([-7, -5]))
    assert out.tolist() == [imin, imin]
    assert builtin_monoid("Minimum").reduce(np.empty(0, np.int64)) == imax
    op = BinaryOp("gcdish", lambda a, b: a + b)
    assert list(Monoid(op, 0.0).segment_reduce(np.array([1, 2, 3, 4]), np.array([0, 2]))) == [3, 7]


def test_descriptor_surface():
    from paper_1908_01407_b200 import Descriptor, MaskMode
    d = Descriptor()
    assert d.switch_ratio == 0.1 and d.max_niter == 10_000
    d.toggle("mask")
    assert d.mask_mode is MaskMode.COMPLEMENT
    d.toggle("inp1")
    assert d.transpose_inp1
    with pytest.raises(KeyError):
        d.toggle("outp")


def test_public_api_matches_reference_all():
    import paper_1908_01407_b200 as gb
    ref_all = ["BinaryOp", "Monoid", "Semiring", "builtin_monoid", "builtin_semiring",
               "SparseMatrix", "Vector", "Descriptor", "Counters", "Direction",
               "MaskMode", "Partition", "matrix_build", "vector_build", "vector_fill",
               "vector_convert", "DirectionDecision", "mxv", "vxm", "spmv_pull", "spmspv_push",
               "decide_direction", "mxm_masked", "ewise_add", "ewise_mult", "assign",
               "assign_scatter", "extract_gather", "apply", "reduce", "reduce_rows",
               "reduce_scalar_matrix", "transpose", "bfs", "sssp", "pagerank",
               "connected_components", "triangle_count", "EdgeList", "RmatParams", "SplitMix64",
               "read_matrix_market", "write_matrix_market", "preprocess", "assign_weights",
               "generate_rmat", "edges_to_matrix", "GraphAlgError", "ShapeError", "FormatError",
               "ParseError", "__version__"]
    assert gb.__all__ == ref_all
    for name in ref_all:
        assert hasattr(gb, name)


def test_product_refuses_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1908_01407_b200 as gb
    with pytest.raises(RuntimeError):
        gb.vector_fill(4, 0)


def test_splitmix_scalar_matches_stream():
    from paper_1908_01407_b200.io import SplitMix64
    from oracle import port
    g = SplitMix64(1)
    want = port.splitmix_stream(1, 0, 5)
    assert [g.next_u64() for _ in range(5)] == [int(x) for x in want]


def test_cli_parser_matches_reference_surface():
    """cli.py:72-100: same positional algorithm and options."""
    from paper_1908_01407_b200 import cli
    p = cli.build_parser()
    a = p.parse_args(["bfs", "--rmat-scale", "16", "--source", "3", "--runs", "4", "--json",
                      "--trace", "--verify", "--direction", "force-pull", "--switch-ratio", "0.2",
                      "--threads", "8", "--max-iters", "7", "--alpha", "0.9", "--eps", "1e-6"])
    assert (a.algorithm, a.rmat_scale, a.source, a.runs, a.as_json, a.trace, a.verify) == \
        ("bfs", 16, 3, 4, True, True, True)
    assert (a.direction, a.switch_ratio, a.threads, a.max_iters, a.alpha, a.eps) == \
        ("force-pull", 0.2, 8, 7, 0.9, 1e-6)
    with pytest.raises(SystemExit):
        p.parse_args(["dfs"])
    d = cli.Harness(a).descriptor(fused=False)
    assert d.direction.value == "force-pull" and d.max_niter == 7 and d.fused is False
    assert d.switch_ratio == 0.2
