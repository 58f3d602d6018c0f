"""The C ABI from a plain C program (tests/abi/abi_bfs.c: no Python, no
PyTorch): R-MAT generation, CSR build and the fused BFS through
include/graphblast.h, checked against the C oracle."""

import json
import os
import subprocess

import numpy as np
import pytest

from oracle import cgraph

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "abi", "abi_bfs")


def test_c_consumer_builds():
    """build() compiles it next to the library (here: CPU only, no run)."""
    if not os.path.exists(BIN):
        subprocess.check_call(["make", "-s", "-C", os.path.join(HERE, "abi")])
    assert os.access(BIN, os.X_OK)


@pytest.mark.gpu
@pytest.mark.parametrize("scale,source", [(12, 0), (14, 0), (14, 5)])
def test_c_consumer_bfs_matches_oracle(scale, source):
    out = subprocess.run([BIN, str(scale), str(source)], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr
    got = json.loads(out.stdout.strip().splitlines()[-1])
    rp, ci = cgraph.rmat_csr(scale)
    lv, trace = cgraph.bfs(rp, ci, source)
    assert got["nnz"] == ci.size
    assert got["reached"] == int((lv > 0).sum()) and got["level_sum"] == int(lv.sum())
    assert [tuple(t) for t in got["trace"]] == [tuple(t) for t in trace]
