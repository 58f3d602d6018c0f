"""The compile-time / environment-selected kernel variants that are not on the
default path still have to be exact: rerun the parity suites in a child
process with each knob set (the knobs are read once per process)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _pytest(env_extra, *args):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *args],
                       cwd=os.path.dirname(HERE), env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_masked_mv_compact_plan():
    # GB_MV_COMPACT=1: reduce only the allowed rows (mv_mask_plan)
    _pytest({"GB_MV_COMPACT": "1"}, os.path.join(HERE, "test_gpu_kernels.py"), "-k", "mv_cases")


@pytest.mark.parametrize("mode", ["0", "2"])
def test_bfs_prefix_modes(mode):
    # the dense-visited-prefix skip: 0 off, 2 probe skip (1, list cut, is the default)
    _pytest({"GB_PREFIX_MODE": mode}, os.path.join(HERE, "test_gpu_bfs.py"), "-k",
            "golden or oracle or ordered or engines or s24")


def test_bfs_shared_memory_push():
    _pytest({"GB_PUSH_SMEM": "1"}, os.path.join(HERE, "test_gpu_bfs.py"), "-k",
            "golden or oracle or ordered or s24")


def test_pagerank_stored_labels():
    _pytest({"GB_PR_ORDER": "0"}, os.path.join(HERE, "test_gpu_algorithms.py"), "-k", "pr or pagerank")


def test_sssp_stored_labels():
    _pytest({"GB_SSSP_ORDER": "0"}, os.path.join(HERE, "test_gpu_algorithms.py"), "-k", "sssp")


@pytest.mark.parametrize("mode", ["0", "2"])
def test_bounded_pull_variants(mode):
    # CC / SSSP pulls: 0 = edge-balanced tiles everywhere, 2 = the bounded
    # row-bin pulls (cc_pull_exit, sssp_pull_exit) on every graph, skewed or
    # not (1, the default, takes them on skewed graphs only)
    _pytest({"GB_PULL_EXIT": mode}, os.path.join(HERE, "test_gpu_algorithms.py"),
            os.path.join(HERE, "test_gpu_loops.py"), os.path.join(HERE, "test_gpu_pins.py"),
            "-k", "cc or sssp")
