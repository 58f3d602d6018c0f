"""The reference's own test suite (pkg/tests: test_algebra.py,
test_containers.py, test_kernels.py, helpers.py -- 136 tests), run UNCHANGED
against this package: `graphalg` and its submodules are aliased to
paper_1908_01407_b200, so every `from graphalg import ...` in those files
binds the B200 implementation ("the reference tests run
unchanged").

The files are test infrastructure copied verbatim from
/root/reference/pkg/tests by vendor.py (run by __graft_entry__.build() where
/root/reference exists) into _vendored/, which is git-ignored -- they are the
reference's code, not this repository's -- and travels to the GPU box with the
working tree like the built libraries.  Every test in it needs the device
(there is no CPU fallback), so all are marked `gpu`.
"""

import importlib
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
VENDORED = os.path.join(HERE, "_vendored")


def _alias_graphalg():
    import paper_1908_01407_b200 as pkg
    sys.modules.setdefault("graphalg", pkg)
    for name in ("algebra", "containers", "kernels", "algorithms", "errors", "io"):
        sys.modules.setdefault(f"graphalg.{name}", importlib.import_module(f"{pkg.__name__}.{name}"))


_alias_graphalg()
if VENDORED not in sys.path:
    sys.path.insert(0, VENDORED)  # `from helpers import ...`

collect_ignore = [] if os.path.isdir(VENDORED) else ["_vendored"]


def pytest_collection_modifyitems(config, items):
    for item in items:
        if str(item.fspath).startswith(VENDORED):
            item.add_marker(pytest.mark.gpu)
            item.add_marker(pytest.mark.reference_suite)
