"""Unmasked pull on a large uniform graph: the bins + column-stripes route
(now the default there) against the edge-balanced tiles (GB_MV_BINS=0 in a
second process) -- identical results for exact folds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200.containers import Vector  # noqa: E402

A = gb.io.rmat_matrix(int(sys.argv[1]) if len(sys.argv) > 1 else 23, a=.25, b=.25, c=.25, d=.25)
n = A.nrows
rng = np.random.default_rng(3)
x = Vector._wrap(n, None, torch.tensor(rng.integers(-50, 50, n), device="cuda"), 0, np.int64)
out = {}
for sr in ("MinimumSelectSecond", "PlusMultiplies", "MaxPlus", "LogicalOrAnd"):
    d = gb.Descriptor(direction=gb.Direction.FORCE_PULL)
    w = gb.mxv(gb.builtin_semiring(sr), A, x, desc=d)
    out[sr] = (w.values, d.counters.matrix_entries_read, d.counters.semiring_multiplies,
               d.counters.semiring_adds)
np.save(sys.argv[2] if len(sys.argv) > 2 else "/tmp/pull.npy",
        np.array([out[k][0] for k in sorted(out)]))
print({k: v[1:] for k, v in out.items()})
