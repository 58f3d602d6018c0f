"""Unmasked pull SpMV (PageRank's multiply) through mxv: row tiles vs row
bins, original vs degree-ordered matrix, with the gather-replay ceiling.

    python tools/time_pull_unmasked.py --scale 22
"""
import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200 import _lib, kernels  # noqa: E402
from paper_1908_01407_b200.containers import SparseMatrix, Vector  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
A0 = gb.io.rmat_matrix(args.scale)
push_o, pull_o, _rank = A0.traversal()
Ao = SparseMatrix._wrap(A0.nrows, A0.ncols, push_o, pull_o, A0.dtype, A0._sym)
ctx = _lib.context()
n = A0.nrows
x = torch.rand(n, dtype=torch.float64, device="cuda") + 0.5
u = Vector._wrap(n, None, x, 0.0, np.float64)
sr = gb.builtin_semiring("PlusMultiplies")
for name, A in (("original", A0), ("ordered", Ao)):
    rate = ctypes.c_double(0)
    st, _k = A._csr.csr_struct(np.float64)
    ctx.call("gb_gather_replay_rate", ctypes.byref(st), _lib.ptr(x), ctypes.byref(rate))
    for impl in ("0", "1"):
        kernels._MV_BINS = impl
        d = gb.Descriptor(direction=gb.Direction.FORCE_PULL)
        gb.mxv(sr, A, u, desc=d)
        torch.cuda.synchronize()
        ctx.profiling(True)
        for _ in range(args.reps):
            gb.mxv(sr, A, u, desc=gb.Descriptor(direction=gb.Direction.FORCE_PULL))
        torch.cuda.synchronize()
        ms = float(np.median([t for (k, _a, t) in ctx.prof_read() if k == 8]))
        ctx.profiling(False)
        print(json.dumps({"matrix": name, "kernel": "bins" if impl == "1" else "tiles",
                          "ms": round(ms, 4), "Ggather_s": round(A.nnz / ms / 1e6, 1),
                          "replay_ceiling_Ggather_s": round(rate.value / 1e9, 1)}))
