"""Gather-replay rate (gb_gather_replay_rate) of R-MAT / uniform s24 in the
caller's labels and in the degree-ordered labels (SparseMatrix.traversal()),
lane-strided vs lane-consecutive (GB_REPLAY_CONSEC): how much the column
order and the lane mapping let a warp's gathers share lines of x."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200 import _lib  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
ctx = _lib.context()
for fam, kw in (("rmat", {}), ("uniform", dict(a=.25, b=.25, c=.25, d=.25))):
    A = gb.io.rmat_matrix(scale, **kw)
    x = torch.rand(A.nrows, dtype=torch.float64, device="cuda") + 0.5
    push_o, pull_o, _rank = A.traversal()
    out = {}
    for lab, o in (("orig", A._csr), ("ordered", pull_o)):
        st, _k = o.csr_struct(np.float64)
        for mode in ("0", "1"):
            os.environ["GB_REPLAY_CONSEC"] = mode
            r = ctypes.c_double(0)
            ctx.call("gb_gather_replay_rate", ctypes.byref(st), _lib.ptr(x), ctypes.byref(r))
            ctx.call("gb_gather_replay_rate", ctypes.byref(st), _lib.ptr(x), ctypes.byref(r))
            out[f"{lab}_{'consec' if mode == '1' else 'strided'}_G_s"] = round(r.value / 1e9, 1)
    print(json.dumps({"graph": f"{fam}-s{scale}", **out}))
    del A, push_o, pull_o, x
    torch.cuda.empty_cache()
