"""Where a bfs() call's time goes at the bench scale: wall time per public
call, CUDA-event time of the same calls, and the native call alone (prebuilt
ctypes arguments), so host overhead between graph launches is visible.

    python tools/bfs_overhead.py [--scale 24] [--reps 50]
"""
import argparse
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200 import _lib  # noqa: E402
from paper_1908_01407_b200.containers import empty  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--reps", type=int, default=50)
args = ap.parse_args()

A = gb.io.rmat_matrix(args.scale)
for _ in range(3):
    gb.bfs(A, 0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

t = time.perf_counter()
e0.record()
for _ in range(args.reps):
    gb.bfs(A, 0)
e1.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t) / args.reps * 1e3
print(f"public bfs(): wall {wall:.4f} ms/call, events {e0.elapsed_time(e1) / args.reps:.4f} ms/call")

push_o, pull_o, rank = A.traversal()
(push, _k1), (pull, _k2) = push_o.csr_struct(), pull_o.csr_struct()
n = A.nrows
levels = empty(n, np.int64)
cap = n + 1
dirs = np.zeros(cap, np.int32)
nv = np.zeros(cap, np.int64)
est = np.zeros(cap, np.int64)
done = C.c_int64(0)
ctx = _lib.context()
fn = ctx.lib.gb_bfs_ordered
argv = (ctx.ptr, C.byref(push), C.byref(pull), _lib.ptr(pull_o.nonempty()), _lib.ptr(rank), 0, cap,
        0.1, _lib.DIR_AUTO, _lib.ptr(levels), dirs.ctypes.data_as(C.c_void_p),
        nv.ctypes.data_as(C.c_void_p), est.ctypes.data_as(C.c_void_p), C.byref(done))
fn(*argv)
torch.cuda.synchronize()
t = time.perf_counter()
e0.record()
for _ in range(args.reps):
    fn(*argv)
e1.record()
torch.cuda.synchronize()
wall = (time.perf_counter() - t) / args.reps * 1e3
print(f"native gb_bfs_ordered: wall {wall:.4f} ms/call, events {e0.elapsed_time(e1) / args.reps:.4f} ms/call")
