"""Profiling driver: build an R-MAT graph on the GPU, warm up, then run `reps`
calls of one algorithm inside a cudaProfilerStart/Stop window (use with
`ncu --profile-from-start off`).

    python tools/prof_bfs.py --algo bfs|sssp|pr|cc|tc|mxv --scale 24 --reps 1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200.io import rmat_matrix  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--algo", default="bfs")
args = ap.parse_args()

A = rmat_matrix(args.scale, weighted=args.algo == "sssp")
gb._lib.context().trim()


def run():
    if args.algo == "bfs":
        gb.bfs(A, 0)
    elif args.algo == "sssp":
        gb.sssp(A, 0)
    elif args.algo == "pr":
        gb.pagerank(A, eps=1e-300, max_iters=3)
    elif args.algo == "cc":
        gb.connected_components(A)
    elif args.algo == "tc":
        gb.triangle_count(A)
    elif args.algo == "mxv":
        u = gb.vector_fill(A.nrows, 1.0)
        gb.mxv(gb.builtin_semiring("PlusMultiplies"), A, u)


for _ in range(2):
    run()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(args.reps):
    run()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
