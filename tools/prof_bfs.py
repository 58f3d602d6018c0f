"""Profiling driver: build the R-MAT graph, then run `reps` BFS inside a
cudaProfilerStart/Stop window (use with ncu --profile-from-start off)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200.io import rmat_matrix  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--algo", default="bfs")
args = ap.parse_args()
A = rmat_matrix(args.scale)
gb._lib.context().trim()
for _ in range(2):
    gb.bfs(A, 0)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(args.reps):
    gb.bfs(A, 0)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
