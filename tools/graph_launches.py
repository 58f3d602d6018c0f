"""Run the fused BFS (graph path) a few times at one scale; used under
`ncu --metrics gpu__time_duration.sum` to list the kernels one BFS launches."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
A = gb.io.rmat_matrix(args.scale)
for _ in range(args.reps):
    gb.bfs(A, 0)
torch.cuda.synchronize()
print("done")
