"""Quick device timing of each fused algorithm at the BASELINE config scales.

    python tools/time_algos.py [--reps 5]
Prints one JSON line per algorithm: ms per call (CUDA events), MTEPS.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200.io import rmat_matrix  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--only", default="")
args = ap.parse_args()

CASES = [
    ("bfs", 24, lambda A: gb.bfs(A, 0)),
    ("cc", 24, lambda A: gb.connected_components(A)),
    ("pr20", 22, lambda A: gb.pagerank(A, eps=1e-300, max_iters=20)),
    ("sssp", 20, lambda A: gb.sssp(A, 0)),
    ("tc", 20, lambda A: gb.triangle_count(A)),
    ("bfs", 20, lambda A: gb.bfs(A, 0)),
    ("cc", 20, lambda A: gb.connected_components(A)),
    ("ccu", 24, lambda A: gb.connected_components(A)),   # uniform a=b=c=d=.25
]
for name, scale, fn in CASES:
    if args.only and name not in args.only.split(","):
        continue
    t0 = time.perf_counter()
    A = (rmat_matrix(scale, a=.25, b=.25, c=.25, d=.25) if name == "ccu"
         else rmat_matrix(scale, weighted=name == "sssp"))
    torch.cuda.synchronize()
    build = time.perf_counter() - t0
    gb._lib.context().trim()
    for _ in range(2):
        fn(A)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        fn(A)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.reps
    print(json.dumps({"algo": name, "scale": scale, "nnz": A.nnz, "ms": round(ms, 3),
                      "mteps": round(A.nnz / ms / 1e3, 1), "build_s": round(build, 2)}), flush=True)
    del A
    torch.cuda.empty_cache()
