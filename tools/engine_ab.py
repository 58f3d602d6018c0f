"""BFS wall/device time per call for both engines (graph, host loop) at a few scales.

    python tools/engine_ab.py [--scales 12,16,20,24]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scales", default="12,16,20,24")
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
lib = _lib.load()
for s in [int(x) for x in args.scales.split(",")]:
    A = gb.io.rmat_matrix(s)
    row = [f"s{s}"]
    for eng in (0, 1):
        lib.gb_bfs_engine(eng)
        for _ in range(3):
            gb.bfs(A, 0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            d = gb.Descriptor()
            gb.bfs(A, 0, desc=d)
        e1.record()
        torch.cuda.synchronize()
        row.append(f"{['graph', 'host'][eng]} {e0.elapsed_time(e1) / args.reps:.4f} ms")
    row.append(f"levels {len(d.direction_log)}")
    print("  ".join(row), flush=True)
    lib.gb_bfs_engine(0)
    del A
