"""PageRank s22 x20 device time in different process states (bench.py's C3
reads slower than tools/time_algos.py): untrimmed vs trimmed context, after
other workloads."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200.io import rmat_matrix  # noqa: E402


def t(A, reps=5):
    for _ in range(2):
        gb.pagerank(A, eps=1e-300, max_iters=20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gb.pagerank(A, eps=1e-300, max_iters=20)
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 3)


A = rmat_matrix(22)
print("fresh, untrimmed", t(A), t(A))
gb._lib.context().trim()
print("trimmed", t(A), t(A))
B = rmat_matrix(20)
gb.triangle_count(B)
del B
print("after tc", t(A))
A = None
gb._lib.context().trim()
torch.cuda.empty_cache()
A = rmat_matrix(22)
print("rebuilt, untrimmed", t(A), t(A))
gb._lib.context().trim()
print("rebuilt, trimmed", t(A), t(A))
