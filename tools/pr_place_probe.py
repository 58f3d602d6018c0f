"""Why PageRank s22 x20 reads 9.6 ms in a fresh process and ~11 ms later:
time it fresh, after the context's caches are trimmed (the PR loop graph
rebuilt on the same arrays), after the degree-ordered layout is rebuilt
with the old one still alive, and after it is rebuilt into freed memory."""
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
print("fresh", t(A), t(A), flush=True)
gb._lib.context().trim()
print("trimmed (loop graph rebuilt)", t(A), t(A), flush=True)
keep = A._csr._ordered
A._csr._ordered = None
A.traversal()
print("layout rebuilt, old alive", t(A), t(A), flush=True)
keep = None
A._csr._ordered = None
gb._lib.context().trim()
torch.cuda.empty_cache()
A.traversal()
print("layout rebuilt into freed memory", t(A), t(A), flush=True)
big = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
A._csr._ordered = None
gb._lib.context().trim()
A.traversal()
print("layout rebuilt above an 8 GB block", t(A), t(A), flush=True)
