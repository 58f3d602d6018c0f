"""Host cost of the first bfs() calls in a fresh process (why do the first
few hundred asynchronous calls cost more host time than the steady state?)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402

A = gb.io.rmat_matrix(int(sys.argv[1]) if len(sys.argv) > 1 else 24)
for _ in range(5):
    gb.bfs(A, 0)
torch.cuda.synchronize()
ts = []
pr = cProfile.Profile()
pr.enable()
for i in range(200):
    t0 = time.perf_counter()
    gb.bfs(A, 0, desc=gb.Descriptor())
    ts.append((time.perf_counter() - t0) * 1e3)
pr.disable()
torch.cuda.synchronize()
print("first 200 host ms:", [round(x, 3) for x in ts[:20]], "... median", sorted(ts)[100])
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
ts = []
for i in range(400):
    t0 = time.perf_counter()
    gb.bfs(A, 0, desc=gb.Descriptor())
    ts.append((time.perf_counter() - t0) * 1e3)
torch.cuda.synchronize()
print("next 400 host ms: median", sorted(ts)[200], "max", max(ts), "mean", sum(ts) / len(ts))
print("alloc stats:", torch.cuda.memory_stats().get("num_alloc_retries"),
      torch.cuda.memory_stats().get("segment.all.allocated"))
