"""Break the bench's end-to-end BFS step into its parts (device BFS, D2H of
the levels, host overheads) to see where the e2e time goes."""
import time

import numpy as np
import torch

import paper_1908_01407_b200 as gb

A = gb.io.rmat_matrix(24)
torch.cuda.synchronize()
n = A.nrows
for i in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v = gb.bfs(A, 0)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    h = v.values
    t2 = time.perf_counter()
    print("iter %d: bfs %.3f ms  values %.3f ms  (%.1f GB/s)" %
          (i, (t1 - t0) * 1e3, (t2 - t1) * 1e3, n * 8 / (t2 - t1) / 1e9))
d = torch.empty(n, dtype=torch.int64, device="cuda")
p = torch.empty(n, dtype=torch.int64, pin_memory=True)
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print("raw pinned D2H %.3f ms (%.1f GB/s)" % ((t1 - t0) * 1e3, n * 8 / (t1 - t0) / 1e9))
t0 = time.perf_counter()
q = torch.empty(n, dtype=torch.int64, pin_memory=True)
print("pinned alloc %.3f ms" % ((time.perf_counter() - t0) * 1e3))
