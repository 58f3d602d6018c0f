"""Single-GPU check at R-MAT s27 (4.2 G edges): generation, traversal layout,
BFS time and peak device memory.  python tools/s27_check.py"""
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1908_01407_b200 as gb
t = time.time()
A = gb.io.rmat_matrix(27)
torch.cuda.synchronize()
print("gen s", time.time() - t, "nnz", A.nnz, "peak GB", torch.cuda.max_memory_allocated() / 1e9, flush=True)
t = time.time()
A.traversal(); torch.cuda.synchronize()
print("trav s", time.time() - t, "peak GB", torch.cuda.max_memory_allocated() / 1e9, "now", torch.cuda.memory_allocated() / 1e9, flush=True)
d = gb.Descriptor()
lv = gb.bfs(A, 0, desc=d); v = lv.values
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): gb.bfs(A, 0)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print("bfs ms", ms, "GTEPS", A.nnz / ms / 1e6, "levels", len(d.direction_log), "reached", int((v > 0).sum()), "peak GB", torch.cuda.max_memory_allocated() / 1e9)
