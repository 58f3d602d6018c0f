"""Fixed per-level cost of the BFS device loop: a path graph (one tiny push
level per vertex), device time per level.  python tools/level_overhead.py"""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1908_01407_b200 as gb
n = 2000
r = np.r_[np.arange(n - 1), np.arange(1, n)]
c = np.r_[np.arange(1, n), np.arange(n - 1)]
A = gb.SparseMatrix.from_tuples(r, c, np.ones(r.size, np.int64), n, n)
for _ in range(3): gb.bfs(A, 0).values
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): lv = gb.bfs(A, 0)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 5
print(f"path n={n}: {t:.3f} ms per bfs, {t / n * 1000:.2f} us per level")
