"""Timing stability of bfs(A, 0) at s24 inside one process: N batches of
50 calls each, device time per call per batch (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402

A = gb.io.rmat_matrix(int(sys.argv[1]) if len(sys.argv) > 1 else 24)
for _ in range(5):
    gb.bfs(A, 0)
torch.cuda.synchronize()
out = []
for b in range(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    descs = []
    e0.record()
    for _ in range(50):
        d = gb.Descriptor()
        descs.append(d)
        gb.bfs(A, 0, desc=d)
    e1.record()
    torch.cuda.synchronize()
    for d in descs:
        assert len(d.direction_log) == 6
    out.append(round(e0.elapsed_time(e1) / 50, 4))
print(out)
