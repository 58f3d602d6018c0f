"""Per-iteration device cost of the fused SSSP loop (graph engine): time
sssp(W, 0) capped at k iterations for k = 1..K and difference consecutive
caps.  python tools/sssp_iter_cost.py [scale]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
W = gb.io.rmat_matrix(scale, weighted=True)


def t(cap, reps=20):
    d = gb.Descriptor(max_niter=cap)
    for _ in range(3):
        gb.sssp(W, 0, desc=gb.Descriptor(max_niter=cap))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gb.sssp(W, 0, desc=d if _ == 0 else gb.Descriptor(max_niter=cap))
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, [(x.chosen, x.frontier_nvals) for x in d.direction_log]


prev = 0.0
for cap in range(1, 11):
    ms, tr = t(cap)
    last = tr[-1] if tr else None
    print(f"cap {cap:2d}: {ms:.3f} ms  (+{ms - prev:.3f})  last {last}")
    prev = ms
