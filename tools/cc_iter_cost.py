"""Per-iteration device cost of the fused CC loop (graph engine): time
connected_components capped at k iterations for k = 1..K and difference
consecutive caps.  python tools/cc_iter_cost.py [scale] [--uniform]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
kw = dict(a=.25, b=.25, c=.25, d=.25) if "--uniform" in sys.argv else {}
A = gb.io.rmat_matrix(scale, **kw)


def t(cap, reps=10):
    d = gb.Descriptor(max_niter=cap)
    for _ in range(2):
        gb.connected_components(A, desc=gb.Descriptor(max_niter=cap))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        gb.connected_components(A, desc=d if i == 0 else gb.Descriptor(max_niter=cap))
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, [(x.chosen, x.frontier_nvals) for x in d.direction_log]


prev = 0.0
for cap in range(1, 9):
    ms, tr = t(cap)
    print(f"cap {cap:2d}: {ms:.3f} ms  (+{ms - prev:.3f})  last {tr[-1] if tr else None}")
    prev = ms
