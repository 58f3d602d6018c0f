"""BFS at R-MAT s24 under the reference rule with different switch ratios
(Descriptor.switch_ratio, containers.py:74-113): device time per call and
the direction trace.  The default 0.1 is the reference's; smaller ratios pull
earlier (direction-optimising BFS with the reference's own knob)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
A = gb.io.rmat_matrix(scale)
want = gb.bfs(A, 0).values
for ratio in (0.1, 0.05, 0.02, 0.01, 0.005):
    def run():
        return gb.bfs(A, 0, desc=gb.Descriptor(switch_ratio=ratio))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    d = gb.Descriptor(switch_ratio=ratio)
    lv = gb.bfs(A, 0, desc=d).values
    print(json.dumps({"switch_ratio": ratio, "ms": round(ms, 4), "gteps": round(A.nnz / ms / 1e6, 1),
                      "same_levels": bool(np.array_equal(lv, want)),
                      "trace": [(x.chosen, x.frontier_nvals) for x in d.direction_log]}))
