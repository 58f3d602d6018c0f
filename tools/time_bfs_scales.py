"""bfs(A, 0) device time per call at several R-MAT scales (CUDA events,
asynchronous calls back to back), e.g. to place the cooperative small-graph
kernel's threshold (GB_BFS_COOP_N)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402

lib = gb._lib.load()
modes = {"graph": 0, "coop": 1 << 30}


def timed(A):
    for _ in range(3):
        gb.bfs(A, 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    descs = []
    e0.record()
    for _ in range(100):
        d = gb.Descriptor()
        descs.append(d)
        gb.bfs(A, 0, desc=d)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 100, [(x.chosen, x.frontier_nvals) for x in descs[-1].direction_log]


for scale in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "12,14,16,18,20").split(",")]:
    A = gb.io.rmat_matrix(scale)
    res = {}
    for rep in range(3):   # alternate the two engines in one process
        for name, lim in modes.items():
            lib.gb_bfs_coop_max_n(lim)
            ms, trace = timed(A)
            res.setdefault(name, []).append(round(ms, 4))
    lib.gb_bfs_coop_max_n(-1)
    print(json.dumps({"scale": scale, "ms": res, "trace": trace}))
