"""One-rank timing of the partitioned BFS loops on the degree-ordered layout
(world size 1: the exchange is local) -- the device-resident loop with and
without the push's prefix cut against the count-driven host loop, beside the
fused single-GPU bfs.  python tools/dist_loop_probe.py [scale]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200 import distributed as gbd  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
A = gb.io.rmat_matrix(scale)
A.traversal()


def dev_ms(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 3), round((time.perf_counter() - t0) / reps * 1e3, 3)


host = gbd.OrderedPartitionedBfs(A, 0, 1, loop="host")
dev = gbd.OrderedPartitionedBfs(A, 0, 1, loop="device")
nocut = gbd.OrderedPartitionedBfs(A, 0, 1, loop="device")
nocut.steps.prefix_cut = False
print("fused bfs        ", dev_ms(lambda: gb.bfs(A, 0)))
for name, run in (("host loop", host), ("device loop", dev), ("device, no cut", nocut)):
    print(f"{name:17s}", dev_ms(lambda: run(0)))
# the dense visited prefix the device loop ended with (DistBfsState.xcur)
print("final xcur", int(dev.steps.state[16]), "of n", A.nrows)
