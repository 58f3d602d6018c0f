"""The operator-level compositions (Descriptor(fused=False): the reference's
algorithms.py loops over mxv / vxm / ewise / assign / reduce) beside the fused
drivers, device time per call.  python tools/time_composed.py [scale]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
A = gb.io.rmat_matrix(scale)
W = gb.io.rmat_matrix(scale, weighted=True)


def dev_ms(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 3)


for name, f in (("bfs", lambda d: gb.bfs(A, 0, desc=d)),
                ("sssp", lambda d: gb.sssp(W, 0, desc=d)),
                ("cc", lambda d: gb.connected_components(A, desc=d)),
                ("pagerank x20", lambda d: gb.pagerank(A, eps=1e-300, max_iters=20, desc=d))):
    fused = dev_ms(lambda: f(gb.Descriptor()))
    comp = dev_ms(lambda: f(gb.Descriptor(fused=False)))
    print(f"s{scale} {name:13s} fused {fused:9.3f} ms   composed {comp:9.3f} ms", flush=True)
