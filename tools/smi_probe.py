"""Does a concurrent `nvidia-smi -lms 50` (bench.py's clock sampler) slow the
timed BFS loop?  Alternates the loop with and without the sampler."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402

A = gb.io.rmat_matrix(int(sys.argv[1]) if len(sys.argv) > 1 else 24)


def loop(steps=200):
    for _ in range(5):
        gb.bfs(A, 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(steps):
        gb.bfs(A, 0, desc=gb.Descriptor())
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / steps, 4), round((t1 - t0) / steps * 1e3, 4)


for rep in range(4):
    print("plain  ", loop(), flush=True)
    p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm", "--format=csv,noheader",
                          "-lms", "50"], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    time.sleep(0.15)
    print("sampler", loop(), flush=True)
    p.terminate()
    p.wait()
