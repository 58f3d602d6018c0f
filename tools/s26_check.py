"""BASELINE config C5 at scale 26 on one B200: build the reference R-MAT graph
on the GPU (n = 67 M, nnz ~ 2.1e9), time bfs(A, 0) and connected_components(A)
(CUDA events), and check both against the C oracle on the same CSR copied to
the host.  Prints one JSON line.

    python tools/s26_check.py [--scale 26] [--reps 5] [--no-oracle]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=26)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--no-oracle", action="store_true")
args = ap.parse_args()

out = {"scale": args.scale}
t0 = time.perf_counter()
A = gb.io.rmat_matrix(args.scale)
torch.cuda.synchronize()
out["build_s"] = round(time.perf_counter() - t0, 2)
out["n"], out["nnz"] = A.nrows, A.nnz
gb._lib.context().trim()


def timed(fn, reps):
    r = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, r


t1 = time.perf_counter()
A.traversal()
torch.cuda.synchronize()
out["relabel_s"] = round(time.perf_counter() - t1, 2)
desc = gb.Descriptor()
ms, lv = timed(lambda: gb.bfs(A, 0, desc=desc), args.reps)
out["bfs_ms"] = round(ms, 3)
out["bfs_gteps"] = round(A.nnz / ms / 1e6, 1)
dl = desc.direction_log[-len(desc.direction_log) // (args.reps + 1):]
out["bfs_trace"] = [(d.chosen, d.frontier_nvals) for d in dl]
ms, cc = timed(lambda: gb.connected_components(A), max(1, args.reps // 2))
out["cc_ms"] = round(ms, 3)
out["peak_gpu_gb"] = round(torch.cuda.mem_get_info()[1] / 1e9 - torch.cuda.mem_get_info()[0] / 1e9, 1)
if not args.no_oracle:
    from oracle import cgraph
    rp = A._csr.offsets.cpu().numpy()
    ci = A._csr.indices.cpu().numpy()
    t2 = time.perf_counter()
    want, tr = cgraph.bfs(rp, ci, 0)
    out["cpu_bfs_s"] = round(time.perf_counter() - t2, 2)
    out["bfs_parity"] = bool(np.array_equal(lv.values, want)) and \
        [t[:2] for t in tr] == [tuple(t) for t in out["bfs_trace"]]
    t2 = time.perf_counter()
    labels = cgraph.cc(rp, ci)
    labels = labels[0] if isinstance(labels, tuple) else labels
    out["cpu_cc_s"] = round(time.perf_counter() - t2, 2)
    out["cc_parity"] = bool(np.array_equal(cc.values, labels))
    out["cpu_threads"] = cgraph.threads()
print(json.dumps(out))
