"""Profiling driver: build an R-MAT graph on the GPU, warm up, then run `reps`
calls of one algorithm inside a cudaProfilerStart/Stop window (use with
`ncu --profile-from-start off`).

    python tools/prof_bfs.py --algo bfs|sssp|pr|cc|ccpush|tc|mxv --scale 24 --reps 1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200.io import rmat_matrix  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--algo", default="bfs")
args = ap.parse_args()

A = (rmat_matrix(args.scale, a=.25, b=.25, c=.25, d=.25) if args.algo.endswith("_u")
     else rmat_matrix(args.scale, weighted=args.algo == "sssp"))
args.algo = args.algo[:-2] if args.algo.endswith("_u") else args.algo   # *_u: uniform graph
gb._lib.context().trim()
if args.algo == "mxvm":
    from paper_1908_01407_b200.containers import Vector
    _g = torch.Generator(device="cuda").manual_seed(1)
    _X = Vector._wrap(A.nrows, None, torch.rand(A.nrows, dtype=torch.float64, device="cuda",
                                                generator=_g) + 0.5, 0.0, np.float64)
    _M = Vector._wrap(A.nrows, None, (torch.rand(A.nrows, device="cuda", generator=_g) < 0.5)
                      .to(torch.int64), 0, np.int64)


if args.algo == "push":
    _o = A.orient(False)
    _nb = _o.indices[int(_o.offsets[0]):int(_o.offsets[1])].cpu().numpy()
    _U = gb.Vector.from_entries(_nb, np.ones(_nb.size, np.int64), A.nrows)
if args.algo == "mxm":
    _L = gb.algorithms._degree_sorted_lower_triangle(A)


def run():
    if args.algo == "bfs":
        gb.bfs(A, 0)
    elif args.algo == "sssp":
        gb.sssp(A, 0)
    elif args.algo == "pr":
        gb.pagerank(A, eps=1e-300, max_iters=3)
    elif args.algo == "cc":
        gb.connected_components(A)
    elif args.algo == "ccpush":   # same labels and iterations, every iteration pushed
        gb.connected_components(A, desc=gb.Descriptor(direction=gb.Direction.FORCE_PUSH))
    elif args.algo == "tc":
        gb.triangle_count(A)
    elif args.algo == "mxvm":
        # bench.py's masked SpMV: w<~m> = A (+.*) x, x dense f64, m 50 % seeded, forced pull
        sr = gb.builtin_semiring("PlusMultiplies")
        d = gb.Descriptor(mask_mode=gb.MaskMode.COMPLEMENT, direction=gb.Direction.FORCE_PULL)
        gb.mxv(sr, A, _X, mask=_M, desc=d)
    elif args.algo == "mxv":
        u = gb.vector_fill(A.nrows, 1.0)
        gb.mxv(gb.builtin_semiring("PlusMultiplies"), A, u)
    elif args.algo == "push":   # operator-level push SpMSpV from the hub's neighbours
        gb.vxm(gb.builtin_semiring("PlusMultiplies"), _U, A,
               desc=gb.Descriptor(direction=gb.Direction.FORCE_PUSH))
    elif args.algo == "mxm":    # the reference's L.L^T .* L masked SpGEMM
        d = gb.Descriptor()
        d.toggle("inp1")
        gb.mxm_masked(gb.builtin_semiring("PlusMultiplies"), _L, _L, mask=_L, desc=d)


for _ in range(2):
    run()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(args.reps):
    run()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
