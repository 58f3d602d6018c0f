"""Experiment: the bench's masked pull SpMV on the original labels vs on the
degree-ordered relabelling (x and mask permuted in, w permuted out), device
time per call with CUDA events.

    python tools/mxv_order_probe.py [--scale 24]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200.containers import MaskMode, SparseMatrix, Vector  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()

A = gb.io.rmat_matrix(args.scale)
n = A.nrows
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 0.5
m = (torch.rand(n, device="cuda", generator=g) < 0.5).to(torch.int64)
sr = gb.builtin_semiring("PlusMultiplies")


def run(M, xv, mv):
    u = Vector._wrap(n, None, xv, 0.0, np.float64)
    mask = Vector._wrap(n, None, mv, 0, np.int64)
    d = gb.Descriptor(mask_mode=MaskMode.COMPLEMENT, direction=gb.Direction.FORCE_PULL)
    return gb.mxv(sr, M, u, mask=mask, desc=d)


def timeit(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / args.reps, out


t0, w0 = timeit(lambda: run(A, x, m))
push_o, pull_o, rank = A.traversal()
Ar = SparseMatrix._wrap(n, n, push_o, pull_o, A.dtype, True)
rank_l = rank.long()
order = torch.empty_like(rank_l)
order[rank_l] = torch.arange(n, device="cuda")
xr, mr = x[order], m[order]
t1, w1 = timeit(lambda: run(Ar, xr, mr))
tp, _ = timeit(lambda: (x[order], m[order]))
print(f"original labels: {t0:.4f} ms   relabelled: {t1:.4f} ms   (torch permute of x+mask {tp:.4f} ms)")
print("max rel diff", float(((w1._vals[rank_l] - w0._vals).abs() / w0._vals.abs().clamp_min(1e-300)).max()))
