"""Masked pull SpMV at R-MAT scale 24 through the public API:
w<!m> = A (+.*) x with x dense f64, m a seeded 50 % mask (complemented),
forced pull.  Prints device time of the kernel, the algorithmic bytes of
SURVEY §8(d) and GB/s, and checks w against a torch index_add reference."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200 import _lib  # noqa: E402
from paper_1908_01407_b200.containers import MaskMode, Vector  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--density", type=float, default=0.5)
ap.add_argument("--uniform", action="store_true", help="a=b=c=d=.25 instead of R-MAT")
args = ap.parse_args()

A = (gb.io.rmat_matrix(args.scale, a=.25, b=.25, c=.25, d=.25) if args.uniform
     else gb.io.rmat_matrix(args.scale))
n = A.nrows
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 0.5
m = (torch.rand(n, device="cuda", generator=g) < args.density).to(torch.int64)
u = Vector._wrap(n, None, x, 0.0, np.float64)
mask = Vector._wrap(n, None, m, 0, np.int64)
sr = gb.builtin_semiring("PlusMultiplies")
ctx = _lib.context()


def run():
    d = gb.Descriptor(mask_mode=MaskMode.COMPLEMENT, direction=gb.Direction.FORCE_PULL)
    return gb.mxv(sr, A, u, mask=mask, desc=d), d


w, d = run()  # warm-up (builds the row plan)
torch.cuda.synchronize()
ctx.profiling(True)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(args.reps):
    w, d = run()
ev[1].record()
torch.cuda.synchronize()
prof = ctx.prof_read()
ctx.profiling(False)
k_ms = [t for (kind, _a, t) in prof if kind == 8]
kernel_ms = float(np.median(k_ms))
call_ms = ev[0].elapsed_time(ev[1]) / args.reps

# reference: torch index_add over allowed rows
off = A._csr.offsets
rows = torch.repeat_interleave(torch.arange(n, device="cuda"), torch.diff(off))
cols = A._csr.indices.long()
allowed = (m == 0)
keep = allowed[rows]
ref = torch.zeros(n, dtype=torch.float64, device="cuda")
ref.index_add_(0, rows[keep], x[cols[keep]])
got = w._vals
err = float((got - ref).abs().max())
rel = float(((got - ref).abs() / ref.abs().clamp_min(1e-300)).max())

import ctypes  # noqa: E402
rate = ctypes.c_double(0)
st, _k = A._csr.csr_struct(np.float64)
ctx.call("gb_gather_replay_rate", ctypes.byref(st), _lib.ptr(x), ctypes.byref(rate))
c = d.counters
R = int(((torch.diff(off) > 0) & allowed).sum())
E_read = c.matrix_entries_read
bytes_alg = n / 8 + min(2 * R, n + 1) * 8 + E_read * 4 + n * 8 + n * 8
print(json.dumps({
    "workload": f"mxv(PlusMultiplies f64, {'uniform' if args.uniform else 'rmat'}-s{args.scale}, "
                f"x dense, mask=~m {args.density:.0%}), pull",
    "n": n, "nnz": A.nnz, "allowed_rows": R, "entries_read": E_read,
    "multiplies": c.semiring_multiplies, "adds": c.semiring_adds,
    "kernel_ms": round(kernel_ms, 4), "call_ms": round(call_ms, 4),
    "bytes_alg": int(bytes_alg), "GBps": round(bytes_alg / (kernel_ms * 1e-3) / 1e9, 1),
    "gather_ceiling_G_s": round(rate.value / 1e9, 1),
    "gathers_G_s": round(E_read / (kernel_ms * 1e-3) / 1e9, 1),
    "max_abs_err": err, "max_rel_err": rel}))
