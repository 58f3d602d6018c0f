import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1908_01407_b200 as gb
from paper_1908_01407_b200.containers import Vector
A = gb.io.rmat_matrix(24, a=.25, b=.25, c=.25, d=.25)
n = A.nrows
x = Vector._wrap(n, None, torch.arange(n, dtype=torch.int64, device="cuda"), 0, np.int64)
sr = gb.builtin_semiring("MinimumSelectSecond")
def t():
    d = gb.Descriptor(direction=gb.Direction.FORCE_PULL)
    for _ in range(2): gb.mxv(sr, A, x, desc=d)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): gb.mxv(sr, A, x, desc=d)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 5
print(os.environ.get("GB_MV_STRIPE_BYTES"), round(t(), 3))
