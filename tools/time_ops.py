"""Device time of the operator layer at s24 (R-MAT): push SpMSpV from the hub's
neighbourhood, unmasked pull, reduce_rows, reduce_scalar_matrix, transpose,
ewise on dense vectors -- a scan for operators that serialise on long rows.
python tools/time_ops.py [scale]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200.containers import Vector  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
A = gb.io.rmat_matrix(scale)
n = A.nrows


def dev_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 3)


sr = gb.builtin_semiring("PlusMultiplies")
plus = gb.builtin_monoid("Plus")
o = A.orient(False)
hub_nb = o.indices[int(o.offsets[0]):int(o.offsets[1])].cpu().numpy()
u_sparse = gb.Vector.from_entries(hub_nb, np.ones(hub_nb.size, np.int64), n)
u_dense = Vector._wrap(n, None, torch.ones(n, dtype=torch.float64, device="cuda"), 0.0, np.float64)
push = gb.Descriptor(direction=gb.Direction.FORCE_PUSH)
pull = gb.Descriptor(direction=gb.Direction.FORCE_PULL)
out = {
    "push SpMSpV from the hub's 406K neighbours (324 M products)":
        dev_ms(lambda: gb.vxm(sr, u_sparse, A, desc=push)),
    "pull SpMV, dense x, unmasked": dev_ms(lambda: gb.mxv(sr, A, u_dense, desc=pull)),
    "reduce_rows Plus": dev_ms(lambda: gb.reduce_rows(plus, A)),
    "reduce_scalar_matrix Plus": dev_ms(lambda: gb.reduce_scalar_matrix(plus, A)),
    "transpose": dev_ms(lambda: gb.transpose(A)),
    "ewise_add dense": dev_ms(lambda: gb.ewise_add(gb.algebra.PLUS, u_dense, u_dense)),
}
for k, v in out.items():
    print(f"{v:9.3f} ms  {k}")
