"""Device time of the operator-level masked SpGEMM (mxm_masked, the
reference's L.L^T .* L triangle count composition) at a few scales, beside
the fused triangle count.  python tools/time_mxm.py [scales]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402


def dev_ms(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 3), r


for scale in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16,18,20").split(",")]:
    A = gb.io.rmat_matrix(scale)
    fused = dev_ms(lambda: gb.triangle_count(A))
    comp = dev_ms(lambda: gb.triangle_count(A, desc=gb.Descriptor(fused=False)))
    L = gb.algorithms._degree_sorted_lower_triangle(A)
    sr = gb.builtin_semiring("PlusMultiplies")

    def masked():
        d = gb.Descriptor()
        d.toggle("inp1")          # L . L^T (algorithms.py:232-236)
        return gb.mxm_masked(sr, L, L, mask=L, desc=d)
    mx = dev_ms(masked)
    print({"scale": scale, "L_nnz": L.nnz, "fused_tc_ms": fused[0], "composed_tc_ms": comp[0],
           "mxm_masked_ms": mx[0], "count": int(fused[1]), "same": int(fused[1]) == int(comp[1])},
          flush=True)
