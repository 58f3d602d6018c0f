"""Small runs of this round's kernels for compute-sanitizer (memcheck /
racecheck): triangle count (bitmap, dense rows, hash set, fallback, long-row
tiles), CC (first pull both ways, transposed pulls), SSSP (heavy-push pull),
the push accumulator, the device-resident partitioned BFS.
    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_01407_b200 as gb  # noqa: E402
from paper_1908_01407_b200 import distributed as gbd  # noqa: E402

A = gb.io.rmat_matrix(16)
W = gb.io.rmat_matrix(16, weighted=True)
print("tc", gb.triangle_count(A))
print("cc", int(gb.connected_components(A).values.max()))
o = A.orient(False)
off = o.offsets.cpu().numpy()
idx = o.indices.cpu().numpy().copy()
for r in range(0, A.nrows, 3):
    idx[off[r]:off[r + 1]] = idx[off[r]:off[r + 1]][::-1].copy()
U = gb.SparseMatrix.from_csr(A.nrows, A.ncols, off, idx, np.ones(idx.size, np.int64), symmetric=True)
print("cc unsorted", int(gb.connected_components(U).values.max()))
print("sssp", float(np.nanmax(np.where(np.isinf(gb.sssp(W, 0).values), np.nan,
                                       gb.sssp(W, 0).values))))
u = gb.Vector.from_entries(np.arange(0, 2000, 3), np.ones(667, np.int64), A.nrows)
d = gb.Descriptor(direction=gb.Direction.FORCE_PUSH)
print("push", gb.vxm(gb.builtin_semiring("MinPlus"), u, A, desc=d).nvals)
g = gbd.BlockGraph.from_matrix(A, 0, 1)
print("dist", int(gbd.bfs_partitioned_device(g, 0).max()))
run = gbd.OrderedPartitionedBfs(A, 0, 1)
print("dist ordered", int(run(0).max()))
torch.cuda.synchronize()
print("done")
