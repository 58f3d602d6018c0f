import sys, os
sys.path.insert(0, os.getcwd())
import paper_1908_01407_b200 as gb
W = gb.io.rmat_matrix(20, weighted=True)
d = gb.Descriptor()
gb.sssp(W, 0, desc=d)
print(W.nrows, [(x.chosen, x.frontier_nvals) for x in d.direction_log])
