import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1908_01407_b200 as gb
A = gb.io.rmat_matrix(16)
def dev(fn, reps=50):
    r = fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0=time.perf_counter(); e0.record()
    for _ in range(reps): r = fn()
    e1.record(); t1=time.perf_counter(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1)/reps,4), round((t1-t0)/reps*1e3,4)
for i in range(3):
    print("plain", dev(lambda: gb.bfs(A, 0)))
    print("desc ", dev(lambda: gb.bfs(A, 0, desc=gb.Descriptor())))
    keep=[]
    print("keep ", dev(lambda: keep.append(gb.bfs(A, 0)) or keep[-1]))
