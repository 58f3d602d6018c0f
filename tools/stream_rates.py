"""Streaming reference rates on this GPU: a 134 MB int64 fill, an int32 -> int64
widening copy (the unpermute traffic) and a 134 MB copy.  python tools/stream_rates.py"""
import torch
n = 16777216
t = torch.empty(n, dtype=torch.int64, device="cuda")
r = torch.randint(0, n, (n,), dtype=torch.int32, device="cuda")
big = torch.empty(2*n, dtype=torch.int32, device="cuda")
def tm(f, reps=50):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
print("fill 134MB int64: %.1f us" % tm(lambda: t.fill_(3)))
print("copy int32->int64 (67MB rd + 134MB wr): %.1f us" % tm(lambda: t.copy_(r)))
print("copy 134MB->134MB: %.1f us" % tm(lambda: t.copy_(big.view(torch.int64))))
