"""Cost of the e2e step's host copies: 131 KB pinned H2D + D2H, alone and with the decode graph."""
import torch
B, HQ, D = 16, 32, 128
q = torch.empty((B, HQ, D), dtype=torch.bfloat16, device="cuda")
out = torch.empty_like(q)
qh = torch.empty((B, HQ, D), dtype=torch.bfloat16).pin_memory()
oh = torch.empty((B, HQ, D), dtype=torch.bfloat16).pin_memory()
def timeit(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
print("h2d only us", round(timeit(lambda: q.copy_(qh, non_blocking=True)), 2))
print("d2h only us", round(timeit(lambda: oh.copy_(out, non_blocking=True)), 2))
print("h2d+d2h us", round(timeit(lambda: (q.copy_(qh, non_blocking=True), oh.copy_(out, non_blocking=True))), 2))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    q.copy_(qh, non_blocking=True)
    oh.copy_(out, non_blocking=True)
print("graph h2d+d2h us", round(timeit(g.replay), 2))
big = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
bd = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
t = timeit(lambda: bd.copy_(big, non_blocking=True), 20)
print("h2d 64MB GB/s", round(64 * 2**20 / t / 1e3, 1))
