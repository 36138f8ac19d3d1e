"""e2e variants for config 2: (a) graph{H2D q copy, kernel -> host out}; (b) graph{kernel reading
pinned q in place -> host out}."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402
B, HKV, HQ, CTX, D = 16, 8, 32, 8192, 128
bank = AdapterBank.initialize(HKV)
caches = []
for _ in range(4):
    c = BatchedKVCache(B, HKV, HQ, CTX + 256)
    k = torch.randn(B, HKV, CTX, D, device="cuda").bfloat16()
    c.prefill(k, k, adapters=bank)
    caches.append(c)
del k
q_host = torch.randn(B, HQ, D).bfloat16().pin_memory()
out_host = torch.empty(B, HQ, D, dtype=torch.bfloat16).pin_memory()
qd = torch.empty(B, HQ, D, dtype=torch.bfloat16, device="cuda")
def run(graphs, n=200):
    for i in range(8):
        graphs[i % 4].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        graphs[i % 4].replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
ga = [c.capture_decode(qd, adapters=bank, q_host=q_host, out_host=out_host)[0] for c in caches]
ref = out_host.clone()
outd = torch.empty(B, HQ, D, dtype=torch.bfloat16, device="cuda")
gc = [c.capture_decode(qd, adapters=bank, q_host=q_host, out=outd)[0] for c in caches]   # H2D + kernel
gd = [c.capture_decode(qd, adapters=bank, out_host=out_host)[0] for c in caches]        # kernel -> host
ge = [c.capture_decode(qd, adapters=bank, out=outd)[0] for c in caches]                 # kernel only
for r in range(2):
    print("a h2d+kernel->host", round(run(ga), 2), " c h2d+kernel", round(run(gc), 2),
          " d kernel->host", round(run(gd), 2), " e kernel", round(run(ge), 2))
