"""Split of the eager flushing step (config-2 shapes, all 128 units flush): append+flush, then decode."""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache  # noqa: E402
B, H, D = 16, 8, 128
bank = AdapterBank.initialize(H)
for rep in range(2):
    c = BatchedKVCache(B, H, 32, 8192 + 512)
    k = torch.randn(B, H, 8064 + 255, D, device="cuda").bfloat16()
    c.prefill(k, k, adapters=bank)
    q = torch.randn(B, 32, D, device="cuda").bfloat16()
    out = torch.empty_like(q)
    c.decode(q, adapters=bank, out=out)
    kt = torch.randn(B, H, D, device="cuda").bfloat16()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(); c.append(kt, kt, adapters=bank); ev[1].record()
    c.decode(q, adapters=bank, out=out); ev[2].record()
    c.decode(q, adapters=bank, out=out); ev[3].record()
    torch.cuda.synchronize()
    print(f"append+flush {ev[0].elapsed_time(ev[1])*1e3:.0f} us, first decode after {ev[1].elapsed_time(ev[2])*1e3:.0f} us,"
          f" next decode {ev[2].elapsed_time(ev[3])*1e3:.0f} us")
