#!/usr/bin/env python
"""BASELINE config 5: KV quantize/pack + FWHT + adapter-state update throughput
on prefill chunks (Qwen3-8B attention shapes: 8 kv heads, d = 128, 32k tokens).

    python tools/bench_prefill.py [--batch B] [--tokens N] [--steps K] [--warmup W]

One step = kvlc_prefill of [B, 8, N, 128] bf16 K/V into an empty 2-bit cache with
random-init adapters (flush of floor((N - R) / G) chunks per (b, kv-head) incl.
the S / P state update, plus the residual-window load).  Prints one JSON line:
tokens/s (sequence tokens x kv heads per second), us/step, algorithmic HBM bytes
and the fraction of the measured copy bandwidth.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache, flush_count  # noqa: E402

D, G, R, RANK = 128, 128, 128, 256


def algo_bytes(B, Hkv, N):
    """Read K, V bf16; write 2-bit codes + fp16 scale/zero of the flushed chunks,
    the bf16 residual window; write S, P once per unit (fp32)."""
    nf = int(flush_count([N])[0])
    units = B * Hkv
    per_unit = 2 * N * D * 2 + nf * (2 * G * D // 4 + 4 * D * 2) + (N - nf * G) * D * 2 * 2 + (D * RANK + RANK) * 4
    return units * per_unit


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--no-adapter", action="store_true")
    args = ap.parse_args()
    B, Hkv, N = args.batch, args.kv_heads, args.tokens
    torch.manual_seed(0)
    k = torch.randn(B, Hkv, N, D, device="cuda").bfloat16()
    v = torch.randn(B, Hkv, N, D, device="cuda").bfloat16()
    bank = None if args.no_adapter else AdapterBank.initialize(Hkv)
    times = []
    for i in range(args.warmup + args.steps):
        c = BatchedKVCache(B, Hkv, 4 * Hkv, N + 256)  # prefill needs an empty cache
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        c.prefill(k, v, adapters=bank)
        e1.record()
        torch.cuda.synchronize()
        if i >= args.warmup:
            times.append(e0.elapsed_time(e1) * 1e3)
        del c
    us = sorted(times)[len(times) // 2]
    nbytes = algo_bytes(B, Hkv, N)
    peak = 6650.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f).get("hbm_gbs", peak))
    except (OSError, ValueError):
        pass
    gbs = nbytes / us / 1e3
    print(json.dumps({"metric": "prefill quantize/pack + FWHT + adapter-state update throughput",
                      "value": B * Hkv * N / us * 1e6, "unit": "kv-head tokens/s", "us_per_step": us,
                      "config": {"workload": "qwen3-8b-shapes prefill (BASELINE config 5)", "batch": B,
                                 "kv_heads": Hkv, "tokens": N, "adapter": not args.no_adapter},
                      "algorithmic_bytes": nbytes, "hbm_gbs": gbs, "roofline_frac": gbs / peak,
                      "peak_gbs": peak}))


if __name__ == "__main__":
    main()
