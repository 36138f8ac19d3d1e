#!/usr/bin/env python
"""bench.py — fused 2-bit KVLinC decode attention on B200 (BASELINE.json metric).

Workload (BASELINE config 2, the headline): Llama-3-8B attention shapes,
batch 16 per GPU, 32 q / 8 kv heads, d = 128, context 8192, 2-bit KVLinC cache
(G = R = 128, D = 256 random-init adapter per kv head), synthetic bf16 data.
A step = one fused decode (Algorithm 1) for every (sequence, q-head): the split
kernel (correction CTAs incl. phi_q, warp-per-chunk quantized splits streaming 2-bit
chunks by TMA, residual halves) + the LSE combine, PDL-chained, one CUDA graph launch.
The same JSON line carries configs 1 and 3-5, the config-3 sweep, the corrected prefill
attention, the serving loop, bf16 FlashAttention-2 / FlashInfer, the e2e (host in / out)
number and a CPU sample of the reference algorithm.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one rank per GPU: every rank decodes its own
batch-16 shard ((b, kv-head) units are independent — no collective on the
data path), timed with CUDA events, max over ranks; value = tokens/s of the
whole job (weak scaling).

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port, oracle/kvlinc_oracle.py — the reference is pure NumPy) on all
host cores of rank 0, same metric / config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("decode-attn µs/step & HBM GB/s vs roofline; speedup vs bf16 FlashAttn decode")
B, HKV, HQ, CTX, D, G, R, RANK = 16, 8, 32, 8192, 128, 128, 128, 256
REPLICAS = 4   # rotating caches: 4 x 101 MB > 126 MB L2, every step streams from HBM


def algo_bytes_step(b, hkv, hq, nq, nr):
    """One decode step = split_kernel + combine_kernel: packed K/V codes, fp16
    scale / zero, bf16 residual window, fp32 S and P, q / out bf16 per unit, W1q / W2q
    per kv head."""
    g = hq // hkv
    per_unit = (2 * nq * D // 4 + (nq // G) * D * 4 + nq * 4 + nr * D * 4 + D * RANK * 4 + RANK * 4
                + g * D * 2 * 2)
    return b * hkv * per_unit + hkv * 2 * D * (RANK // 2) * 4


def workload_config(world):
    return {"workload": "llama3-8b-shapes fused 2-bit KVLinC decode (BASELINE config 2)",
            "batch_per_gpu": B, "global_batch": B * world, "q_heads": HQ, "kv_heads": HKV,
            "head_dim": D, "ctx": CTX, "bits": 2, "group": G, "residual_window": R,
            "adapter_rank": RANK, "parallelism": f"dp{world} over (b, kv-head) units",
            "l2": f"{REPLICAS} rotating cache replicas ({REPLICAS} x 101 MB > 126 MB L2)"}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines()]
        except OSError:
            return None
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        if not sm:
            return None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for name, val in zip(names, r[5:9]):
                if val.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]),
                "samples": len(sm), "reasons": sorted(reasons)}


# ----------------------------------------------------------------------------- traffic
DECODE_SOURCES = ("kvlc_decode.cu", "kvlc_quant.cuh", "kvlc_quant_wpc.cuh", "kvlc_common.cuh", "kvlc_tc.cuh")


def decode_source_hash():
    import hashlib
    h = hashlib.sha256()
    for f in DECODE_SOURCES:
        h.update(open(os.path.join(ROOT, "paper_2510_05373_b200", "csrc", f), "rb").read())
    return h.hexdigest()


def traffic_record():
    """dram__bytes_read + write per split_kernel launch from the committed ncu capture
    (profiles/split_kernel_traffic.json, tools/update_traffic.py), used only while the hash
    of the decode sources it was captured from matches the sources being benchmarked."""
    tpath = os.path.join(ROOT, "profiles", "split_kernel_traffic.json")
    if not os.path.exists(tpath):
        return None, "no capture"
    t = json.load(open(tpath))
    if t.get("source_sha256") != decode_source_hash():
        return None, "stale: the decode sources changed since the ncu capture"
    return t.get("dram_bytes_per_launch"), f"ncu --set full capture {t.get('capture', '')}".strip()


# ----------------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache, flush_count

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    torch.manual_seed(1234 + rank)
    bank = AdapterBank.initialize(HKV, device=dev)
    caches = []
    for _ in range(REPLICAS):
        c = BatchedKVCache(B, HKV, HQ, CTX + 256, device=dev)
        k = torch.randn(B, HKV, CTX, D, device=dev).bfloat16()
        v = torch.randn(B, HKV, CTX, D, device=dev).bfloat16()
        c.prefill(k, v, adapters=bank)
        del k, v
        caches.append(c)
    torch.cuda.synchronize()
    nq = int(flush_count([CTX])[0]) * G
    nr = CTX - nq
    q = torch.randn(B, HQ, D, device=dev).bfloat16()
    out = torch.empty_like(q)
    K, W = args.steps, args.warmup
    for i in range(W):
        caches[i % REPLICAS].decode(q, adapters=bank, out=out)
    torch.cuda.synchronize()
    # one CUDA graph per replica: the step's split_kernel + combine_kernel (PDL pair)
    graphs = [c.capture_decode(q, adapters=bank, out=out)[0] for c in caches]
    for i in range(W):
        graphs[i % REPLICAS].replay()
    torch.cuda.synchronize()

    # ---- device-resident timed region (inputs resident in HBM) ----
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        t0.record()
        for i in range(K):
            graphs[i % REPLICAS].replay()
        t1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = t0.elapsed_time(t1) / K

    # ---- the dominant kernel: one CUDA graph of KG back-to-back launches (replicas
    # rotating, so every launch streams its codes from HBM), timed with events on the
    # launch stream; the per-launch average excludes the host launch latency ----
    KG = 4 * REPLICAS
    gk = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gk):
        for i in range(KG):
            caches[i % REPLICAS].decode(q, adapters=bank, out=out)
    gk.replay()
    torch.cuda.synchronize()
    reps = max(1, K // KG)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gk.replay()
    e1.record()
    torch.cuda.synchronize()
    split_ms = e0.elapsed_time(e1) / (reps * KG)
    del gk

    # ---- end-to-end through the public API: pinned host q in, host out back, every step ----
    q_host = torch.empty((B, HQ, D), dtype=torch.bfloat16).pin_memory()
    q_host.copy_(q.cpu())
    out_host = torch.empty((B, HQ, D), dtype=torch.bfloat16).pin_memory()
    # one CUDA graph per replica: the step's H2D q copy and the decode, whose combine
    # writes the result into pinned host memory (the step's D2H transfer)
    del graphs
    graphs_e2e = [c.capture_decode(q, adapters=bank, out=out, q_host=q_host, out_host=out_host)[0]
                  for c in caches]
    for i in range(W):
        graphs_e2e[i % REPLICAS].replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(K):
        graphs_e2e[i % REPLICAS].replay()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / K
    del graphs_e2e

    times = torch.tensor([step_ms, split_ms, e2e_ms], device=dev)
    if world > 1:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    step_ms, split_ms, e2e_ms = (float(x) for x in times.tolist())
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak_gbs = float(peaks.get("hbm_gbs", 6650.0))
    multi = None
    if world > 1 and not args.no_extra:   # every rank takes part (collectives)
        torch.cuda.empty_cache()
        multi = run_multi_gpu(args, rank, world, dev, peak_gbs)
    if rank != 0:
        return None

    step_bytes = algo_bytes_step(B, HKV, HQ, nq, nr)
    achieved = step_bytes / (split_ms * 1e-3) / 1e9
    traffic, traffic_note = traffic_record()

    result = {
        "metric": METRIC, "value": B * world / (step_ms * 1e-3), "unit": "tokens/s",
        "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": step_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16 activations / 2-bit codes / fp16 meta / fp32 accumulate",
        "data": "synthetic N(0,1) bf16 K/V/q, random-init adapters (seed = kv head)",
        "config": workload_config(world),
        "us_per_step": step_ms * 1e3,
        "hbm_gbs_step": step_bytes / (step_ms * 1e-3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
                     "frac": achieved / peak_gbs, "traffic": traffic, "traffic_source": traffic_note,
                     "kernel": "split_kernel + combine_kernel (kvlc_decode.cu, the PDL-chained pair "
                               "of one step; traffic: split_kernel)", "split_us": split_ms * 1e3,
                     "algorithmic_bytes_per_launch": step_bytes,
                     "timing": f"mean of {KG}-launch CUDA graph replays (back to back, L2-cold replicas)",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s"},
        "step_roofline_frac": step_bytes / (step_ms * 1e-3) / 1e9 / peak_gbs,
        "e2e": {"value": B * world / (e2e_ms * 1e-3), "unit": "tokens/s",
                "h2d_bytes_per_step": B * HQ * D * 2, "d2h_bytes_per_step": B * HQ * D * 2,
                "ms_per_step": e2e_ms,
                "path": "BatchedKVCache.capture_decode(q_host=, out_host=): kvlc_stage_input copies "
                        "q from pinned host memory, split_kernel, combine_kernel stores out into pinned "
                        "host memory; one CUDA graph launch per step (3 kernels, PDL-chained)",
                "gpu_launches": 3 * K},
        "gpu_launches": 2 * K,
        "launch": "CUDA graph per step: split_kernel_wpc (correction CTAs incl. phi_q, warp-per-chunk "
                  "quantized splits streaming K / V half-chunks by TMA bulk copies, residual halves) + "
                  "combine_kernel (LSE merge per (b, q-head)), chained by programmatic dependent launch",
        "clocks": clk.summary(),
    }
    if multi is not None:
        result["multi_gpu"] = multi
    if world == 1 and not args.no_fa:
        result["bf16_flash_attn"] = run_flash_attn(args, dev, step_ms)
        result["bf16_flashinfer"] = run_flashinfer(args, dev, step_ms)
        fa_us = [x["us_per_step"] for x in (result["bf16_flash_attn"], result["bf16_flashinfer"])
                 if "us_per_step" in x]
        if fa_us:
            result["speedup_vs_best_bf16"] = min(fa_us) / (step_ms * 1e3)
    if world == 1 and not args.no_extra:
        result["serving_loop"] = run_serving_loop(caches[0], q, bank, dev)
        del caches
        torch.cuda.empty_cache()
        result["other_configs"] = run_other_configs(dev, peak_gbs)
    if world == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline_sample()
    return result


def _time_rotating(caches, q, bank, reps=6):
    """Mean decode-step time over a CUDA graph of back-to-back launches that rotate over
    `caches` (replicas whose bytes together exceed the L2, so every launch streams from HBM)."""
    import torch
    out = torch.empty_like(q)
    for c in caches:
        c.decode(q, adapters=bank, out=out)
    kg = 4 * len(caches) if len(caches) > 1 else 8
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(kg):
            caches[i % len(caches)].decode(q, adapters=bank, out=out)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * kg)


def _decode_point(dev, b, hkv, hq, n, peak_gbs):
    """One decode shape, timed over L2-cold rotating replicas (>= 300 MB streamed per cycle)."""
    import torch
    from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache, flush_count
    nq = int(flush_count([n])[0]) * G
    nbytes = algo_bytes_step(b, hkv, hq, nq, n - nq)
    nrep = max(1, min(6, -(-300_000_000 // nbytes)))
    bank = AdapterBank.initialize(hkv, device=dev)
    caches = []
    for _ in range(nrep):
        c = BatchedKVCache(b, hkv, hq, n + 256, device=dev)
        k = torch.randn(b, hkv, n, D, device=dev).bfloat16()
        v = torch.randn(b, hkv, n, D, device=dev).bfloat16()
        c.prefill(k, v, adapters=bank)
        del k, v
        caches.append(c)
    q = torch.randn(b, hq, D, device=dev).bfloat16()
    ms = _time_rotating(caches, q, bank)
    del caches
    torch.cuda.empty_cache()
    return {"us_per_step": ms * 1e3, "tokens_per_s": b / (ms * 1e-3), "hbm_gbs": nbytes / (ms * 1e-3) / 1e9,
            "roofline_frac": nbytes / (ms * 1e-3) / 1e9 / peak_gbs, "algorithmic_bytes": nbytes,
            "l2": f"{nrep} rotating replicas ({nrep * nbytes / 1e6:.0f} MB per cycle)" if nrep > 1
                  else "single cache larger than L2"}


def run_serving_loop(cache, q, bank, dev):
    """Config-2 decode loop with appends, every step a CUDA graph launch
    (BatchedKVCache.capture_serving_step): steady steps append one token per sequence +
    fused decode; every 128 steps all sequences flush in lockstep (the worst case: real
    batches stagger their flushes), a step whose graph also holds the tensor-core ring
    flush.  The graphs of a period are captured ahead (step.prepare()).  Mutates `cache`."""
    import torch
    kt = torch.randn(cache.B, cache.Hkv, D, device=dev).bfloat16()
    vt = torch.randn(cache.B, cache.Hkv, D, device=dev).bfloat16()
    step, out = cache.capture_serving_step(q, kt, vt, adapters=bank)
    # one full flush period first (the process's first flush pays one-time setup)
    step.prepare()
    for _ in range(cache.steps_until_flush() + 1):
        step.replay()
    step.prepare()
    n = cache.steps_until_flush()
    for _ in range(3):
        step.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n - 3):
        step.replay()
    e1.record()
    step.replay()                            # every sequence flushes one chunk
    e2.record()
    torch.cuda.synchronize()
    step_us = e0.elapsed_time(e1) * 1e3 / (n - 3)
    # queued behind the steady steps like every other step of the loop (its graph launch
    # overlaps the GPU work ahead of it; r02 before: timed from an idle GPU, ~20 us of
    # host graph-launch latency inside)
    flush_us = e1.elapsed_time(e2) * 1e3
    return {"graph_step_us": step_us, "flush_step_us": flush_us,
            "us_per_step_amortised": (127 * step_us + flush_us) / 128,
            "note": "append + decode per step, one CUDA graph launch each (steady state, second flush "
                    "period); the flushing step (all 128 units in lockstep) is a graph with the tensor-core "
                    "ring flush (quant_kernel: a key CTA + 2 value CTAs per unit, flush_tc_kernel adding "
                    "into S), timed queued behind the steady steps like them"}


def run_other_configs(dev, peak_gbs):
    """BASELINE configs 3-5 on this GPU.  Configs 3 / 4 time the same fused decode step
    over L2-cold rotating replicas; config 3 also as the batch x context sweep of
    BASELINE.json (B 1 / 16 / 64 x ctx 4k / 32k, plus the B16 x 8k point); config 5 times
    kvlc_prefill (quantize/pack + FWHT + adapter-state update) of Qwen3-8B shapes."""
    import torch
    from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache, flush_count
    out = {"config1_tiny_b1_8heads_ctx1k": _decode_point(dev, 1, 8, 8, 1024, peak_gbs),
           "config3_qwen2.5-7b_b16_ctx8k": _decode_point(dev, 16, 4, 28, 8192, peak_gbs),
           "config4_llama3-8b_b1_ctx128k": _decode_point(dev, 1, 8, 32, 131072, peak_gbs)}
    sweep = {}
    for b, n in ((1, 4096), (16, 4096), (64, 4096), (1, 32768), (16, 32768), (64, 32768)):
        sweep[f"b{b}_ctx{n // 1024}k"] = _decode_point(dev, b, 4, 28, n, peak_gbs)
    out["config3_sweep_qwen2.5-7b"] = sweep
    out["prefill_corrected_attention"] = run_prefill_attention(dev, peak_gbs)
    out["adapter_train_step"] = run_train_step(dev)
    # config 5: prefill of 32k tokens x 8 kv heads (Qwen3-8B attention shapes)
    b, hkv, n = 1, 8, 32768
    bank = AdapterBank.initialize(hkv, device=dev)
    k = torch.randn(b, hkv, n, D, device=dev).bfloat16()
    v = torch.randn(b, hkv, n, D, device=dev).bfloat16()
    times = []
    for i in range(4):
        c = BatchedKVCache(b, hkv, 4 * hkv, n + 256, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        c.prefill(k, v, adapters=bank)
        e1.record()
        torch.cuda.synchronize()
        if i:
            times.append(e0.elapsed_time(e1))
        del c
    ms = statistics.median(times)
    nf = int(flush_count([n])[0])
    nbytes = b * hkv * (2 * n * D * 2 + nf * (2 * G * D // 4 + 4 * D * 2) + (n - nf * G) * D * 2 * 2
                        + (D * RANK + RANK) * 4)
    out["config5_qwen3-8b_prefill_32k"] = {
        "us_per_step": ms * 1e3, "kv_head_tokens_per_s": b * hkv * n / (ms * 1e-3),
        "hbm_gbs": nbytes / (ms * 1e-3) / 1e9, "roofline_frac": nbytes / (ms * 1e-3) / 1e9 / peak_gbs,
        "kernel": "quant_kernel (codes, FWHT, operand images) + flush_tc_kernel (tcgen05: 3-pass fp16 phi_k GEMM, 2-pass S GEMM on exact codes, TMEM accumulators)"}
    return out


def run_multi_gpu(args, rank, world, dev, peak_gbs):
    """N > 1 only: the partitioned configs of BASELINE.json on the whole job.
      * strong scaling, configs 2 and 3: a fixed global batch of 16 sequences sharded by
        batch across the ranks ((b, kv-head) units are independent: no collective);
      * config 4 split-KV: one 131k-token sequence, chunks split contiguously across the
        ranks (distributed.plan_sequence_shards), S / P all-reduced once after prefill,
        each step = kvlc_decode_partial on every rank + ONE all-gather of [record |
        correction] over NCCL + kvlc_merge_records (SequenceShardedDecoder).
    Every time is the max over ranks of CUDA-event time on each rank's stream."""
    import torch
    import torch.distributed as dist
    from paper_2510_05373_b200.batched import AdapterBank, BatchedKVCache, merge_records
    from paper_2510_05373_b200.distributed import (GpuOps, SequenceShardedDecoder, allreduce_states,
                                                   plan_sequence_shards)

    def tmax(x):
        t = torch.tensor([float(x)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    out = {}
    for name, (hkv, hq, n) in {"config2_strong_b16_ctx8k": (8, 32, 8192),
                               "config3_strong_b16_ctx8k": (4, 28, 8192)}.items():
        if 16 % world:
            out[name] = {"skipped": f"global batch 16 does not shard evenly over {world} GPUs"}
            continue
        bl = 16 // world
        dist.barrier()
        pt = _decode_point(dev, bl, hkv, hq, n, peak_gbs)
        us = tmax(pt["us_per_step"])
        out[name] = {"scaling": "strong", "global_batch": 16, "batch_per_gpu": bl, "us_per_step": us,
                     "tokens_per_s": 16 / (us * 1e-6), "algorithmic_bytes_per_gpu": pt["algorithmic_bytes"],
                     "roofline_frac_per_gpu": pt["algorithmic_bytes"] / (us * 1e-6) / 1e9 / peak_gbs,
                     "comm": "none (units independent)"}
    # config 4: sequence-parallel split-KV
    n, hkv, hq = 131072, 8, 32
    shards = plan_sequence_shards(n, world)
    sh = shards[rank]
    gen = torch.Generator(device=dev).manual_seed(4242)   # every rank draws the same sequence
    k = torch.randn(1, hkv, n, D, device=dev, generator=gen).bfloat16()
    v = torch.randn(1, hkv, n, D, device=dev, generator=gen).bfloat16()
    q = torch.randn(1, hq, D, device=dev, generator=gen).bfloat16()
    bank = AdapterBank.initialize(hkv, device=dev)
    cache = BatchedKVCache(1, hkv, hq, sh.tok_hi - sh.tok_lo + 256, device=dev)
    cache.prefill(k[:, :, sh.tok_lo:sh.tok_hi].contiguous(), v[:, :, sh.tok_lo:sh.tok_hi].contiguous(),
                  adapters=bank, keep_window=sh.tail)
    del k, v
    allreduce_states(cache)
    ops = GpuOps(cache, bank)
    dec = SequenceShardedDecoder(sh, ops)
    K, W = args.steps, args.warmup
    for _ in range(W):
        dec.decode(q)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        o = dec.decode(q)
    e1.record()
    torch.cuda.synchronize()
    step_us = tmax(e0.elapsed_time(e1) * 1e3 / K)
    dist.barrier()
    e0.record()
    for _ in range(K):
        rec, corr = ops.partial(q, sh.tail)
    e1.record()
    torch.cuda.synchronize()
    part_us = tmax(e0.elapsed_time(e1) * 1e3 / K)
    send = torch.cat([rec, corr], dim=-1).contiguous()
    buf = torch.empty((world * send.shape[0],) + tuple(send.shape[1:]), dtype=send.dtype, device=dev)
    dist.barrier()
    e0.record()
    for _ in range(K):
        dist.all_gather_into_tensor(buf, send)
        b4 = buf.view((world,) + tuple(send.shape))
        merge_records(b4[..., :rec.shape[-1]].contiguous(), b4[world - 1, ..., rec.shape[-1]:].contiguous())
    e1.record()
    torch.cuda.synchronize()
    merge_us = tmax(e0.elapsed_time(e1) * 1e3 / K)
    nq_local = int(cache.n_chunks[0]) * G
    local_bytes = algo_bytes_step(1, hkv, hq, nq_local, int(cache.res_len[0]) if sh.tail else 0)
    out["config4_splitkv_b1_ctx128k"] = {
        "scaling": "strong", "comm_nranks": world, "us_per_step": step_us, "tokens_per_s": 1 / (step_us * 1e-6),
        "partial_us": part_us, "allgather_merge_us": merge_us,
        "chunks_per_rank": [s2.chunk_hi - s2.chunk_lo for s2 in shards],
        "algorithmic_bytes_per_gpu_rank": local_bytes,
        "collective": "one NCCL all_gather per step of [record | correction] (B x Hq x 389 fp32 per rank)",
        "out_finite": bool(torch.isfinite(o).all().item())}
    return out


def run_train_step(dev):
    """One adapter-calibration step (adapter.py:180-251) in float64 repo
    kernels: the batched loss / gradients over 64 query positions sharing 4096 keys
    (kvlc_adapter_grads) and Adam on the four weights (kvlc_adam_step)."""
    import torch
    from paper_2510_05373_b200 import _lib
    n, b, d, rank = 4096, 64, 128, 256
    g = torch.Generator(device=dev).manual_seed(9)
    f64 = lambda *sh: torch.randn(*sh, device=dev, generator=g, dtype=torch.float64)
    a = torch.softmax(f64(n, n).tril(), -1).contiguous()
    q, kh, ke = f64(n, d), f64(n, d), 0.1 * f64(n, d)
    w = [0.09 * f64(d, rank // 2) for _ in range(4)]
    gr = [torch.empty_like(x) for x in w]
    m = [torch.zeros_like(x) for x in w]
    v2 = [torch.zeros_like(x) for x in w]
    pos = torch.sort(torch.randperm(n, device=dev, generator=g)[:b].int())[0]
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    ws = torch.empty(_lib.load().kvlc_adapter_grads_workspace(n, b, d, rank), dtype=torch.uint8, device=dev)

    def step(t):
        _lib.call("kvlc_adapter_grads", a.data_ptr(), q.data_ptr(), kh.data_ptr(), ke.data_ptr(), n, d, pos.data_ptr(),
                  b, *[x.data_ptr() for x in w], rank, *[x.data_ptr() for x in gr], loss.data_ptr(), ws.data_ptr(),
                  ws.numel(), _lib.stream_handle())
        for i in range(4):
            _lib.call("kvlc_adam_step", w[i].data_ptr(), m[i].data_ptr(), v2[i].data_ptr(), gr[i].data_ptr(),
                      w[i].numel(), 0.01, 0.9, 0.999, 1e-8, t, _lib.stream_handle())

    step(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(2, 7):
        step(t)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    return {"us_per_step": ms * 1e3, "keys": n, "positions": b, "head_dim": d, "rank": rank, "dtype": "f64",
            "kernels": "feature maps, pa_rows_kernel, gemm_f64_kernel x6, softmax_bwd_kernel x2, adam_kernel x4"}


def run_prefill_attention(dev, peak_gbs):
    """Corrected causal prefill attention (attention.py:99-155) on the
    tensor cores: 8 heads x 8192 tokens with rank-256 adapters (kvlc_corrected_attention, the
    fp16 operand images included; phi_q / phi_k precomputed outside the timed region)."""
    import torch
    from paper_2510_05373_b200 import _lib
    heads, n = 8, 8192
    g = torch.Generator(device=dev).manual_seed(5)
    q, k, v = (torch.randn(heads, n, D, device=dev, generator=g) for _ in range(3))
    ph = [torch.softmax(torch.randn(heads, n, 2, 128, device=dev, generator=g), -1).reshape(heads, n, 256)
          for _ in range(2)]
    out = torch.empty_like(q)
    ws = torch.empty(_lib.load().kvlc_corrected_attention_workspace(n, heads, 256), dtype=torch.uint8, device=dev)

    def call():
        _lib.call("kvlc_corrected_attention", q.data_ptr(), k.data_ptr(), v.data_ptr(), ph[0].data_ptr(),
                  ph[1].data_ptr(), n, heads, 256, out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_handle())

    call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    pairs = heads * n * (n + 1) / 2
    flops = pairs * 2 * (D + RANK + D)   # q.k, phi_q.phi_k, w.v once each
    return {"us_per_step": ms * 1e3, "heads": heads, "tokens": n, "adapter_rank": RANK,
            "tflops_algorithmic": flops / (ms * 1e-3) / 1e12,
            "kernel": "pa_kernel (mma.sync m16n8k16, fp16 hi/lo q/k/v in 3 passes, phi in 1 pass, fp32 accumulate)"}


def run_flash_attn(args, dev, ours_ms):
    """bf16 FlashAttention-2 decode (flash_attn_with_kvcache) on the same shapes."""
    import torch
    try:
        from flash_attn import flash_attn_with_kvcache
    except Exception as e:  # pragma: no cover
        return {"unavailable": str(e)}
    kc = torch.randn(B, CTX, HKV, D, device=dev).bfloat16()
    vc = torch.randn(B, CTX, HKV, D, device=dev).bfloat16()
    q = torch.randn(B, 1, HQ, D, device=dev).bfloat16()
    lens = torch.full((B,), CTX, dtype=torch.int32, device=dev)
    for _ in range(args.warmup):
        flash_attn_with_kvcache(q, kc, vc, cache_seqlens=lens)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        flash_attn_with_kvcache(q, kc, vc, cache_seqlens=lens)
    e1.record()
    torch.cuda.synchronize()
    fa_ms = e0.elapsed_time(e1) / args.steps
    fa_bytes = 2 * B * CTX * HKV * D * 2 + 2 * B * HQ * D * 2
    return {"impl": "flash_attn 2.8.3 flash_attn_with_kvcache (bf16 KV)", "us_per_step": fa_ms * 1e3,
            "hbm_gbs": fa_bytes / (fa_ms * 1e-3) / 1e9, "speedup_ours_vs_fa": fa_ms / ours_ms}


def run_flashinfer(args, dev, ours_ms):
    """bf16 FlashInfer batch decode (paged KV, 16-token pages) on the same shapes."""
    import torch
    try:
        import flashinfer
        page = 16
        npages = CTX // page
        kv = torch.randn(B * npages, 2, page, HKV, D, device=dev).bfloat16()
        q = torch.randn(B, HQ, D, device=dev).bfloat16()
        indptr = torch.arange(0, B + 1, device=dev, dtype=torch.int32) * npages
        indices = torch.arange(0, B * npages, device=dev, dtype=torch.int32)
        last = torch.full((B,), page, dtype=torch.int32, device=dev)
        wsbuf = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
        w = flashinfer.BatchDecodeWithPagedKVCacheWrapper(wsbuf, "NHD")
        w.plan(indptr, indices, last, HQ, HKV, D, page, q_data_type=torch.bfloat16, kv_data_type=torch.bfloat16)
        for _ in range(args.warmup):
            w.run(q, kv)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            w.run(q, kv)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
    except Exception as e:  # pragma: no cover
        return {"unavailable": f"{type(e).__name__}: {e}"[:300]}
    fb = 2 * B * CTX * HKV * D * 2 + 2 * B * HQ * D * 2
    return {"impl": f"flashinfer {getattr(flashinfer, '__version__', '?')} BatchDecodeWithPagedKVCacheWrapper "
                    f"(bf16 KV, page {page})", "us_per_step": ms * 1e3, "hbm_gbs": fb / (ms * 1e-3) / 1e9,
            "speedup_ours_vs_flashinfer": ms / ours_ms}


# ----------------------------------------------------------------------------- CPU reference
def _oracle_unit_worker(args):
    """One (b, kv-head) unit of the workload on one core: build its cache with the
    oracle's streaming rule, then time decode_step_blocked for its g q-heads."""
    kvh, reps, seed = args[:3]
    as_is = len(args) > 3 and args[3]
    from threadpoolctl import threadpool_limits
    import numpy as np
    from oracle import kvlinc_oracle as orc
    with threadpool_limits(1):
        g = orc.rng(seed)
        k = g.standard_normal((CTX, D)).astype(np.float32).astype(np.float64)
        v = g.standard_normal((CTX, D)).astype(np.float32).astype(np.float64)
        ad = orc.init_adapter(D, RANK, seed=kvh)
        cache = orc.build_cache(k, v, ad)
        qs = g.standard_normal((HQ // HKV, D))
        times = []
        for _ in range(reps):
            t = time.perf_counter()
            for h in range(HQ // HKV):
                orc.decode_blocked(qs[h], cache, ad, as_is=as_is)
            times.append(time.perf_counter() - t)
        return times


def _config1_worker():
    """BASELINE config 1 on one core: 8 (b, kv-head) units of 1024 tokens (MHA), one decode each."""
    from threadpoolctl import threadpool_limits
    import numpy as np
    from oracle import kvlinc_oracle as orc
    with threadpool_limits(1):
        g = orc.rng(11)
        units = []
        for h in range(8):
            k = g.standard_normal((1024, D)).astype(np.float32).astype(np.float64)
            v = g.standard_normal((1024, D)).astype(np.float32).astype(np.float64)
            ad = orc.init_adapter(D, RANK, seed=h)
            units.append((orc.build_cache(k, v, ad), ad, g.standard_normal(D)))
        times = []
        for _ in range(3):
            t = time.perf_counter()
            for c, ad, qv in units:
                orc.decode_blocked(qv, c, ad)
            times.append(time.perf_counter() - t)
    return statistics.median(times)


def cpu_baseline_sample():
    """Single-core sample: one kv unit (4 q-heads) of the workload, extrapolated
    to the full step (B*Hkv = 128 units); the O(N) value-slicing port (median of 3) and,
    once, the reference's as-is order (whole value store dequantized per block,
    cache.py:110, O(N^2 / G); identical outputs)."""
    t_unit = statistics.median(_oracle_unit_worker((0, 3, 7)))
    t_asis = _oracle_unit_worker((0, 1, 7, True))[0]
    t_c1 = _config1_worker()
    step_s = t_unit * B * HKV
    return {"value": B / step_s, "unit": "tokens/s", "cores": 1, "kind": "port",
            "sample": f"1 of {B * HKV} (b, kv-head) units, {HQ // HKV} q-heads, ctx {CTX}, "
                      f"oracle decode_step_blocked (O(N) value slicing), median of 3; "
                      f"{t_unit * 1e3:.1f} ms per unit, extrapolated x{B * HKV}",
            "ms_per_step": step_s * 1e3,
            "as_is": {"value": B / (t_asis * B * HKV), "unit": "tokens/s", "ms_per_unit": t_asis * 1e3,
                      "sample": "same unit, the reference's whole-store value dequantization per block "
                                "(cache.py:110), 1 run"},
            "config1": {"ms_per_step": t_c1 * 1e3, "unit": "ms per decode step", "cores": 1,
                        "sample": "BASELINE config 1 whole step: B1, 8 MHA heads, ctx 1024, oracle "
                                  "decode_step_blocked per head, median of 3"}}


def run_reference(args, world):
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    K, W = args.steps, args.warmup
    with mp.get_context("fork").Pool(cores) as pool:
        # each worker owns one unit; a step's sample = `cores` units decoded in parallel
        res = pool.map(_oracle_unit_worker, [(i % HKV, K + W, 100 + i) for i in range(cores)])
    per_round = [max(r[i] for r in res) for i in range(W, W + K)]   # wall time of one round
    rounds = -(-B * HKV // cores)
    step_s = statistics.mean(per_round) * rounds
    value = B / step_s
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
            "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": step_s * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "float64 host / float32 block arithmetic (reference semantics)",
            "data": "synthetic N(0,1) K/V/q, random-init adapters",
            "config": workload_config(1),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port",
                             "sample": f"each step: {cores} of {B * HKV} (b, kv-head) units decoded "
                                       f"in parallel (1 per core), x{rounds} rounds extrapolated"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-fa", action="store_true", help="skip the bf16 FlashAttention comparison")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle sample")
    ap.add_argument("--no-extra", action="store_true", help="skip BASELINE configs 3-5 (other_configs)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, world)), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        # KVLC_BENCH_BACKEND=gloo with more ranks than GPUs: a functional check of the
        # multi-rank code paths on one GPU (ranks share it; numbers are not timings of N GPUs)
        backend = os.environ.get("KVLC_BENCH_BACKEND", "nccl")
        local_rank = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    result = run_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
