"""CPU, world_size 2 (gloo): the sequence-parallel split-KV exchange.

Exercises `distributed.plan_sequence_shards`, the S/P all-reduce, the record
all-gather and the LSE merge rule of `SequenceShardedDecoder` with the
oracle standing in for the GPU kernels (`OracleOps`), against the
single-process blocked decode (decode_step_blocked, attention.py:197-276).
The GPU binding of the same decoder is `distributed.GpuOps`.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import kvlinc_oracle as orc
from paper_2510_05373_b200.distributed import (SequenceShardedDecoder, plan_sequence_shards,
                                               shard_units)

D = 64          # small head dim keeps the oracle fast; the rule is dimension independent
RANK_D = 32
LOG2E = 1.4426950408889634


def make_data(n, hq, seed=3):
    g = orc.rng(seed)
    return g.standard_normal((n, D)), g.standard_normal((n, D)), g.standard_normal((hq, D))


class OracleOps:
    """Record producer / merger restating the kernels' math in float64."""

    def __init__(self, cache, adapter):
        self.c = cache
        self.ad = adapter

    def partial(self, q, include_tail):
        c, hq = self.c, q.shape[0]
        rec = np.zeros((1, hq, 4 + 2 * D))
        corr = np.zeros((1, hq, 1 + D))
        nq = c.quantized_tokens
        for h in range(hq):
            parts = []
            if nq:
                parts.append(("rot", c.keys_dequant(0, nq), c.values_dequant(0, nq)))
            if include_tail and c.residual_len:
                parts.append(("raw", c.residual_keys(), c.residual_values()))
            logits = [kk @ q[h] / np.sqrt(D) * LOG2E for _, kk, _ in parts]
            if not parts:
                rec[0, h, 0] = -np.inf
                continue
            m = max(lg.max() for lg in logits)
            rec[0, h, 0] = m
            for (basis, _, vv), lg in zip(parts, logits):
                p = np.exp2(lg - m)
                rec[0, h, 1] += p.sum()
                off = 4 if basis == "rot" else 4 + D
                rec[0, h, off:off + D] += p @ vv
            if include_tail and self.ad is not None and c.s_state is not None:
                fq = orc.phi_q(self.ad, q[h])
                corr[0, h, 0] = c.p_state @ fq
                corr[0, h, 1:] = c.s_state @ fq
        return torch.from_numpy(rec), torch.from_numpy(corr)

    def merge(self, recs, corr, literal):
        recs, corr = recs.numpy(), corr.numpy()
        n, _, hq, _ = recs.shape
        out = np.zeros((1, hq, D))
        H = orc.hadamard(D)
        for h in range(hq):
            m = recs[:, 0, h, 0]
            M = m.max()
            w = np.where(np.isfinite(m), np.exp2(m - M), 0.0)
            den = (w * recs[:, 0, h, 1]).sum()
            nr = (w[:, None] * recs[:, 0, h, 4:4 + D]).sum(0)
            nw = (w[:, None] * recs[:, 0, h, 4 + D:]).sum(0)
            cd, cn = corr[0, h, 0], corr[0, h, 1:]
            if cd != 0 or np.any(cn):
                if literal:
                    nr, den = nr + cn, den + cd
                elif M >= 0:
                    s = np.exp2(-M)
                    nr, den = nr + s * cn, den + s * cd
                else:
                    s = np.exp2(M)
                    nr, nw, den = s * nr + cn, s * nw, s * den + cd
            out[0, h] = (nr @ H.T + nw) / den
        return torch.from_numpy(out)


def _worker(rank, world, port, n, hq, literal, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        k, v, q = make_data(n, hq)
        ad = orc.init_adapter(D, RANK_D, seed=2)
        sh = plan_sequence_shards(n, world)[rank]
        c = orc.build_cache(k[sh.tok_lo:sh.tok_hi], v[sh.tok_lo:sh.tok_hi], ad,
                            window=128 if sh.tail else 0)
        assert c.quantized_tokens == (sh.chunk_hi - sh.chunk_lo) * 128
        # S/P are sums over all flushed chunks: all-reduce the shards' states
        s = torch.from_numpy(c.s_state if c.s_state is not None else np.zeros((D, RANK_D)))
        p = torch.from_numpy(c.p_state if c.p_state is not None else np.zeros(RANK_D))
        dist.all_reduce(s)
        dist.all_reduce(p)
        c.s_state, c.p_state = s.numpy(), p.numpy()
        dec = SequenceShardedDecoder(sh, OracleOps(c, ad))
        out = dec.decode(q, literal=literal).numpy()[0]
        if rank == 0:
            result_q.put(out)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n,literal", [(1500, False), (1300, True), (300, False)])
def test_split_kv_two_ranks_matches_single_device(n, literal):
    world, hq = 2, 3
    ctx = mp.get_context("spawn")
    q_out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, hq, literal, q_out))
             for r in range(world)]
    for p in procs:
        p.start()
    out = q_out.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    k, v, q = make_data(n, hq)
    ad = orc.init_adapter(D, RANK_D, seed=2)
    full = orc.build_cache(k, v, ad)
    ref = np.stack([orc.decode_blocked(q[h], full, ad, literal=literal) for h in range(hq)])
    assert np.max(np.abs(out - ref)) <= 1e-5 * max(1.0, np.abs(ref).max())


def test_plans():
    sh = plan_sequence_shards(131072, 8)
    assert sum(s.chunk_hi - s.chunk_lo for s in sh) == (131072 - 128) // 128
    assert sh[-1].tail and not any(s.tail for s in sh[:-1])
    assert sh[0].tok_lo == 0 and sh[-1].tok_hi == 131072
    assert all(a.tok_hi == b.tok_lo for a, b in zip(sh, sh[1:]))
    units = [shard_units(16, 8, 8, r) for r in range(8)]
    assert sum(len(u) for u in units) == 128 and len({x for u in units for x in u}) == 128
