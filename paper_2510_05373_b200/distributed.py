"""Multi-GPU partitioning of the decode hot path (one process per GPU).

Two strategies:

* Batch / kv-head sharding (`shard_units`): (b, kv-head) units are fully
  independent — each owns its codes, metadata, residual window, S/P and
  adapter — so every rank decodes its own shard with no collective at all
  (weak scaling).

* Sequence-parallel split-KV for one long sequence (`SequenceShardedDecoder`):
  the flushed chunks are split contiguously across ranks; the last rank (the
  tail owner) also holds the residual window and computes the correction
  record.  Each rank emits one LSE record per (b, q-head) — (m, l, y_rot,
  y_raw) — over its chunks; the records are all-gathered over NCCL and merged
  by `kvlc_merge_records` (_reduce_blocks, attention.py:158-194, applied to
  rank-level partials; the correction enters as the m = 0 partial, or
  unscaled in literal mode).  The adapter state S/P is a sum over all flushed
  chunks, so the shards' prefill states are all-reduced once.

The exchange / merge logic is written against a small `ops` interface so the
same code runs on GPUs (libkvlinc kernels, NCCL) and, in the CPU test-suite,
with gloo and the oracle standing in for the kernels.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

G = 128
R = 128


def shard_units(batch: int, kv_heads: int, world: int, rank: int):
    """(b, kvh) units owned by `rank`: contiguous blocks of the batch first,
    then of kv heads when the batch is smaller than the world."""
    units = [(b, h) for b in range(batch) for h in range(kv_heads)]
    per = -(-len(units) // world)
    return units[rank * per:(rank + 1) * per]


@dataclass(frozen=True)
class SeqShard:
    rank: int
    chunk_lo: int     # global index of the first flushed chunk this rank owns
    chunk_hi: int
    tok_lo: int       # token range this rank prefills
    tok_hi: int
    tail: bool        # owns the residual window + correction


def plan_sequence_shards(n_tokens: int, world: int) -> list[SeqShard]:
    """Split one sequence of n_tokens across `world` ranks.

    The streaming rule flushes floor((n - R) / G) chunks (cache.py:129); those
    chunks are split contiguously and evenly, and the remaining window tokens
    go to the last rank, which therefore sees exactly the single-device
    cache's tail."""
    n_chunks = (n_tokens - R) // G if n_tokens >= R else 0
    bounds = np.linspace(0, n_chunks, world + 1).round().astype(int)
    shards = []
    for r in range(world):
        lo, hi = int(bounds[r]), int(bounds[r + 1])
        tail = r == world - 1
        shards.append(SeqShard(r, lo, hi, lo * G, n_tokens if tail else hi * G, tail))
    return shards


class SequenceShardedDecoder:
    """Split-KV decode of long sequences over a process group.

    ops must provide:
      partial(q, include_tail) -> (rec [B, Hq, W], corr [B, Hq, 1 + d])
      merge(recs [n, B, Hq, W], corr, literal) -> out [B, Hq, d]
    (`GpuOps` below binds them to a BatchedKVCache shard.)"""

    def __init__(self, shard: SeqShard, ops, group=None):
        self.shard = shard
        self.ops = ops
        self.group = group

    def decode(self, q: torch.Tensor, literal: bool = False) -> torch.Tensor:
        """One collective per step: every rank's record and correction row travel in one
        all-gather buffer ([rec | corr] per (b, q-head)); the merge takes the tail owner's
        correction (the other ranks' rows are zero)."""
        world = dist.get_world_size(self.group)
        rec, corr = self.ops.partial(q, self.shard.tail)
        wr = rec.shape[-1]
        send = torch.cat([rec, corr.to(rec.dtype)], dim=-1).contiguous()
        buf = torch.empty((world * send.shape[0],) + tuple(send.shape[1:]), dtype=send.dtype,
                          device=send.device)
        dist.all_gather_into_tensor(buf, send, group=self.group)
        buf = buf.view((world,) + tuple(send.shape))
        recs = buf[..., :wr].contiguous()
        corr_all = buf[world - 1, ..., wr:].contiguous()
        return self.ops.merge(recs, corr_all, literal)


def allreduce_states(cache, group=None):
    """Sum the shards' adapter states S, P (each shard accumulated its chunks)."""
    dist.all_reduce(cache.S, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(cache.P, op=dist.ReduceOp.SUM, group=group)


class GpuOps:
    """Binds SequenceShardedDecoder to a BatchedKVCache shard on this GPU."""

    def __init__(self, cache, adapters=None):
        self.cache = cache
        self.adapters = adapters

    def partial(self, q, include_tail):
        n = int(self.cache.n_chunks.max())
        return self.cache.decode_partial(q, 0, n, include_tail, adapters=self.adapters)

    def merge(self, recs, corr, literal):
        from .batched import merge_records
        return merge_records(recs, corr, literal=literal)
