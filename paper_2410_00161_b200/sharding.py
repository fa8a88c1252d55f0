"""Multi-GPU: sequences are the shard unit; the only collective is an
all-gather of per-rank eviction / free-block counters.

The reference couples nothing across sequences except the shared free pool
(compress loops sequences independently, compression.py:327-354; budgets are
per sequence, engine.py:367-377; decode is per (seq, layer),
attention.py:92-127).  So each rank owns a private unified cache, free pool
and tables for its sequences (rank-local block ids) and no KV, metric or table
ever crosses NVLink.  After a compression round every rank contributes
(free blocks, blocks freed, KVs evicted, moves) to one NCCL all-gather so the
scheduler on every rank sees the global memory picture.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_sequences(seq_ids, rank: int, world: int) -> list:
    """Round-robin placement: sequence s lives on rank s mod world (in input order)."""
    return [s for i, s in enumerate(seq_ids) if i % world == rank]


def gather_counts(counts, group=None) -> list:
    """All-gather a short list of int64 counters from every rank.

    NCCL (CUDA tensors) when the default backend is nccl, else gloo on CPU.
    Returns [[counts of rank 0], [counts of rank 1], ...].
    """
    if not dist.is_available() or not dist.is_initialized():
        return [list(counts)]
    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    local = torch.tensor(list(counts), dtype=torch.int64, device=dev)
    out = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(out, local, group=group)
    return [t.tolist() for t in out]


def gather_round_counts(manager, round_counts, group=None) -> list:
    """(free blocks, freed, evicted KVs, moves) of every rank after a round."""
    return gather_counts([manager.free_count] + list(round_counts), group)
