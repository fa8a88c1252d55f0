"""Block-granular eviction scheduling (K3) and MoveCache compaction (K4).

Drop-in for pkg/src/pagedkv/compression.py.  The reference pipeline
(build_views -> sort_by_head_metric -> eviction_thresholds ->
order_candidate_blocks -> eviction_mask -> move_cache ->
free_schedule_blocks, compression.py:122-309) runs on the GPU without
sorting (csrc/evict.cu):

* ``schedule_evictions`` -> per-head evicted-block counts and the clamped
  per-sequence budgets (bit-exact with the reference given identical
  metrics);
* ``execute_cache_moves`` -> compaction of every evicting head, trailing
  block frees, context reset and logical renumbering;
* ``compress`` -> both in one device pass, returning the reference's
  ``CompressionSchedule`` (same records, same ``to_dict`` schema,
  compression.py:36-119).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Mapping

import numpy as np
import torch

from . import _lib
from .block_manager import BlockManager
from .cache import BlockTables, UnifiedKVCache, pool_struct, with_scratch
from .metrics import MetricsStore


@dataclass
class HeadEviction:
    layer: int
    head: int
    evicted_blocks: int
    evicted_kvs: int
    moves: list  # (src_flat, dst_flat)
    freed: list


@dataclass
class SequenceSchedule:
    seq_id: int
    requested_budget: int
    budget: int  # after clamping
    heads: list = field(default_factory=list)

    @property
    def freed_blocks(self) -> list:
        return [b for h in self.heads for b in h.freed]

    @property
    def evicted_kvs(self) -> int:
        return sum(h.evicted_kvs for h in self.heads)


@dataclass
class CompressionSchedule:
    """Outcome of one compression round, serializable for report streams."""

    sequences: list = field(default_factory=list)

    @property
    def freed_count(self) -> int:
        return sum(len(s.freed_blocks) for s in self.sequences)

    @property
    def evicted_kvs(self) -> int:
        return sum(s.evicted_kvs for s in self.sequences)

    def to_dict(self) -> dict:
        return {
            "freed_blocks": self.freed_count,
            "evicted_kvs": self.evicted_kvs,
            "sequences": [
                {
                    "seq_id": s.seq_id,
                    "requested_budget": s.requested_budget,
                    "budget": s.budget,
                    "heads": [
                        {
                            "layer": h.layer,
                            "head": h.head,
                            "evicted_blocks": h.evicted_blocks,
                            "evicted_kvs": h.evicted_kvs,
                            "freed": list(h.freed),
                            "moves": [list(m) for m in h.moves],
                        }
                        for h in s.heads
                        if h.evicted_blocks
                    ],
                }
                for s in self.sequences
            ],
        }


@dataclass
class EvictionPlan:
    """Device-resident result of a schedule/compress call for one round."""

    seq_ids: list
    requested: list
    rows: torch.Tensor          # int32 [n]
    budgets: torch.Tensor       # int64 [n]
    clamped: torch.Tensor       # int64 [n]
    evict: torch.Tensor         # int32 [n, l*H]
    evicted_kvs: torch.Tensor   # int32 [n, l*H]
    move_offsets: torch.Tensor  # int64 [n*l*H + 1]
    move_counts: torch.Tensor   # int32 [n, l*H]
    totals: torch.Tensor        # int64 [4]: freed, evicted kvs, moves, free blocks
    moves: torch.Tensor | None = None   # int32 [cap, 2]
    freed: torch.Tensor | None = None   # int32 [n, l*H, max_blocks]
    max_slots: int = 0
    executed: bool = False

    def evict_counts(self) -> dict:
        """{seq_id: per-head evicted blocks in layer-major head order}."""
        ev = self.evict.cpu().numpy()
        return {s: ev[i].tolist() for i, s in enumerate(self.seq_ids)}

    def schedule(self, num_layers: int, num_kv_heads: int, record_moves: bool = True) -> CompressionSchedule:
        """Host CompressionSchedule (synchronises)."""
        clamped = self.clamped.cpu().tolist()
        ev = self.evict.cpu().numpy()
        kvs = self.evicted_kvs.cpu().numpy() if self.executed else np.zeros_like(ev)
        offs = self.move_offsets.cpu().numpy()
        cnts = self.move_counts.cpu().numpy() if self.executed else np.zeros_like(ev)
        moves = self.moves.cpu().numpy() if (record_moves and self.executed and self.moves is not None) else None
        freed = self.freed.cpu().numpy() if (self.executed and self.freed is not None) else None
        hp = num_layers * num_kv_heads
        sched = CompressionSchedule()
        for i, s in enumerate(self.seq_ids):
            seq = SequenceSchedule(seq_id=s, requested_budget=self.requested[i], budget=clamped[i])
            sched.sequences.append(seq)
            if clamped[i] <= 0:
                continue
            for h in range(hp):
                e = int(ev[i, h])
                if e == 0:
                    continue
                g = i * hp + h
                mv = []
                if moves is not None:
                    o = int(offs[g])
                    mv = [(int(a), int(b)) for a, b in moves[o: o + int(cnts[i, h])]]
                fr = freed[i, h, :e].tolist() if freed is not None else []
                seq.heads.append(HeadEviction(layer=h // num_kv_heads, head=h % num_kv_heads,
                                              evicted_blocks=e, evicted_kvs=int(kvs[i, h]),
                                              moves=mv, freed=fr))
        return sched


def _prepare(tables: BlockTables, budgets: Mapping[int, int], want_moves: bool, want_freed: bool) -> EvictionPlan:
    dev = tables.device
    seq_ids = list(budgets)
    requested = [int(budgets[s]) for s in seq_ids]
    n = len(seq_ids)
    hp = tables.num_layers * tables.num_kv_heads
    b = tables.block_size
    rows_host = [tables.row(s) for s in seq_ids]
    bound = max((tables.ctx_bound[r] for r in rows_host), default=0)
    max_slots = min(tables.max_blocks, -(-bound // b) + 1) * b
    nb_bound = max_slots // b
    cap = sum(min(max(r, 0), hp * nb_bound) for r in requested) * b + 1
    # inputs go up from pinned staging without a host sync; every output
    # below is written in full by the kernels (K3 writes clamped / evict /
    # move_offsets, K4 move_counts / evicted_kvs, totals are zeroed in-stream)
    stage = torch.tensor(rows_host + requested, dtype=torch.int64).pin_memory().to(dev, non_blocking=True)
    plan = EvictionPlan(
        seq_ids=seq_ids, requested=requested,
        rows=stage[:n].to(torch.int32),
        budgets=stage[n:],
        clamped=torch.empty(n, dtype=torch.int64, device=dev),
        evict=torch.empty((n, hp), dtype=torch.int32, device=dev),
        evicted_kvs=torch.empty((n, hp), dtype=torch.int32, device=dev),
        move_offsets=torch.empty(n * hp + 1, dtype=torch.int64, device=dev),
        move_counts=torch.empty((n, hp), dtype=torch.int32, device=dev),
        totals=torch.empty(4, dtype=torch.int64, device=dev),
        moves=torch.empty((cap, 2), dtype=torch.int32, device=dev) if want_moves else None,
        freed=torch.empty((n, hp, tables.max_blocks), dtype=torch.int32, device=dev) if want_freed else None,
        max_slots=max_slots,
    )
    return plan


def _args(plan: EvictionPlan) -> _lib.EvictArgs:
    a = _lib.EvictArgs()
    a.seq_rows = plan.rows.data_ptr()
    a.budgets = plan.budgets.data_ptr()
    a.n_seqs = len(plan.seq_ids)
    a.max_slots_per_head = plan.max_slots
    a.clamped = plan.clamped.data_ptr()
    a.evict = plan.evict.data_ptr()
    a.evicted_kvs = plan.evicted_kvs.data_ptr()
    a.freed = _lib.ptr(plan.freed)
    a.moves = _lib.ptr(plan.moves)
    a.moves_capacity = plan.moves.shape[0] if plan.moves is not None else 0
    a.move_offsets = plan.move_offsets.data_ptr()
    a.move_counts = plan.move_counts.data_ptr()
    a.totals = plan.totals.data_ptr()
    return a


def _scratch_bytes(plan: EvictionPlan, hp: int) -> int:
    n = len(plan.seq_ids)
    T = n * hp
    # keys + per-head counters + per-sequence digit histograms + candidate lists (short heads)
    # + the K/V copy queue (one u64 per 32 moves of capacity, + one per head)
    cap = plan.moves.shape[0] if plan.moves is not None else 0
    return (T * ((plan.max_slots + 3) // 4 * 4) * 4 + T * 36 + n * (2048 * 4 + 44) + T * 2 * 256 * 8
            + (cap // 32 + T + 2) * 8 + (T * (2 * 2048 + 1024 + 2) * 4 if plan.max_slots > 8192 else 0) + (1 << 16))


def schedule_evictions(tables: BlockTables, store: MetricsStore, budgets: Mapping[int, int],
                       manager: BlockManager | None = None) -> EvictionPlan:
    """Per-head evicted-block counts for each sequence's block budget E_s
    (compression.py:122-231); budgets are clamped to the evictable blocks.
    Asynchronous: returns device tensors; nothing in the cache changes."""
    plan = _prepare(tables, budgets, want_moves=True, want_freed=True)
    if not plan.seq_ids:
        return plan
    hp = tables.num_layers * tables.num_kv_heads
    p = with_scratch(pool_struct(tables=tables, store=store, manager=manager), tables.device,
                     _scratch_bytes(plan, hp))
    a = _args(plan)
    _lib.check(_lib.lib().kvc_schedule_evictions(ctypes.byref(p), ctypes.byref(a), _lib.stream_ptr(tables.device)),
               "schedule_evictions")
    return plan


def execute_cache_moves(cache: UnifiedKVCache, tables: BlockTables, manager: BlockManager,
                        store: MetricsStore, plan: EvictionPlan, sync: bool = True,
                        record_moves: bool = True):
    """Apply a plan: MoveCache compaction, trailing frees, renumbering
    (compression.py:234-309).  Returns the CompressionSchedule (sync=True)
    or the plan with device outputs filled (sync=False)."""
    if plan.seq_ids:
        hp = tables.num_layers * tables.num_kv_heads
        p = with_scratch(pool_struct(cache=cache, tables=tables, manager=manager, store=store), tables.device,
                         _scratch_bytes(plan, hp))
        a = _args(plan)
        _lib.check(_lib.lib().kvc_execute_moves(ctypes.byref(p), ctypes.byref(a), _lib.stream_ptr(tables.device)),
                   "execute_cache_moves")
        plan.executed = True
    return _finish(tables, plan, sync, record_moves)


def _finish(tables, plan, sync, record_moves):
    if not sync:
        return plan
    _lib.DeviceContext.get(tables.device).raise_status()
    sched = plan.schedule(tables.num_layers, tables.num_kv_heads, record_moves)
    refresh_ctx_bounds(tables, plan.seq_ids)
    return sched


def refresh_ctx_bounds(tables: BlockTables, seq_ids) -> None:
    """Tighten the host context bounds of compressed rows (one small read)."""
    if not seq_ids:
        return
    rows = [tables.row(s) for s in seq_ids]
    mx = tables.ctx[torch.tensor(rows, device=tables.device).long()].flatten(1).max(dim=1).values.tolist()
    for r, m in zip(rows, mx):
        tables.ctx_bound[r] = int(m)


def compress(cache: UnifiedKVCache, tables: BlockTables, manager: BlockManager, store: MetricsStore,
             budgets: Mapping[int, int], sync: bool = True, record_moves: bool = True, events=None):
    """Run the full eviction pipeline for a batch of per-sequence budgets
    (compression.py:312-355): one scheduling + compaction pass on the GPU.
    `events` = (start, end) CUDA events recorded around the device work."""
    plan = _prepare(tables, budgets, want_moves=True, want_freed=True)
    if plan.seq_ids:
        hp = tables.num_layers * tables.num_kv_heads
        p = with_scratch(pool_struct(cache=cache, tables=tables, manager=manager, store=store), tables.device,
                         _scratch_bytes(plan, hp))
        a = _args(plan)
        if events:
            events[0].record()
        _lib.check(_lib.lib().kvc_compress(ctypes.byref(p), ctypes.byref(a), _lib.stream_ptr(tables.device)),
                   "compress")
        if events:
            events[1].record()
        plan.executed = True
    return _finish(tables, plan, sync, record_moves)
