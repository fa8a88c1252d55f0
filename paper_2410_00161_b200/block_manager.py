"""Device block allocator (K0): smallest-free-first, all-or-nothing.

Drop-in for pkg/src/pagedkv/block_manager.py.  The free pool is a byte flag
per block plus per-1024-block free counts in HBM; allocation is a
scan-compaction over those flags on the GPU (csrc/alloc.cu), handing the
k-th smallest free id to the k-th request exactly like the reference's
min-heap (block_manager.py:34-52).  Request order: prefill = layer-major
heads, a consecutive run per head (:56-72); decode = sorted(seq), then
(layer, head) (:74-97).
"""

from __future__ import annotations

import ctypes
from typing import Iterable, Sequence

import torch

from . import _lib
from .cache import BlockTables, pool_struct, with_scratch
from .errors import BlockOwnershipError, PreemptionNeeded


def blocks_needed_prefill(token_count: int, num_layers: int, num_kv_heads: int, block_size: int) -> int:
    """Blocks a fresh prefill of ``token_count`` tokens allocates: l*H*ceil(L/b)."""
    if token_count < 1:
        raise ValueError("token_count must be >= 1")
    return num_layers * num_kv_heads * -(-token_count // block_size)


class BlockManager:
    """Tracks the device free pool and hands blocks to/from the block tables."""

    def __init__(self, num_blocks: int, tables: BlockTables):
        self.num_blocks = num_blocks
        self.tables = tables
        self.device = tables.device
        tiles = -(-num_blocks // _lib.KVC_FREE_TILE)
        self.free_flag = torch.ones(num_blocks, dtype=torch.uint8, device=self.device)
        counts = torch.full((tiles,), _lib.KVC_FREE_TILE, dtype=torch.int32)
        counts[-1] = num_blocks - (tiles - 1) * _lib.KVC_FREE_TILE
        self.free_tile = counts.to(self.device)

    # -- accounting --------------------------------------------------------------

    @property
    def free_count(self) -> int:
        return int(self.free_tile.sum())

    @property
    def allocated_count(self) -> int:
        return self.num_blocks - self.free_count

    def _pool(self, store=None, scratch=0):
        p = pool_struct(tables=self.tables, manager=self, store=store)
        return with_scratch(p, self.device, scratch)

    def _alloc_scratch(self, demand: int, extra: int = 0) -> int:
        tiles = self.free_tile.numel()
        return tiles * 8 + demand * 4 + extra + (1 << 16)

    # -- allocation ----------------------------------------------------------------

    def _take(self, seq_id: int, layer: int, head: int) -> int:
        """Give one block to one head (the reference's heap pop, :47-52)."""
        t = self.tables
        counts = torch.zeros(t.num_layers * t.num_kv_heads, dtype=torch.int32)
        counts[layer * t.num_kv_heads + head] = 1
        self._alloc_heads(seq_id, counts)
        return t.blocks(seq_id, layer, head)[-1]

    def _alloc_heads(self, seq_id: int, counts: torch.Tensor) -> int:
        """Per-head runs for one sequence; raises PreemptionNeeded when short."""
        t = self.tables
        total = int(counts.sum())
        free = self.free_count
        if total > free:
            raise PreemptionNeeded(total - free)
        row = t.row(seq_id)
        nb_max = int((t.nblocks[row].flatten().cpu() + counts).max()) if total else 0
        t.ensure_capacity(nb_max)
        dev_counts = counts.to(self.device, torch.int32)
        p = self._pool(scratch=self._alloc_scratch(total, counts.numel() * 8))
        _lib.check(_lib.lib().kvc_alloc_heads(ctypes.byref(p), row, dev_counts.data_ptr(), total,
                                              _lib.stream_ptr(self.device)), "alloc_heads")
        _lib.DeviceContext.get(self.device).raise_status()
        return total

    def allocate_prefill(self, seq_id: int, token_count: int) -> int:
        """Allocate ceil(L/b) blocks for every head of a new sequence.

        Raises PreemptionNeeded (allocating nothing) when the pool is short.
        """
        t = self.tables
        if t.has_sequence(seq_id):
            raise ValueError(f"sequence {seq_id} already allocated")
        per_head = -(-token_count // t.block_size)
        demand = per_head * t.num_layers * t.num_kv_heads
        free = self.free_count
        if demand > free:
            raise PreemptionNeeded(demand - free)
        t.add_sequence(seq_id)
        t.ensure_capacity(per_head)
        p = self._pool(scratch=self._alloc_scratch(demand))
        _lib.check(_lib.lib().kvc_alloc_prefill(ctypes.byref(p), t.row(seq_id), per_head,
                                                _lib.stream_ptr(self.device)), "alloc_prefill")
        return demand

    def allocate_decode_step(self, seq_ids: Sequence[int], sync: bool = True):
        """Allocate one block for every head whose next position opens a block.

        Demand is a pure function of the context lengths (order independent).
        Raises PreemptionNeeded naming the shortfall without allocating
        anything.  ``sync=False`` returns the device count tensor instead and
        leaves the status word for a later check (the hot decode path).
        """
        t = self.tables
        ordered = sorted(seq_ids)
        rows = t.rows_tensor(ordered)
        # capacity: a head can gain at most one block per step
        need = max((-(-(t.ctx_bound[t.row(s)] + 1) // t.block_size) for s in ordered), default=0)
        t.ensure_capacity(need)
        counts = torch.zeros(len(ordered), dtype=torch.int32, device=self.device)
        heads = len(ordered) * t.num_layers * t.num_kv_heads
        p = self._pool(scratch=self._alloc_scratch(heads, heads * 4))
        _lib.check(_lib.lib().kvc_alloc_decode(ctypes.byref(p), rows.data_ptr(), len(ordered),
                                               counts.data_ptr(), _lib.stream_ptr(self.device)),
                   "alloc_decode")
        if not sync:
            return counts
        _lib.DeviceContext.get(self.device).raise_status()
        host = counts.tolist()
        by_seq = dict(zip(ordered, host))
        return {s: by_seq[s] for s in seq_ids}

    # -- freeing ---------------------------------------------------------------------

    def free_blocks(self, blocks: Iterable[int], store=None) -> None:
        """Return owned blocks to the pool and drop their table entries.

        Freed blocks must form a trailing slice of their owner's table;
        context lengths are clamped to the remaining capacity
        (block_manager.py:101-129).  Validation reads the tables back.
        """
        blocks = list(blocks)
        if not blocks:
            return
        snap = self.tables.snapshot()
        owner = {}
        for s, (tabs, _) in snap.items():
            for m, row in enumerate(tabs):
                for h, tab in enumerate(row):
                    for blk in tab:
                        owner[blk] = (s, m, h)
        by_head: dict = {}
        for blk in blocks:
            o = owner.get(blk)
            if o is None:
                raise BlockOwnershipError(f"block {blk} is not allocated")
            by_head.setdefault(o, set()).add(blk)
        heads, drop = [], []
        for (s, m, h), freed in by_head.items():
            tab = snap[s][0][m][h]
            keep = len(tab) - len(freed)
            if set(tab[keep:]) != freed:
                raise BlockOwnershipError(
                    f"blocks {sorted(freed)} are not the trailing slice of seq {s} layer {m} head {h}"
                )
            heads.append([self.tables.row(s), m, h])
            drop.append(len(freed))
        self._free_trailing(heads, drop, store)

    def _free_trailing(self, heads, drop, store=None) -> None:
        dev = self.device
        h = torch.tensor(heads, dtype=torch.int32, device=dev).reshape(-1, 3)
        d = torch.tensor(drop, dtype=torch.int32, device=dev)
        p = self._pool(store=store)
        _lib.check(_lib.lib().kvc_free_trailing(ctypes.byref(p), h.data_ptr(), d.data_ptr(), len(drop),
                                                _lib.stream_ptr(dev)), "free_trailing")

    def free_sequence(self, seq_id: int, store=None) -> list[int]:
        """Release every block of a sequence and drop its tables."""
        freed = list(self.tables.owned_blocks(seq_id))
        p = self._pool(store=store)
        _lib.check(_lib.lib().kvc_free_sequence(ctypes.byref(p), self.tables.row(seq_id),
                                                _lib.stream_ptr(self.device)), "free_sequence")
        self.tables.remove_sequence(seq_id)
        return freed
