"""Unified device KV pool and per-(sequence, layer, KV-head) block tables.

Drop-in for pkg/src/pagedkv/cache.py.  The pool is one contiguous bf16
allocation of ``num_blocks x block_size x head_dim`` keys and values shared
by every layer and head (cache.py:34-57); a KV at position ``i`` of a head
lives at block ``table[i // b]``, offset ``i % b`` (cache.py:130-140).

Differences from the reference, all forced by device residency:

* tables live in HBM as int32 ``[max_seqs, layers, heads, max_blocks]`` with
  per-head lengths ``nblocks`` and context lengths ``ctx``; ``blocks()``
  returns a *snapshot* list (the reference returns its live list);
* sequence ids map to table rows through a host dictionary;
* the tables grow (re-allocate) when a head would exceed ``max_blocks``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterator

import numpy as np
import torch

from . import _lib
from .errors import AllocationOrderError, CacheCorruptionError, PositionError


@dataclass(frozen=True)
class SlotHandle:
    """Physical address of one KV slot (cache.py:23-31)."""

    block: int
    offset: int

    def flat(self, block_size: int) -> int:
        return self.block * block_size + self.offset


class UnifiedKVCache:
    """Pre-allocated bf16 key/value pool of shape (num_blocks, block_size, head_dim)."""

    def __init__(self, num_blocks: int, block_size: int, head_dim: int, device=None,
                 dtype=torch.bfloat16):
        if num_blocks < 1 or block_size < 1 or head_dim < 1:
            raise ValueError("num_blocks, block_size and head_dim must be >= 1")
        if dtype != torch.bfloat16:
            raise ValueError("the B200 kernels store KV in bf16")
        self.device = _lib.require_cuda(device)
        self.num_blocks = num_blocks
        self.block_size = block_size
        self.head_dim = head_dim
        self.keys = torch.zeros((num_blocks, block_size, head_dim), dtype=dtype, device=self.device)
        self.values = torch.zeros_like(self.keys)

    @property
    def keys_flat(self) -> torch.Tensor:
        # Row-major view: slot (n, o) is row n*block_size + o.
        return self.keys.view(self.num_blocks * self.block_size, self.head_dim)

    @property
    def values_flat(self) -> torch.Tensor:
        return self.values.view(self.num_blocks * self.block_size, self.head_dim)


class CtxBound:
    """Host upper bound on the context length of every (row, layer), so that
    launches size their work without reading C back from the device.

    ``bound[row]`` is the bound over the row's layers and ``bound[row] = v``
    sets every layer of the row; ``bump(rows, layer)`` records one decode
    append to one layer (one paged_decode call), ``bump_rows(rows)`` one to
    every layer (one whole decode step), so a step of l per-layer calls
    raises the row bound by 1, not by l."""

    def __init__(self, max_seqs: int, num_layers: int):
        self.a = np.zeros((max_seqs, max(1, num_layers)), dtype=np.int64)

    def __len__(self) -> int:
        return self.a.shape[0]

    def __getitem__(self, row: int) -> int:
        return int(self.a[row].max())

    def __setitem__(self, row: int, value: int) -> None:
        self.a[row, :] = int(value)

    def bump(self, rows, layer: int) -> None:
        self.a[np.asarray(rows, dtype=np.int64), layer] += 1

    def bump_rows(self, rows) -> None:
        self.a[np.asarray(rows, dtype=np.int64), :] += 1


class BlockTables:
    """Device block tables + context lengths for up to ``max_seqs`` sequences."""

    def __init__(self, num_layers: int, num_kv_heads: int, block_size: int,
                 max_seqs: int = 64, max_blocks: int | None = None, device=None):
        self.device = _lib.require_cuda(device)
        self.num_layers = num_layers
        self.num_kv_heads = num_kv_heads
        self.block_size = block_size
        self.max_seqs = max_seqs
        self.max_blocks = max_blocks or 64
        shape = (max_seqs, num_layers, num_kv_heads)
        self.tables = torch.zeros(shape + (self.max_blocks,), dtype=torch.int32, device=self.device)
        self.nblocks = torch.zeros(shape, dtype=torch.int32, device=self.device)
        self.ctx = torch.zeros(shape, dtype=torch.int32, device=self.device)
        self._rows: dict[int, int] = {}
        self._free_rows = list(range(max_seqs - 1, -1, -1))
        # host upper bound on any head's context length, per (row, layer) (no sync)
        self.ctx_bound = CtxBound(max_seqs, num_layers)

    # -- capacity ---------------------------------------------------------------

    def ensure_capacity(self, max_blocks: int) -> None:
        """Grow the per-head table capacity (stream-ordered copy)."""
        if max_blocks <= self.max_blocks:
            return
        new = max(max_blocks, int(self.max_blocks * 1.5))
        grown = torch.zeros(self.tables.shape[:3] + (new,), dtype=torch.int32, device=self.device)
        grown[..., : self.max_blocks] = self.tables
        self.tables = grown
        self.max_blocks = new

    # -- sequence lifecycle -------------------------------------------------------

    def add_sequence(self, seq_id: int) -> None:
        if seq_id in self._rows:
            raise ValueError(f"sequence {seq_id} already has tables")
        if not self._free_rows:
            raise ValueError(f"no free table row (max_seqs={self.max_seqs})")
        row = self._free_rows.pop()
        self._rows[seq_id] = row
        self.nblocks[row].zero_()
        self.ctx[row].zero_()
        self.ctx_bound[row] = 0

    def remove_sequence(self, seq_id: int) -> None:
        row = self._rows.pop(seq_id)
        self.nblocks[row].zero_()
        self.ctx[row].zero_()
        self.ctx_bound[row] = 0
        self._free_rows.append(row)

    def has_sequence(self, seq_id: int) -> bool:
        return seq_id in self._rows

    @property
    def sequences(self) -> list[int]:
        return list(self._rows)

    def row(self, seq_id: int) -> int:
        return self._rows[seq_id]

    def rows_tensor(self, seq_ids) -> torch.Tensor:
        return torch.tensor([self._rows[s] for s in seq_ids], dtype=torch.int32, device=self.device)

    # -- per-head access (synchronising reads) -------------------------------------

    def blocks(self, seq_id: int, layer: int, head: int) -> list[int]:
        row = self._rows[seq_id]
        n = int(self.nblocks[row, layer, head])
        return self.tables[row, layer, head, :n].tolist()

    def context_len(self, seq_id: int, layer: int, head: int) -> int:
        return int(self.ctx[self._rows[seq_id], layer, head])

    def set_context_len(self, seq_id: int, layer: int, head: int, value: int) -> None:
        row = self._rows[seq_id]
        self.ctx[row, layer, head] = value
        self.ctx_bound.a[row, layer] = max(int(self.ctx_bound.a[row, layer]), int(value))

    def heads(self, seq_id: int) -> Iterator[tuple[int, int]]:
        for layer in range(self.num_layers):
            for head in range(self.num_kv_heads):
                yield layer, head

    def owned_blocks(self, seq_id: int) -> Iterator[int]:
        row = self._rows[seq_id]
        nb = self.nblocks[row].cpu().numpy()
        tab = self.tables[row].cpu().numpy()
        for layer, head in self.heads(seq_id):
            yield from tab[layer, head, : nb[layer, head]].tolist()

    def sequence_block_count(self, seq_id: int) -> int:
        return int(self.nblocks[self._rows[seq_id]].sum())

    def allocated_kv_count(self, seq_id: int) -> int:
        return int(self.ctx[self._rows[seq_id]].sum())

    def head_slots_flat(self, seq_id: int, layer: int, head: int) -> np.ndarray:
        """Flat slot indices of every allocated slot of a head, in table order."""
        blocks = np.asarray(self.blocks(seq_id, layer, head), dtype=np.int64)
        b = self.block_size
        return (blocks[:, None] * b + np.arange(b, dtype=np.int64)).ravel()

    def slot_for(self, seq_id: int, layer: int, head: int, position: int) -> SlotHandle:
        b = self.block_size
        table = self.blocks(seq_id, layer, head)
        u, o = divmod(position, b)
        if u >= len(table):
            raise CacheCorruptionError(
                f"position {position} of seq {seq_id} layer {layer} head {head} "
                f"maps to table entry {u} but only {len(table)} blocks are allocated"
            )
        return SlotHandle(table[u], o)

    def snapshot(self):
        """Host copy {seq_id: (tables list[l][H] of lists, ctx (l, H))}."""
        nb = self.nblocks.cpu().numpy()
        tab = self.tables.cpu().numpy()
        ctx = self.ctx.cpu().numpy()
        out = {}
        for s, row in self._rows.items():
            out[s] = (
                [[tab[row, m, h, : nb[row, m, h]].tolist() for h in range(self.num_kv_heads)]
                 for m in range(self.num_layers)],
                ctx[row].astype(np.int64),
            )
        return out


def pool_struct(cache=None, tables=None, manager=None, store=None, device=None) -> _lib.KvcPool:
    """Assemble the C-ABI pool descriptor from whichever facade objects a call
    needs; missing parts are NULL (the kernels skip them)."""
    ref = cache or tables or manager or store
    dev = device or ref.device
    dctx = _lib.DeviceContext.get(dev)
    p = _lib.KvcPool()
    if cache is not None:
        p.k_cache = cache.keys.data_ptr()
        p.v_cache = cache.values.data_ptr()
        p.head_dim = cache.head_dim
        p.num_blocks = cache.num_blocks
        p.block_size = cache.block_size
    if store is not None:
        p.metric = store.metrics.data_ptr()
        p.logical = store.logical.data_ptr()
        p.protected_ = store.protected_u8.data_ptr()
        p.fresh = store.fresh_u8.data_ptr()
        p.num_blocks = store.num_blocks
        p.block_size = store.block_size
    if manager is not None:
        p.free_flag = manager.free_flag.data_ptr()
        p.free_tile = manager.free_tile.data_ptr()
        p.num_blocks = manager.num_blocks
    if tables is not None:
        p.tables = tables.tables.data_ptr()
        p.nblocks = tables.nblocks.data_ptr()
        p.ctx = tables.ctx.data_ptr()
        p.block_size = tables.block_size
        p.num_layers = tables.num_layers
        p.num_kv_heads = tables.num_kv_heads
        p.max_seqs = tables.max_seqs
        p.max_blocks = tables.max_blocks
    p.status = dctx.status.data_ptr()
    return p


def with_scratch(p: _lib.KvcPool, device, nbytes: int) -> _lib.KvcPool:
    buf = _lib.DeviceContext.get(device).scratch(nbytes)
    p.scratch = buf.data_ptr()
    p.scratch_bytes = buf.numel()
    return p


def lookup_kv(tables: BlockTables, cache: UnifiedKVCache, seq_id: int, layer: int, head: int,
              position: int):
    """Read the key/value vectors stored at a head's logical position (cache.py:143-160)."""
    ctx = tables.context_len(seq_id, layer, head)
    if position < 0 or position >= ctx:
        raise PositionError(f"position {position} out of range for context length {ctx}")
    handle = tables.slot_for(seq_id, layer, head, position)
    return cache.keys[handle.block, handle.offset].clone(), cache.values[handle.block, handle.offset].clone()


def append_kv(tables: BlockTables, cache: UnifiedKVCache, seq_id: int, layer: int, head: int,
              key, value) -> SlotHandle:
    """Store one KV at the head's next position; the backing block must exist
    (cache.py:163-184).  Runs the kvc_append_kv kernel (store untouched)."""
    ctx = tables.context_len(seq_id, layer, head)
    try:
        handle = tables.slot_for(seq_id, layer, head, ctx)
    except CacheCorruptionError as exc:
        raise AllocationOrderError(
            f"no block allocated for position {ctx} of seq {seq_id} layer {layer} head {head}"
        ) from exc
    dev = cache.device
    k = torch.as_tensor(np.asarray(key) if not torch.is_tensor(key) else key).to(dev, torch.bfloat16).reshape(1, -1)
    v = torch.as_tensor(np.asarray(value) if not torch.is_tensor(value) else value).to(dev, torch.bfloat16).reshape(1, -1)
    heads = torch.tensor([[tables.row(seq_id), layer, head]], dtype=torch.int32, device=dev)
    p = pool_struct(cache=cache, tables=tables)
    _lib.check(_lib.lib().kvc_append_kv(_lib.ctypes.byref(p), heads.data_ptr(), k.data_ptr(), v.data_ptr(),
                                        1, 0, _lib.stream_ptr(dev)), "append_kv")
    tables.ctx_bound[tables.row(seq_id)] = max(tables.ctx_bound[tables.row(seq_id)], ctx + 1)
    return handle


def fragmentation(tables: BlockTables) -> int:
    """Total allocated-but-unused slots across all heads (cache.py:187-198)."""
    b = tables.block_size
    if not tables.sequences:
        return 0
    rows = tables.rows_tensor(tables.sequences).long()
    lens = tables.ctx[rows].long()
    return int(((lens + b - 1) // b * b - lens).sum())
