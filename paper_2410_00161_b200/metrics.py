"""Per-slot eviction metrics on the device.

Drop-in for pkg/src/pagedkv/metrics.py.  ``MetricsStore`` keeps the metric
(fp32), logical index (int32, -1 = empty) and the protected / fresh shields
(one byte each) per physical slot, layout-aligned with the unified pool
(metrics.py:122-186).  ``protected``/``fresh`` are live bool views, like the
reference's numpy arrays, so callers can poke them directly.

The prefill observation-window metric runs on K2 (csrc/window.cu) straight
from the prompt's Q window and K (the reference materialises the (n_q, L, L)
attention first, attention.py:62-89 -> metrics.py:68-89); decode-time
accumulation is fused into K1 (attention.paged_decode) and also available
standalone as ``accumulate_decode`` (metrics.py:189-211).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .cache import BlockTables, SlotHandle, pool_struct

FULL = "full"
WINDOW = "window"
L1 = "L1"
L2 = "L2"


@dataclass(frozen=True)
class MetricConfig:
    mode: str = WINDOW
    aggregation: str = L2
    window: int = 8  # observation window (tokens), window mode
    pool: int = 7  # max-pooling width, odd
    excluded: int = 10  # excluded query window (tokens), full mode
    protect_window: bool = True  # shield observation-window keys from eviction

    def __post_init__(self):
        if self.mode not in (FULL, WINDOW):
            raise ValueError(f"mode must be '{FULL}' or '{WINDOW}'")
        if self.aggregation not in (L1, L2):
            raise ValueError(f"aggregation must be '{L1}' or '{L2}'")
        if self.mode == WINDOW and self.window < 1:
            raise ValueError("window must be >= 1")
        if self.pool < 1 or self.pool % 2 == 0:
            raise ValueError("pool must be odd and >= 1")
        if self.excluded < 0:
            raise ValueError("excluded must be >= 0")

    @property
    def metric_mode(self) -> int:
        """kvc metric_mode code: 1 = L1, 2 = L2."""
        return 2 if self.aggregation == L2 else 1


class MetricsStore:
    """Per-slot eviction state in HBM, aligned with the unified cache."""

    def __init__(self, num_blocks: int, block_size: int, device=None):
        self.device = _lib.require_cuda(device)
        self.num_blocks = num_blocks
        self.block_size = block_size
        shape = (num_blocks, block_size)
        self.metrics = torch.zeros(shape, dtype=torch.float32, device=self.device)
        self.logical = torch.full(shape, -1, dtype=torch.int32, device=self.device)
        self.protected_u8 = torch.zeros(shape, dtype=torch.uint8, device=self.device)
        self.fresh_u8 = torch.zeros(shape, dtype=torch.uint8, device=self.device)

    @property
    def protected(self) -> torch.Tensor:
        return self.protected_u8.view(torch.bool)

    @property
    def fresh(self) -> torch.Tensor:
        return self.fresh_u8.view(torch.bool)

    @property
    def metrics_flat(self) -> torch.Tensor:
        return self.metrics.view(-1)

    @property
    def logical_flat(self) -> torch.Tensor:
        return self.logical.view(-1)

    @property
    def protected_flat(self) -> torch.Tensor:
        return self.protected.view(-1)

    @property
    def fresh_flat(self) -> torch.Tensor:
        return self.fresh.view(-1)

    def on_append(self, handle: SlotHandle, logical: int, fresh: bool = False) -> None:
        """Initialize the slot of a freshly appended KV (metric 0)."""
        self.metrics[handle.block, handle.offset] = 0.0
        self.logical[handle.block, handle.offset] = logical
        self.protected_u8[handle.block, handle.offset] = 0
        self.fresh_u8[handle.block, handle.offset] = int(fresh)

    def write_prompt_pass(self, tables: BlockTables, seq_id: int, layer: int, metrics, protected) -> None:
        """Install prefill metrics for every head of one layer (metrics.py:160-175)."""
        dev = self.device
        m = torch.as_tensor(metrics).to(dev, torch.float32).contiguous()
        L = m.shape[-1]
        prot = None
        if protected is not None:
            prot = torch.as_tensor(np.asarray(protected) if not torch.is_tensor(protected) else protected)
            prot = prot.to(dev).to(torch.uint8).contiguous()
        p = pool_struct(tables=tables, store=self)
        _lib.check(_lib.lib().kvc_write_prompt_pass(ctypes.byref(p), tables.row(seq_id), layer, m.data_ptr(),
                                                    m.stride(0), _lib.ptr(prot), L, _lib.stream_ptr(dev)),
                   "write_prompt_pass")

    def clear_blocks(self, blocks) -> None:
        """Reset freed blocks to the empty-slot state."""
        idx = torch.as_tensor(list(blocks), dtype=torch.long, device=self.device)
        if idx.numel() == 0:
            return
        self.metrics[idx] = 0.0
        self.logical[idx] = -1
        self.protected_u8[idx] = 0
        self.fresh_u8[idx] = 0

    def clear_fresh(self, tables: BlockTables | None = None, seq_ids=None) -> None:
        """Clear the created-this-step shield: every slot (reference semantics,
        metrics.py:185-186) or, given the decode batch, only the slots that step
        created (the last slot of each head)."""
        if seq_ids is None:
            p = pool_struct(store=self)
            _lib.check(_lib.lib().kvc_clear_fresh(ctypes.byref(p), None, 0, _lib.stream_ptr(self.device)),
                       "clear_fresh")
            return
        rows = tables.rows_tensor(seq_ids)
        p = pool_struct(tables=tables, store=self)
        _lib.check(_lib.lib().kvc_clear_fresh(ctypes.byref(p), rows.data_ptr(), rows.numel(),
                                              _lib.stream_ptr(self.device)), "clear_fresh")


def accumulate_decode(store: MetricsStore, tables: BlockTables, seq_id: int, layer: int, rows, cfg: MetricConfig) -> None:
    """Fold one decode step's attention into the live metrics of a layer.

    ``rows[k]`` holds the (group_size, C_k) weights of KV head k's query group
    in slot order (the arrays paged_attention returns); key j gains
    sum over its group of f(A[h, j]) (metrics.py:189-211).
    """
    dev = store.device
    row = tables.row(seq_id)
    ctx = tables.ctx[row, layer].tolist()
    r = None
    cmax = max(ctx) if ctx else 0
    mats = []
    for head, rw in enumerate(rows):
        rw = torch.as_tensor(np.asarray(rw) if not torch.is_tensor(rw) else rw).to(dev, torch.float32)
        if rw.dim() == 1:
            rw = rw[None]
        if rw.shape[-1] != ctx[head]:
            raise ValueError(
                f"attention row covers {rw.shape[-1]} keys but head {head} has {ctx[head]} live KVs"
            )
        r = rw.shape[0]
        mats.append(rw)
    if not mats:
        return
    packed = torch.zeros((len(mats), r, max(cmax, 1)), dtype=torch.float32, device=dev)
    for head, rw in enumerate(mats):
        packed[head, :, : rw.shape[-1]] = rw
    p = pool_struct(tables=tables, store=store)
    _lib.check(_lib.lib().kvc_accumulate_rows(ctypes.byref(p), row, layer, packed.data_ptr(), r,
                                              packed.shape[-1], cfg.metric_mode, _lib.stream_ptr(dev)),
               "accumulate_decode")


# ---------------------------------------------------------------------------
# reference-signature prompt metrics on an explicit attention tensor
# ---------------------------------------------------------------------------


def _attn_call(attn, cfg: MetricConfig, num_kv_heads: int, mode: int) -> torch.Tensor:
    dev = _lib.require_cuda(attn.device if torch.is_tensor(attn) and attn.is_cuda else None)
    a_t = torch.as_tensor(np.asarray(attn) if not torch.is_tensor(attn) else attn).to(dev, torch.float32)
    a_t = a_t.contiguous()
    if a_t.dim() != 3 or a_t.shape[1] != a_t.shape[2]:
        raise ValueError("attn must be (num_query_heads, L, L)")
    n_q, L = a_t.shape[0], a_t.shape[1]
    if n_q % num_kv_heads != 0:
        raise ValueError("query head count not divisible by num_kv_heads")
    out = torch.empty((num_kv_heads, L), dtype=torch.float32, device=dev)
    if L == 0:
        return out
    a = _lib.AttnMetricArgs()
    a.num_query_heads, a.L, a.attn, a.mode = n_q, L, a_t.data_ptr(), mode
    a.window, a.pool, a.excluded, a.aggregation = cfg.window, cfg.pool, cfg.excluded, cfg.metric_mode
    a.metrics_out = out.data_ptr()
    p = _lib.KvcPool()
    p.status = _lib.DeviceContext.get(dev).status.data_ptr()
    p.num_kv_heads = num_kv_heads
    from .cache import with_scratch
    with_scratch(p, dev, num_kv_heads * L * 4 + 256)
    _lib.check(_lib.lib().kvc_attn_metrics(ctypes.byref(p), ctypes.byref(a), _lib.stream_ptr(dev)), "attn_metrics")
    return out


def window_metrics(attn, cfg: MetricConfig, num_kv_heads: int):
    """Observation-window metrics from an (n_q, L, L) causal attention tensor
    (metrics.py:68-89): f of the last ``cfg.window`` rows summed per key over
    the key's query group, max-pooled over keys.  Returns (metrics (H, L) fp32
    device tensor, protected (L,) bool device tensor); NumPy arrays (float64,
    bool) when attn is a NumPy array, as the reference returns.  The serving path
    (prefill_sequence, window_metrics_qk) computes the same from Q and K on
    tcgen05 without the attention tensor."""
    out = _attn_call(attn, cfg, num_kv_heads, 0)
    L = out.shape[1]
    start = max(L - cfg.window, 0)
    protected = torch.arange(L, device=out.device) >= start
    if not cfg.protect_window:
        protected[:] = False
    if _lib.is_host_array(attn):  # NumPy in, NumPy out (the reference's types)
        return _lib.to_host(out), _lib.to_host(protected)
    return out, protected


def full_metrics(attn, cfg: MetricConfig, num_kv_heads: int) -> torch.Tensor:
    """Full-range metrics of an attention tensor: key j aggregates query rows
    i >= j + excluded (metrics.py:92-109).  No pooling, no protection."""
    out = _attn_call(attn, cfg, num_kv_heads, 1)
    return _lib.to_host(out) if _lib.is_host_array(attn) else out


def prompt_metrics(attn, cfg: MetricConfig, num_kv_heads: int):
    """Dispatch on cfg.mode (metrics.py:112-119): (metrics, protected)."""
    if cfg.mode == WINDOW:
        return window_metrics(attn, cfg, num_kv_heads)
    m = full_metrics(attn, cfg, num_kv_heads)
    if _lib.is_host_array(attn):
        return m, np.zeros(m.shape[1], dtype=bool)
    return m, torch.zeros(m.shape[1], dtype=torch.bool, device=m.device)
