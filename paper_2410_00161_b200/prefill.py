"""Prefill write path and observation-window metric (K2).

The reference engine's prefill (pkg/src/pagedkv/engine.py:335-358) scatters a
prompt's K/V into every head's blocks, builds the full (n_q, L, L) causal
attention (attention.py:62-89), reduces it to window metrics
(metrics.py:68-89) and installs them per slot (metrics.py:160-175).  Here
the K/V scatter is one vectorised kernel per layer and the metric is K2
(csrc/window.cu): only the last w query rows are multiplied against K on
tcgen05 tensor cores, and the pooled result is written straight into the
metrics store through the block table.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .attention import AttentionConfig
from .block_manager import BlockManager
from .cache import BlockTables, UnifiedKVCache, pool_struct, with_scratch
from .errors import ConfigError
from .metrics import FULL, WINDOW, MetricConfig, MetricsStore


def _dev_bf16(x, dev) -> torch.Tensor:
    if not torch.is_tensor(x):
        x = torch.as_tensor(np.asarray(x))
    return x.to(dev, torch.bfloat16).contiguous()


def _window_call(q, k, cfg: MetricConfig, num_kv_heads: int, head_dim: int, dev, pool_p=None,
                 seq_row: int = -1, layer: int = 0, metrics_out=None, write_k: bool = False) -> bool:
    """K2 for one layer (q (n_q, L|w', d), k (H, L, d)) or several consecutive
    layers (q (l, n_q, L|w', d), k (l, H, L, d)) in one C call.

    write_k: the kernel also stores the K rows of every whole 16-key block
    into the cache (the prompt's K read once for the metric and the write).
    Returns False, with nothing done, when the shape takes the per-layer
    kernels, which cannot (the caller then scatters K itself)."""
    multi = k.dim() == 4
    if not multi:
        q, k = q[None], k[None]
        if metrics_out is not None:
            metrics_out = metrics_out[None]
    nl, n_q, L = k.shape[0], q.shape[1], k.shape[2]
    w = min(cfg.window, L)
    q_win = q[:, :, L - w:, :] if q.shape[2] == L else q
    if q_win.shape[2] != w:
        raise ValueError(f"query window has {q_win.shape[2]} rows, expected {w}")
    q_win = q_win.contiguous()
    k = k.contiguous()
    a = _lib.WindowArgs()
    a.seq_row = seq_row
    a.layer = layer
    a.num_query_heads = n_q
    a.L = L
    a.q_win = q_win.data_ptr()
    a.k = k.data_ptr()
    a.window = cfg.window
    a.pool = cfg.pool
    a.aggregation = cfg.metric_mode
    a.protect_window = int(cfg.protect_window)
    a.metrics_out = _lib.ptr(metrics_out)
    a.n_layers = nl
    a.q_layer_stride = q_win[0].numel()
    a.k_layer_stride = k[0].numel()
    a.out_layer_stride = metrics_out[0].numel() if metrics_out is not None else 0
    a.write_k = int(bool(write_k))
    if pool_p is None:
        pool_p = _lib.KvcPool()
        pool_p.status = _lib.DeviceContext.get(dev).status.data_ptr()
    pool_p.num_kv_heads = num_kv_heads
    pool_p.head_dim = head_dim
    # raw [2][H][L] f32 + partials [H][<=304][<=64] float2 + barrier counters
    with_scratch(pool_p, dev, num_kv_heads * (2 * (L + 3) * 4 + 304 * 64 * 8 + 64) + (1 << 16))
    rc = _lib.lib().kvc_window_metric(ctypes.byref(pool_p), ctypes.byref(a), _lib.stream_ptr(dev))
    if write_k and rc == _lib.ERR_UNSUPPORTED:
        return False
    _lib.check(rc, "window_metric")
    return True


def window_metrics_qk(q, k, cfg: MetricConfig, num_kv_heads: int, device=None):
    """Observation-window metrics of one layer from its prompt Q and K.

    q: (n_q, L, d) or just the last min(w, L) query rows (n_q, w', d);
    k: (num_kv_heads, L, d).  Returns (metrics (num_kv_heads, L) fp32 tensor,
    protected (L,) bool tensor) like pagedkv.metrics.window_metrics, which the
    reference computes from the full attention tensor (metrics.py:68-89).
    """
    dev = _lib.require_cuda(device if device is not None else (q.device if torch.is_tensor(q) and q.is_cuda else None))
    qt, kt = _dev_bf16(q, dev), _dev_bf16(k, dev)
    L = kt.shape[1]
    out = torch.empty((num_kv_heads, L), dtype=torch.float32, device=dev)
    _window_call(qt, kt, cfg, num_kv_heads, kt.shape[2], dev, metrics_out=out)
    start = max(L - cfg.window, 0)
    protected = torch.arange(L, device=dev) >= start
    if not cfg.protect_window:
        protected[:] = False
    return out, protected


def _full_call(q, k, cfg: MetricConfig, num_kv_heads: int, dev, out) -> None:
    """KVC-full metric of one layer on tcgen05: q (n_q, L, d), k (H, L, d) bf16
    -> out (H, L) f32 (csrc/fullmetric.cu)."""
    n_q, L, d = q.shape
    a = _lib.FullArgs()
    a.num_query_heads = n_q
    a.L = L
    a.q = q.data_ptr()
    a.k = k.data_ptr()
    a.excluded = cfg.excluded
    a.aggregation = cfg.metric_mode
    a.metrics_out = out.data_ptr()
    p = _lib.KvcPool()
    p.status = _lib.DeviceContext.get(dev).status.data_ptr()
    p.num_kv_heads = num_kv_heads
    p.head_dim = d
    nt = -(-L // 128)
    with_scratch(p, dev, n_q * nt * 128 * 4 + (1 << 16))
    _lib.check(_lib.lib().kvc_full_metric(ctypes.byref(p), ctypes.byref(a), _lib.stream_ptr(dev)), "full_metric")


def full_metrics_qk(q, k, cfg: MetricConfig, num_kv_heads: int, device=None):
    """KVC-full metrics of one layer (metrics.py:92-109): q (n_q, L, d) all
    prompt queries, k (num_kv_heads, L, d).  Returns (metrics (H, L) fp32,
    protected (L,) all False) like prompt_metrics in full mode."""
    dev = _lib.require_cuda(device if device is not None else (q.device if torch.is_tensor(q) and q.is_cuda else None))
    qt, kt = _dev_bf16(q, dev), _dev_bf16(k, dev)
    out = torch.empty((num_kv_heads, kt.shape[1]), dtype=torch.float32, device=dev)
    _full_call(qt, kt, cfg, num_kv_heads, dev, out)
    return out, torch.zeros(kt.shape[1], dtype=torch.bool, device=dev)


def _install_full(cache, tables, store, seq_id, qt, kt, cfg: MetricConfig) -> None:
    """Full-mode prefill metric: per layer K_full -> write_prompt_pass (no protection)."""
    dev = cache.device
    nl, H, L = kt.shape[0], kt.shape[1], kt.shape[2]
    buf = torch.empty((H, L), dtype=torch.float32, device=dev)
    row = tables.row(seq_id)
    p = pool_struct(cache=cache, tables=tables, store=store)
    for layer in range(nl):
        _full_call(qt[layer], kt[layer], cfg, H, dev, buf)
        _lib.check(_lib.lib().kvc_write_prompt_pass(ctypes.byref(p), row, layer, buf.data_ptr(), L, None, L,
                                                    _lib.stream_ptr(dev)), "write_prompt_pass")


def write_prefill_kv(cache: UnifiedKVCache, tables: BlockTables, seq_id: int, layer: int, k, v) -> None:
    """Scatter one layer's prompt K/V (heads, L, d) into the head tables; C := L."""
    dev = cache.device
    kt, vt = _dev_bf16(k, dev), _dev_bf16(v, dev)
    L = kt.shape[1]
    p = pool_struct(cache=cache, tables=tables)
    _lib.check(_lib.lib().kvc_write_prefill_kv(ctypes.byref(p), tables.row(seq_id), layer, kt.data_ptr(),
                                               vt.data_ptr(), L, _lib.stream_ptr(dev)), "write_prefill_kv")
    row = tables.row(seq_id)
    tables.ctx_bound[row] = max(tables.ctx_bound[row], L)


def write_prefill_kv_layers(cache: UnifiedKVCache, tables: BlockTables, seq_id: int, k, v,
                            v_only: bool = False) -> None:
    """Scatter every layer's prompt K/V (layers, heads, L, d) in one launch; C := L.
    v_only: V, and K of each head's partial last block only (K2 with
    write_k stored the whole blocks' K rows)."""
    dev = cache.device
    kt, vt = _dev_bf16(k, dev), _dev_bf16(v, dev)
    nl, L = kt.shape[0], kt.shape[2]
    p = pool_struct(cache=cache, tables=tables)
    fn = _lib.lib().kvc_write_prefill_v_layers if v_only else _lib.lib().kvc_write_prefill_kv_layers
    _lib.check(fn(ctypes.byref(p), tables.row(seq_id), 0, nl, kt.data_ptr(), vt.data_ptr(), L, _lib.stream_ptr(dev)),
               "write_prefill_kv_layers")
    row = tables.row(seq_id)
    tables.ctx_bound[row] = max(tables.ctx_bound[row], L)


def prefill_layer(cache: UnifiedKVCache, tables: BlockTables, store: MetricsStore, seq_id: int, layer: int,
                  q, k, v, cfg: MetricConfig) -> None:
    """One layer of the engine prefill: scatter K/V, window metric, install
    (engine.py:340-353).  Asynchronous."""
    if cfg.mode != WINDOW:
        raise ConfigError("mode", "the device prefill metric implements the observation window")
    dev = cache.device
    write_prefill_kv(cache, tables, seq_id, layer, k, v)
    qt, kt = _dev_bf16(q, dev), _dev_bf16(k, dev)
    p = pool_struct(cache=cache, tables=tables, store=store)
    _window_call(qt, kt, cfg, tables.num_kv_heads, cache.head_dim, dev, pool_p=p,
                 seq_row=tables.row(seq_id), layer=layer)


def prefill_sequence(cache: UnifiedKVCache, tables: BlockTables, manager: BlockManager, store: MetricsStore,
                     seq_id: int, q, k, v, cfg: MetricConfig, attn: AttentionConfig | None = None) -> int:
    """Allocate + write + score a prompt: q (l, n_q, L or w, d) (all L rows
    for the full metric), k/v (l, H, L, d).

    Raises PreemptionNeeded (nothing allocated) when the pool is short.
    Returns the number of blocks allocated.  Asynchronous after allocation:
    all layers' scatters, then one K2 call covering every layer.
    """
    dev = cache.device
    L = k.shape[2]
    if cfg.mode == FULL and q.shape[2] != L:
        raise ValueError("the full metric needs every prompt query: q (l, n_q, L, d)")
    demand = manager.allocate_prefill(seq_id, L)
    kt, vt, qt = _dev_bf16(k, dev), _dev_bf16(v, dev), _dev_bf16(q, dev)
    if cfg.mode == FULL:
        write_prefill_kv_layers(cache, tables, seq_id, kt, vt)
        _install_full(cache, tables, store, seq_id, qt, kt, cfg)
        return demand
    # K2 streams the prompt's K anyway: it also stores the whole blocks' K
    # rows, after the scatter has written V (+ each head's partial last K
    # block) and set C := L, so K is read from HBM once instead of twice
    p = pool_struct(cache=cache, tables=tables, store=store)
    if tables.block_size == 16:
        write_prefill_kv_layers(cache, tables, seq_id, kt, vt, v_only=True)
        if _window_call(qt, kt, cfg, tables.num_kv_heads, cache.head_dim, dev, pool_p=p,
                        seq_row=tables.row(seq_id), layer=0, write_k=True):
            return demand
    write_prefill_kv_layers(cache, tables, seq_id, kt, vt)  # shapes K2 cannot store K for
    _window_call(qt, kt, cfg, tables.num_kv_heads, cache.head_dim, dev, pool_p=p, seq_row=tables.row(seq_id), layer=0)
    return demand


def prefill_compress_sequence(cache: UnifiedKVCache, tables: BlockTables, manager: BlockManager,
                              store: MetricsStore, seq_id: int, q, k, v, cfg: MetricConfig, budget_blocks: int,
                              sync: bool = True, record_moves: bool = True, events=None):
    """Prefill a prompt and compress it in one pass, without ever writing the
    rows that are evicted (B200-native fusion of engine.py:340-358's prefill
    with the on-prefill compress, compression.py:312-355).

    Allocation, the window metric (K2) and the schedule/compaction (K3/K4 on
    slot metadata) are the same kernels as prefill_sequence + compress; the
    K/V of each surviving prompt position is then written straight to its
    final slot.  Tables, ctx, free list, slot metadata and the K/V of every
    live slot end up identical to prefill_sequence followed by
    compress(..., {seq_id: budget_blocks}); freed blocks hold no prompt data.
    Returns the CompressionSchedule (sync=True) or the EvictionPlan.
    `events` = (start, end) CUDA events around the device work after allocation.
    """
    from . import compression as C
    if cfg.mode != WINDOW:
        raise ConfigError("mode", "the device prefill metric implements the observation window")
    dev = cache.device
    L = k.shape[2]
    manager.allocate_prefill(seq_id, L)
    kt, vt, qt = _dev_bf16(k, dev), _dev_bf16(v, dev), _dev_bf16(q, dev)
    row = tables.row(seq_id)
    if events:
        events[0].record()
    tables.ctx[row].fill_(L)  # C := L (what the scatter would set); K2 installs positions < C
    tables.ctx_bound[row] = max(tables.ctx_bound[row], L)
    p = pool_struct(cache=cache, tables=tables, store=store)
    _window_call(qt, kt, cfg, tables.num_kv_heads, cache.head_dim, dev, pool_p=p, seq_row=row, layer=0)
    plan = C._prepare(tables, {seq_id: budget_blocks}, want_moves=True, want_freed=True)
    hp = tables.num_layers * tables.num_kv_heads
    T = len(plan.seq_ids) * hp
    slots = (plan.max_slots + 3) // 4 * 4
    p = with_scratch(pool_struct(cache=cache, tables=tables, manager=manager, store=store), dev,
                     C._scratch_bytes(plan, hp))
    src_pos = torch.empty((max(T, 1), slots), dtype=torch.int32, device=dev)
    a = C._args(plan)
    a.src_pos = src_pos.data_ptr()
    _lib.check(_lib.lib().kvc_prefill_compress(ctypes.byref(p), ctypes.byref(a), kt.data_ptr(), vt.data_ptr(), L,
                                               _lib.stream_ptr(dev)), "prefill_compress")
    if events:
        events[1].record()
    plan.executed = True
    plan._keepalive = src_pos
    return C._finish(tables, plan, sync, record_moves)
