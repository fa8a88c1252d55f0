"""Paged GQA decode attention over ragged per-KV-head tables (K1).

Drop-in for pagedkv.attention.paged_attention (attention.py:92-127) plus the
batched, fused engine path ``paged_decode``: one launch per layer appends the
step's K/V, attends every (sequence, KV head) of the batch and folds the
attention mass into the eviction metrics (engine.py:426-444,
metrics.py:189-211).  Both run the same sm_100a kernels: csrc/decode_mma.cu
(block size 16, head_dim 64/128/256, group <= 8: TMA ring + mma.sync, split-KV)
and csrc/decode.cu for the other shapes.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .cache import BlockTables, UnifiedKVCache, pool_struct, with_scratch
from .errors import NumericError


@dataclass(frozen=True)
class AttentionConfig:
    num_query_heads: int
    num_kv_heads: int
    head_dim: int
    num_layers: int

    def __post_init__(self):
        if self.num_query_heads % self.num_kv_heads != 0:
            raise ValueError("num_query_heads must be divisible by num_kv_heads")

    @property
    def group_size(self) -> int:
        return self.num_query_heads // self.num_kv_heads


def _bf16(x, dev) -> torch.Tensor:
    if not torch.is_tensor(x):
        x = torch.as_tensor(np.asarray(x))
    return x.to(dev, torch.bfloat16).contiguous()


def paged_decode(query: torch.Tensor, cache: UnifiedKVCache, tables: BlockTables, seq_ids,
                 layer: int, cfg: AttentionConfig, store=None, metric_mode: int = 0,
                 k_new: torch.Tensor | None = None, v_new: torch.Tensor | None = None,
                 fresh: bool = True, out: torch.Tensor | None = None, out_f32: bool = False,
                 rows_out: torch.Tensor | None = None, rows_tensor: torch.Tensor | None = None,
                 host_rows: list | None = None, max_ctx: int | None = None,
                 splits: int = 0, early_pull: int = 0) -> torch.Tensor:
    """Batched single-token decode for one layer (asynchronous, no host sync).

    query (B, n_q, d) bf16; k_new/v_new (B, H, d) bf16 are appended at each
    head's position C before attending (their blocks must already exist);
    metric_mode 1/2 adds sum_h p (L1) or p^2 (L2) to every attended slot's
    metric.  rows_out, if given, receives the (B, H, r, stride) weights.
    Returns out (B, n_q, d) bf16 (f32 with out_f32).

    early_pull: the caller guarantees that the last work on the current
    stream is this same call for another layer (consecutive layers of one
    decode step, with rows_tensor given so nothing is enqueued in between);
    the kernel may then start pulling work and streaming KV before that
    launch finishes (kvc_decode_args.early_pull).  2 marks the first layer
    of such a chain: no early pull, but the launch leaves room for the next
    layer's.
    """
    dev = cache.device
    B = query.shape[0]
    if host_rows is None:
        host_rows = [tables.row(s) for s in seq_ids]
    if rows_tensor is None:
        rows_tensor = torch.tensor(host_rows, dtype=torch.int32, device=dev)
    if out is None:
        out = torch.empty((B, cfg.num_query_heads, cfg.head_dim),
                          dtype=torch.float32 if out_f32 else torch.bfloat16, device=dev)
    append = k_new is not None
    if max_ctx is None:
        max_ctx = max((tables.ctx_bound[r] for r in host_rows), default=1)
        max_ctx += 1 if append else 0
    if append:  # one more KV in this layer of every row (a step's l calls raise the row bound by 1)
        tables.ctx_bound.bump(host_rows, layer)
    a = _lib.DecodeArgs()
    a.seq_rows = rows_tensor.data_ptr()
    a.batch = B
    a.layer = layer
    a.num_query_heads = cfg.num_query_heads
    a.q = query.data_ptr()
    a.k_new = _lib.ptr(k_new)
    a.v_new = _lib.ptr(v_new)
    a.out = out.data_ptr()
    a.out_f32 = int(out.dtype == torch.float32)
    a.rows_out = _lib.ptr(rows_out)
    a.rows_stride = rows_out.shape[-1] if rows_out is not None else 0
    a.metric_mode = metric_mode
    a.append_fresh = int(fresh)
    a.max_ctx = max(1, int(max_ctx))
    a.splits = splits
    a.early_pull = int(early_pull)  # False/0, True/1, or 2 (first layer of a chain)
    p = pool_struct(cache=cache, tables=tables, store=store)
    need = _lib.lib().kvc_decode_scratch_bytes(ctypes.byref(p), B, cfg.num_query_heads, a.max_ctx)
    with_scratch(p, dev, need)
    stream = _lib.stream_ptr(dev)
    a.queue = _lib.DeviceContext.get(dev).decode_queue(2 + B * tables.num_kv_heads, stream or 0).data_ptr()
    _lib.check(_lib.lib().kvc_paged_decode(ctypes.byref(p), ctypes.byref(a), stream), "paged_decode")
    return out


def paged_attention(query, cache: UnifiedKVCache, tables: BlockTables, seq_id: int, layer: int,
                    cfg: AttentionConfig):
    """Single-token decode attention over the paged (possibly compressed) cache.

    ``query`` is (num_query_heads, head_dim).  Each query head gathers the
    live KVs of its KV head through the block table, in slot order 0..C-1.
    Returns the (num_query_heads, head_dim) fp32 output plus, per KV head,
    the (group_size, C) attention weights (attention.py:92-127).
    """
    dev = cache.device
    qt = query if torch.is_tensor(query) else torch.as_tensor(np.asarray(query))
    if not torch.isfinite(qt).all():
        raise NumericError("non-finite values in attention inputs")
    q = _bf16(qt, dev).reshape(1, cfg.num_query_heads, cfg.head_dim)
    row = tables.row(seq_id)
    ctx = tables.ctx[row, layer].tolist()
    cmax = max(max(ctx), 1)
    r = cfg.group_size
    rows = torch.zeros((1, cfg.num_kv_heads, r, cmax), dtype=torch.float32, device=dev)
    rt = torch.tensor([row], dtype=torch.int32, device=dev)
    out = paged_decode(q, cache, tables, None, layer, cfg, out_f32=True, rows_out=rows,
                       rows_tensor=rt, host_rows=[row], max_ctx=cmax)
    _lib.DeviceContext.get(dev).raise_status()
    res = out[0], [rows[0, h, :, : ctx[h]] for h in range(cfg.num_kv_heads)]
    if _lib.is_host_array(query):  # NumPy in, NumPy out (the reference's types)
        return _lib.to_host(res[0]), [_lib.to_host(x) for x in res[1]]
    return res


def dense_attention(q, k, v):
    """Causal multi-head attention over (H, L, d) inputs (attention.py:46-59):
    gqa_attention with one query head per KV head.  Returns (out, attn)."""
    n, d = q.shape[0], q.shape[-1]
    return gqa_attention(q, k, v, AttentionConfig(n, n, d, 1))


def gqa_attention(q, k, v, cfg: AttentionConfig):
    """Dense causal grouped-query attention (attention.py:62-89): query head h
    reads KV head h // group_size.  q (n_q, L, d), k/v (n_k, L, d).  Returns
    (out (n_q, L, d), attn (n_q, L, L)) as fp32 device tensors (NumPy float64
    arrays when q is a NumPy array, as the reference returns); the attention
    is row-stochastic and zero above the diagonal.  Materialises O(n_q L^2)
    like the reference; for prompt metrics at length use window_metrics_qk /
    full_metrics_qk, which never form it."""
    dev = _lib.require_cuda(q.device if torch.is_tensor(q) and q.is_cuda else None)
    f32 = lambda x: torch.as_tensor(np.asarray(x) if not torch.is_tensor(x) else x).to(dev, torch.float32).contiguous()
    qt, kt, vt = f32(q), f32(k), f32(v)
    if not (torch.isfinite(qt).all() and torch.isfinite(kt).all() and torch.isfinite(vt).all()):
        raise NumericError("non-finite values in attention inputs")
    if qt.shape[0] != cfg.num_query_heads or kt.shape[0] != cfg.num_kv_heads:
        raise ValueError("head counts do not match the attention config")
    if kt.shape != vt.shape or qt.shape[1:] != kt.shape[1:]:
        raise ValueError("inconsistent Q/K/V shapes")
    n_q, L, d = qt.shape
    out = torch.empty((n_q, L, d), dtype=torch.float32, device=dev)
    attn = torch.empty((n_q, L, L), dtype=torch.float32, device=dev)
    if L == 0:
        return (_lib.to_host(out), _lib.to_host(attn)) if _lib.is_host_array(q) else (out, attn)
    a = _lib.DenseArgs()
    a.num_query_heads, a.L = n_q, L
    a.q, a.k, a.v, a.out, a.attn = qt.data_ptr(), kt.data_ptr(), vt.data_ptr(), out.data_ptr(), attn.data_ptr()
    p = _lib.KvcPool()
    ctx = _lib.DeviceContext.get(dev)
    p.status = ctx.status.data_ptr()
    p.num_kv_heads = cfg.num_kv_heads
    p.head_dim = d
    _lib.check(_lib.lib().kvc_gqa_attention(ctypes.byref(p), ctypes.byref(a), _lib.stream_ptr(dev)), "gqa_attention")
    ctx.raise_status()
    if _lib.is_host_array(q):  # NumPy in, NumPy out (the reference's types)
        return _lib.to_host(out), _lib.to_host(attn)
    return out, attn
