"""CUDA-graph decode step: the serving engine's per-token work (engine.py:
264-300 / 420-444) captured once and replayed.

One replay = K0 decode allocation (every head whose next position opens a
block gets one, block_manager.py:74-97) + for each layer K1 (append + paged
GQA attention + L2/L1 metric, attention.py:92-127, metrics.py:189-211) +
the clear of the created-this-step shield (engine.py:298).  Replaying removes
the per-launch host work (argument structs, ctypes calls), which is what
bounds small decode batches; the kernels are the same ones paged_decode runs.

The graph bakes in device pointers and launch shapes, so it keeps its own
workspace and work-queue, captures with `headroom` decode steps of context
slack (the score rows are sized for it), and is recaptured automatically
when the headroom is used up or the block tables were reallocated.
Device-side conditions (PreemptionNeeded, AllocationOrderError, ...) land in
the status word as usual; check them with DeviceContext.raise_status().

Host I/O (`host_io`): for callers whose per-step inputs live in pinned host
memory, each host buffer set gets its own captured graph in which the Q/K/V
uploads (a copy stream, in layer order, awaited per doubling layer group)
and layer m's output download (a second copy stream, right after layer m)
overlap the other layers' attention, instead of bracketing the whole step.
"""

from __future__ import annotations

import ctypes
import os

import torch

from . import _lib
from .attention import AttentionConfig
from .block_manager import BlockManager
from .cache import BlockTables, UnifiedKVCache, pool_struct
from .metrics import MetricsStore


class DecodeStepGraph:
    """Captured decode step for a fixed batch of sequences.

    Inputs are written into the static buffers ``q`` (layers, B, n_q, d),
    ``k_new`` / ``v_new`` (layers, B, H, d); ``out`` (layers, B, n_q, d)
    receives the attention outputs.  ``step()`` replays asynchronously.
    """

    def __init__(self, cache: UnifiedKVCache, tables: BlockTables, manager: BlockManager, store: MetricsStore,
                 seq_ids, cfg: AttentionConfig, metric_mode: int = 2, fresh: bool = True, headroom: int = 256,
                 buffers: dict | None = None, metric_overlap: bool = True, host_io: list | None = None,
                 allocate: bool = True, clear_fresh: bool = True):
        """allocate / clear_fresh: include the K0 decode allocation and the
        fresh-flag clear in the step (a caller that allocates itself - the
        Engine, which must see PreemptionNeeded before decoding - turns
        them off and replays the layers only)."""
        self.cache, self.tables, self.manager, self.store = cache, tables, manager, store
        self.allocate = allocate
        self.clear_fresh = clear_fresh
        self.seq_ids = list(seq_ids)
        self.cfg = cfg
        self.metric_mode = metric_mode
        self.fresh = fresh
        self.headroom = headroom
        # the metric accumulation of layer m runs on a side branch of the graph
        # beside layer m+1's attention (workspaces alternate between layers)
        self.metric_overlap = metric_overlap and metric_mode != 0
        dev = cache.device
        self.device = dev
        B, l = len(self.seq_ids), tables.num_layers
        H, n_q, d = tables.num_kv_heads, cfg.num_query_heads, cfg.head_dim
        bf = torch.bfloat16
        b = buffers or {}
        self.q = b.get("q", torch.zeros((l, B, n_q, d), dtype=bf, device=dev))
        self.k_new = b.get("k_new", torch.zeros((l, B, H, d), dtype=bf, device=dev))
        self.v_new = b.get("v_new", torch.zeros((l, B, H, d), dtype=bf, device=dev))
        self.out = b.get("out", torch.empty((l, B, n_q, d), dtype=bf, device=dev))
        self.rows = [tables.row(s) for s in self.seq_ids]
        self.rows_t = torch.tensor(self.rows, dtype=torch.int32, device=dev)
        self.alloc_order = sorted(range(B), key=lambda i: self.seq_ids[i])  # reference order: sorted(seq)
        self.rows_sorted_t = torch.tensor([self.rows[i] for i in self.alloc_order], dtype=torch.int32, device=dev)
        self.counts = torch.zeros(B, dtype=torch.int32, device=dev)
        # pinned host buffer sets {q, k_new, v_new, out} shaped like the device ones
        self.host_io = list(host_io or [])
        for h in self.host_io:
            for name in ("q", "k_new", "v_new", "out"):
                x, ref = h[name], getattr(self, name)
                if x.shape != ref.shape or x.dtype != ref.dtype or x.is_cuda or not x.is_pinned():
                    raise ValueError(f"host_io {name}: need a pinned host tensor {tuple(ref.shape)} {ref.dtype}")
        self.graph = None
        self.graphs: dict = {}  # None: device buffers; i: host_io[i]
        self.replays = 0

    # -- capture ------------------------------------------------------------------

    def _bounds(self):
        t = self.tables
        return max(t.ctx_bound[r] for r in self.rows)

    def _prepare(self) -> None:
        """Workspaces, queue and per-layer argument structs shared by the
        captured graphs (rebuilt when the tables are reallocated or the
        context headroom runs out)."""
        t, dev = self.tables, self.device
        B, l, H = len(self.rows), t.num_layers, t.num_kv_heads
        self.cap_ctx = self._bounds() + self.headroom
        t.ensure_capacity(-(-(self.cap_ctx + 1) // t.block_size) + 1)
        self.tables_ptr = t.tables.data_ptr()
        lib = _lib.lib()
        # dedicated workspaces: the shared scratch may be regrown by other calls
        p = pool_struct(cache=self.cache, tables=t, manager=self.manager, store=self.store)
        dec_need = lib.kvc_decode_scratch_bytes(ctypes.byref(p), B, self.cfg.num_query_heads, self.cap_ctx + 1)
        heads = B * l * H
        alloc_need = self.manager.free_tile.numel() * 8 + heads * 8 + (1 << 16)
        nws = (int(os.environ.get("KVC_GRAPH_WS", "2")) if self.metric_overlap else 1)
        self.ws = [torch.empty(max(dec_need, alloc_need) + (1 << 20), dtype=torch.uint8, device=dev)
                   for _ in range(nws)]
        self.queue = torch.zeros(2 + B * H, dtype=torch.int32, device=dev)
        p.scratch, p.scratch_bytes = self.ws[0].data_ptr(), self.ws[0].numel()
        pools = [p]
        for w in self.ws[1:]:
            p1 = pool_struct(cache=self.cache, tables=t, manager=self.manager, store=self.store)
            p1.scratch, p1.scratch_bytes = w.data_ptr(), w.numel()
            pools.append(p1)
        self.side = torch.cuda.Stream(dev) if self.metric_overlap else None
        args = []
        for m in range(l):
            a = _lib.DecodeArgs()
            a.seq_rows = self.rows_t.data_ptr()
            a.batch = B
            a.layer = m
            a.num_query_heads = self.cfg.num_query_heads
            a.q = self.q[m].data_ptr()
            a.k_new = self.k_new[m].data_ptr()
            a.v_new = self.v_new[m].data_ptr()
            a.out = self.out[m].data_ptr()
            a.out_f32 = 0
            a.rows_out = None
            a.rows_stride = 0
            a.metric_mode = self.metric_mode
            a.append_fresh = int(self.fresh)
            a.max_ctx = self.cap_ctx + 1
            a.splits = 0
            a.queue = self.queue.data_ptr()
            a.metric_stream = self.side.cuda_stream if self.side is not None else None
            # layer m > 0 follows layer m-1's kernel B directly on the stream;
            # layer 0 follows the allocator, which writes tables / nblocks
            # (2: no early pull, but room for layer 1's)
            a.early_pull = 1 if m > 0 else 2
            args.append(a)
        self._keep = (pools, args)
        self.graphs = {}
        self.captured_at = self._bounds()

    def _capture(self, key=None) -> None:
        dev = self.device
        if not self._valid_prep():
            self._prepare()
        pools, args = self._keep
        p = pools[0]
        lib = _lib.lib()
        B = len(self.rows)
        h = self.host_io[key] if key is not None else None
        if h is not None:
            self.io_in = getattr(self, "io_in", None) or torch.cuda.Stream(dev)
            self.io_out = getattr(self, "io_out", None) or torch.cuda.Stream(dev)

        def body(s):
            stream = s.cuda_stream
            ev_in = []
            if h is not None:  # every layer's upload, in layer order, beside the step
                fork = torch.cuda.Event()
                fork.record(s)
                self.io_in.wait_event(fork)
                self.io_out.wait_event(fork)
                with torch.cuda.stream(self.io_in):
                    for m in range(len(args)):
                        self.q[m].copy_(h["q"][m], non_blocking=True)
                        self.k_new[m].copy_(h["k_new"][m], non_blocking=True)
                        self.v_new[m].copy_(h["v_new"][m], non_blocking=True)
                        ev = torch.cuda.Event()
                        ev.record(self.io_in)
                        ev_in.append(ev)
            if self.allocate:
                _lib.check(lib.kvc_alloc_decode(ctypes.byref(p), self.rows_sorted_t.data_ptr(), B,
                                                self.counts.data_ptr(), stream), "alloc_decode")
            done = []
            # only the first layer of each doubling group (layers 0 | 1 | 2-3 |
            # 4-7 | ...) waits for the uploads of its group: an extra graph
            # edge into a decode kernel costs its programmatic (PDL) overlap
            # with the previous layer (measured: e2e 10.3k -> 10.6k tok/s
            # against one wait per layer); the group sizes stay ahead of the
            # copy engine
            waits, g0 = {0}, 1
            while g0 < len(args):
                waits.add(g0)
                g0 *= 2
            for m, a in enumerate(args):
                if h is not None and m in waits:
                    nxt = min([w for w in waits if w > m], default=len(args))
                    s.wait_event(ev_in[nxt - 1])
                nws = len(pools)
                grp = max(1, nws // 2)
                if self.side is not None and m % grp == 0 and m + grp - 1 - nws >= 0:
                    # layers m .. m+grp-1 reuse the workspaces of layers m-nws ..
                    # m+grp-1-nws: wait for the last of those metric passes
                    s.wait_event(done[m + grp - 1 - nws])
                _lib.check(lib.kvc_paged_decode(ctypes.byref(pools[m % len(pools)]), ctypes.byref(a), stream),
                           "paged_decode")
                if self.side is not None:
                    ev = torch.cuda.Event()
                    ev.record(self.side)
                    done.append(ev)
                if h is not None:  # layer m's output goes down while the next layers run
                    ev = torch.cuda.Event()
                    ev.record(s)
                    self.io_out.wait_event(ev)
                    with torch.cuda.stream(self.io_out):
                        h["out"][m].copy_(self.out[m], non_blocking=True)
            for ev in done[-2:]:  # join the side branch before the fresh clear
                s.wait_event(ev)
            if h is not None:
                ev = torch.cuda.Event()
                ev.record(self.io_out)
                s.wait_event(ev)
            if self.clear_fresh:
                _lib.check(lib.kvc_clear_fresh(ctypes.byref(p), self.rows_t.data_ptr(), B, stream), "clear_fresh")

        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                body(s)
        torch.cuda.current_stream(dev).wait_stream(s)
        self.graphs[key] = g
        self.graph = g

    def _valid_prep(self) -> bool:
        return (hasattr(self, "_keep") and self.tables.tables.data_ptr() == self.tables_ptr
                and self._bounds() + 1 <= self.cap_ctx)

    def _valid(self) -> bool:
        return self.graph is not None and self._valid_prep()

    def step(self, io: int | None = None) -> torch.Tensor:
        """One decode step for the batch: allocation, every layer, fresh clear.
        Asynchronous; returns the output buffer (``host_io[io]["out"]`` when
        `io` selects a pinned host buffer set, whose inputs are uploaded and
        outputs downloaded inside the step).  The first call runs the step
        eagerly (configuring every kernel outside a capture) and captures the
        graph for the following calls."""
        h = self.host_io[io] if io is not None else None
        if self.graph is None:
            if h is not None:
                self.q.copy_(h["q"], non_blocking=True)
                self.k_new.copy_(h["k_new"], non_blocking=True)
                self.v_new.copy_(h["v_new"], non_blocking=True)
            self._eager_step()
            if h is not None:
                h["out"].copy_(self.out, non_blocking=True)
            self._capture(io)
            return self.out if h is None else h["out"]
        if not self._valid_prep():
            self._prepare()
        if io not in self.graphs:
            self._capture(io)
        self.graphs[io].replay()
        self.tables.ctx_bound.bump_rows(self.rows)
        self.replays += 1
        return self.out if h is None else h["out"]

    def _eager_step(self) -> None:
        """The same step through paged_decode (kernel attributes, tensor maps)."""
        from .attention import paged_decode
        if self.allocate:
            self.manager.allocate_decode_step(self.seq_ids, sync=False)
        for m in range(self.tables.num_layers):
            paged_decode(self.q[m], self.cache, self.tables, None, m, self.cfg, store=self.store,
                         metric_mode=self.metric_mode, k_new=self.k_new[m], v_new=self.v_new[m], fresh=self.fresh,
                         out=self.out[m], rows_tensor=self.rows_t, host_rows=self.rows, early_pull=1 if m > 0 else 2)
        if self.clear_fresh:
            self.store.clear_fresh(self.tables, self.seq_ids)
