"""GPU test rig: device facade objects <-> CPU oracle state (test helper)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import kvc_oracle as O
from paper_2410_00161_b200 import BlockManager, BlockTables, MetricsStore, UnifiedKVCache


def as_np(x) -> np.ndarray:
    """A facade result as NumPy: device tensors are copied back; the
    reference-signature calls already return NumPy for NumPy inputs."""
    return x.cpu().numpy() if torch.is_tensor(x) else np.asarray(x)


class DevRig:
    def __init__(self, num_blocks, block_size, head_dim, layers, heads, max_seqs=8, max_blocks=None):
        self.cache = UnifiedKVCache(num_blocks, block_size, head_dim)
        self.tables = BlockTables(layers, heads, block_size, max_seqs=max_seqs,
                                  max_blocks=max_blocks or 64)
        self.manager = BlockManager(num_blocks, self.tables)
        self.store = MetricsStore(num_blocks, block_size)
        self.b = block_size
        self.d = head_dim
        self.layers = layers
        self.heads = heads
        self.num_blocks = num_blocks

    # -- state transfer -----------------------------------------------------

    def load(self, st: O.OracleState):
        """Install an oracle state verbatim (KV rounded to bf16, metric to fp32)."""
        dev = self.cache.device
        self.cache.keys_flat.copy_(torch.from_numpy(st.keys).to(dev, torch.bfloat16))
        self.cache.values_flat.copy_(torch.from_numpy(st.values).to(dev, torch.bfloat16))
        self.store.metrics_flat.copy_(torch.from_numpy(st.metric).to(dev, torch.float32))
        self.store.logical_flat.copy_(torch.from_numpy(st.logical).to(dev, torch.int32))
        self.store.protected_flat.copy_(torch.from_numpy(st.protected).to(dev))
        self.store.fresh_flat.copy_(torch.from_numpy(st.fresh).to(dev))
        self.manager.free_flag.copy_(torch.from_numpy(st.free.astype(np.uint8)).to(dev))
        tile = 1024
        nt = self.manager.free_tile.numel()
        counts = np.add.reduceat(st.free.astype(np.int64), np.arange(0, nt * tile, tile)[:nt])
        self.manager.free_tile.copy_(torch.from_numpy(counts.astype(np.int32)).to(dev))
        maxb = max([len(t) for rows in st.tables.values() for row in rows for t in row] + [1])
        self.tables.ensure_capacity(maxb + 2)
        for s in sorted(st.tables):
            self.tables.add_sequence(s)
            row = self.tables.row(s)
            for m in range(self.layers):
                for h in range(self.heads):
                    tab = st.tables[s][m][h]
                    if tab:
                        self.tables.tables[row, m, h, : len(tab)] = torch.tensor(tab, dtype=torch.int32)
                    self.tables.nblocks[row, m, h] = len(tab)
                    self.tables.ctx[row, m, h] = int(st.ctx[s][m, h])
            self.tables.ctx_bound[row] = int(st.ctx[s].max()) if st.ctx[s].size else 0
        torch.cuda.synchronize()

    def to_oracle(self) -> O.OracleState:
        st = O.OracleState(self.num_blocks, self.b, self.d, self.layers, self.heads)
        st.keys = self.cache.keys_flat.float().cpu().numpy().astype(np.float64)
        st.values = self.cache.values_flat.float().cpu().numpy().astype(np.float64)
        st.metric = self.store.metrics_flat.cpu().numpy().astype(np.float64)
        st.logical = self.store.logical_flat.cpu().numpy().astype(np.int64)
        st.protected = self.store.protected_flat.cpu().numpy().copy()
        st.fresh = self.store.fresh_flat.cpu().numpy().copy()
        st.free = self.manager.free_flag.cpu().numpy().astype(bool)
        for s, (tabs, ctx) in self.tables.snapshot().items():
            st.tables[s] = tabs
            st.ctx[s] = ctx
        return st


def bf16_round(x: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.asarray(x, dtype=np.float64)).to(torch.bfloat16).double().numpy()


def f32_round(x: np.ndarray) -> np.ndarray:
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def random_state(rng, num_blocks, b, d, layers, heads, seqs, max_len, min_len=1, scatter=True,
                 metric_kind="iid"):
    """Oracle state with random per-head lengths, bf16-exact KV and fp32-exact metrics."""
    st = O.OracleState(num_blocks, b, d, layers, heads)
    if scatter:
        # fragment the pool: pre-take a random subset so ids are non-contiguous
        st.free[rng.random(num_blocks) < 0.3] = False
    for s in seqs:
        st.tables[s] = [[[] for _ in range(heads)] for _ in range(layers)]
        st.ctx[s] = np.zeros((layers, heads), dtype=np.int64)
        for m in range(layers):
            for h in range(heads):
                n = int(rng.integers(min_len, max_len + 1))
                nb = -(-n // b)
                ids = O._take_smallest(st, nb)
                if scatter:
                    ids = rng.permutation(ids)
                st.tables[s][m][h] = [int(x) for x in ids]
                st.ctx[s][m, h] = n
                f = st.live_slots(s, m, h)
                st.keys[f] = bf16_round(rng.standard_normal((n, d)))
                st.values[f] = bf16_round(rng.standard_normal((n, d)))
                if metric_kind == "iid":
                    st.metric[f] = f32_round(rng.random(n))
                else:
                    st.metric[f] = f32_round(np.round(rng.random(n), 1))
                st.logical[f] = np.arange(n)
    if scatter:
        owned = {blk for rows in st.tables.values() for row in rows for t in row for blk in t}
        st.free[:] = True
        st.free[list(owned)] = False
    return st
