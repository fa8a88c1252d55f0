"""CPU oracle for the KV-Compress variable-head-rate paged-KV path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2410_00161_b200`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs use it, always as the checker or
the timed CPU baseline, never as the product path.

This is a restatement (not a copy) of the reference ``pagedkv`` package's
algorithm for the hot path, written against the flat array layout the device
uses so device state can be loaded into it verbatim:

* slot ``f = block * b + offset`` is row ``f`` of ``keys``/``values``/per-slot
  arrays (``pkg/src/pagedkv/cache.py:50-57``);
* per-(seq, layer, head) block lists and context lengths
  (``cache.py:60-140``);
* smallest-free-first block allocation (``block_manager.py:34-97``);
* paged single-query GQA decode (``attention.py:92-127``) and decode metric
  accumulation (``metrics.py:189-211``);
* observation-window metrics restated over the last ``w`` query rows only
  (``attention.py:62-89`` -> ``metrics.py:68-89``), avoiding the reference's
  (n_q, L, L) attention tensor;
* the eviction pipeline ``compress`` (``compression.py:122-355``).

All numerics are float64; integer/index outputs are exact.  Parity is pinned
by ``tests/test_oracle_golden.py`` against (a) the reference test suite's
known-answer tests, re-expressed, and (b) golden vectors produced by running
the reference itself (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


class OracleError(Exception):
    """Base class; ``kind`` names the reference exception class raised."""

    def __init__(self, kind: str, message: str = ""):
        super().__init__(f"{kind}: {message}")
        self.kind = kind


class OraclePreemption(Exception):
    """Restates ``PreemptionNeeded(shortfall)`` (errors.py:59-67)."""

    def __init__(self, shortfall: int):
        super().__init__(f"short by {shortfall} blocks")
        self.shortfall = shortfall


# ---------------------------------------------------------------------------
# State
# ---------------------------------------------------------------------------


@dataclass
class OracleState:
    """Pool + per-slot store + tables, in the device's flat layout.

    ``keys``/``values`` are (N*b, d) float64 (cache.py:47-57).  Per-slot
    ``metric`` f64, ``logical`` int64 (-1 = empty), ``protected``/``fresh``
    bool (metrics.py:130-134).  ``free`` marks free block ids; allocation
    always takes the smallest free ids (block_manager.py:34-52).
    """

    num_blocks: int
    block_size: int
    head_dim: int
    num_layers: int
    num_kv_heads: int
    keys: np.ndarray = field(init=False)
    values: np.ndarray = field(init=False)
    metric: np.ndarray = field(init=False)
    logical: np.ndarray = field(init=False)
    protected: np.ndarray = field(init=False)
    fresh: np.ndarray = field(init=False)
    free: np.ndarray = field(init=False)
    tables: dict = field(init=False)  # seq -> list[l][H] of python lists
    ctx: dict = field(init=False)  # seq -> (l, H) int64

    def __post_init__(self):
        slots = self.num_blocks * self.block_size
        self.keys = np.zeros((slots, self.head_dim))
        self.values = np.zeros((slots, self.head_dim))
        self.metric = np.zeros(slots)
        self.logical = np.full(slots, -1, dtype=np.int64)
        self.protected = np.zeros(slots, dtype=bool)
        self.fresh = np.zeros(slots, dtype=bool)
        self.free = np.ones(self.num_blocks, dtype=bool)
        self.tables = {}
        self.ctx = {}

    # -- addressing (cache.py:124-140) ----------------------------------------

    def head_slots(self, seq: int, layer: int, head: int) -> np.ndarray:
        blocks = np.asarray(self.tables[seq][layer][head], dtype=np.int64)
        return (blocks[:, None] * self.block_size + np.arange(self.block_size)).reshape(-1)

    def live_slots(self, seq: int, layer: int, head: int) -> np.ndarray:
        return self.head_slots(seq, layer, head)[: int(self.ctx[seq][layer, head])]

    def head_order(self):
        """Layer-major head enumeration; defines head_idx (cache.py:109-112)."""
        return [(m, h) for m in range(self.num_layers) for h in range(self.num_kv_heads)]

    @property
    def free_count(self) -> int:
        return int(self.free.sum())

    def block_count(self, seq: int) -> int:
        return sum(len(t) for row in self.tables[seq] for t in row)

    def fragmentation(self) -> int:
        """Sum over heads of ceil(C/b)*b - C (cache.py:187-198)."""
        b = self.block_size
        return int(sum(((-(-c // b)) * b - c).sum() for c in self.ctx.values()))


# ---------------------------------------------------------------------------
# Allocation (block_manager.py)
# ---------------------------------------------------------------------------


def blocks_needed_prefill(tokens: int, layers: int, heads: int, b: int) -> int:
    """l*H*ceil(L/b) (block_manager.py:19-25)."""
    if tokens < 1:
        raise ValueError("token_count must be >= 1")
    return layers * heads * ((tokens + b - 1) // b)


def _take_smallest(st: OracleState, n: int) -> np.ndarray:
    ids = np.flatnonzero(st.free)[:n]
    st.free[ids] = False
    return ids


def alloc_prefill(st: OracleState, seq: int, tokens: int) -> int:
    """All-or-nothing prefill: per head ceil(L/b) ids, heads in layer-major
    order, each head a consecutive run of the smallest free ids
    (block_manager.py:56-72)."""
    if seq in st.tables:
        raise ValueError(f"sequence {seq} already allocated")
    per_head = -(-tokens // st.block_size)
    demand = per_head * st.num_layers * st.num_kv_heads
    if demand > st.free_count:
        raise OraclePreemption(demand - st.free_count)
    st.tables[seq] = [[[] for _ in range(st.num_kv_heads)] for _ in range(st.num_layers)]
    st.ctx[seq] = np.zeros((st.num_layers, st.num_kv_heads), dtype=np.int64)
    ids = _take_smallest(st, demand)
    for i, (m, h) in enumerate(st.head_order()):
        st.tables[seq][m][h].extend(int(x) for x in ids[i * per_head : (i + 1) * per_head])
    return demand


def alloc_decode(st: OracleState, seq_ids) -> dict:
    """One block per head whose C is a multiple of b; requests served in
    sorted(seq), (layer, head) order; all-or-nothing (block_manager.py:74-97)."""
    b = st.block_size
    needs = {}
    for s in seq_ids:
        needs[s] = [(m, h) for (m, h) in st.head_order() if st.ctx[s][m, h] % b == 0]
    demand = sum(len(v) for v in needs.values())
    if demand > st.free_count:
        raise OraclePreemption(demand - st.free_count)
    ids = iter(_take_smallest(st, demand))
    for s in sorted(needs):
        for m, h in needs[s]:
            st.tables[s][m][h].append(int(next(ids)))
    return {s: len(v) for s, v in needs.items()}


def free_blocks(st: OracleState, blocks) -> None:
    """Trailing-slice frees with ctx clamp (block_manager.py:101-129)."""
    owner = {}
    for s, rows in st.tables.items():
        for m, row in enumerate(rows):
            for h, tab in enumerate(row):
                for blk in tab:
                    owner[blk] = (s, m, h)
    by_head = {}
    for blk in blocks:
        if blk not in owner:
            raise OracleError("BlockOwnershipError", f"block {blk} is not allocated")
        by_head.setdefault(owner[blk], set()).add(blk)
    for (s, m, h), freed in by_head.items():
        tab = st.tables[s][m][h]
        keep = len(tab) - len(freed)
        if set(tab[keep:]) != freed:
            raise OracleError("BlockOwnershipError", "not a trailing slice")
        del tab[keep:]
        st.ctx[s][m, h] = min(st.ctx[s][m, h], keep * st.block_size)
        st.free[list(freed)] = True


def clear_blocks(st: OracleState, blocks) -> None:
    """Reset freed slots to the empty state (metrics.py:177-183)."""
    b = st.block_size
    for blk in blocks:
        sl = slice(blk * b, (blk + 1) * b)
        st.metric[sl] = 0.0
        st.logical[sl] = -1
        st.protected[sl] = False
        st.fresh[sl] = False


def free_sequence(st: OracleState, seq: int) -> list:
    freed = [blk for row in st.tables[seq] for tab in row for blk in tab]
    free_blocks(st, freed)
    del st.tables[seq]
    del st.ctx[seq]
    return freed


# ---------------------------------------------------------------------------
# Append / decode attention / metric accumulation
# ---------------------------------------------------------------------------


def append(st: OracleState, seq, layer, head, key, value, fresh=True) -> int:
    """Write at position C, C += 1, slot gets metric 0 / logical C / fresh
    (cache.py:163-184 + metrics.py:153-158 as driven by engine.py:427-438)."""
    c = int(st.ctx[seq][layer, head])
    tab = st.tables[seq][layer][head]
    u, o = divmod(c, st.block_size)
    if u >= len(tab):
        raise OracleError("AllocationOrderError", f"no block for position {c}")
    f = tab[u] * st.block_size + o
    st.keys[f] = key
    st.values[f] = value
    st.metric[f] = 0.0
    st.logical[f] = c
    st.protected[f] = False
    st.fresh[f] = fresh
    st.ctx[seq][layer, head] = c + 1
    return f


def paged_decode(st: OracleState, query: np.ndarray, seq: int, layer: int):
    """Single-query GQA decode over the live slots in table order.

    query (n_q, d); query head q reads KV head q // r.  Returns
    (out (n_q, d), rows: list of (r, C_h)) (attention.py:92-127).
    """
    n_q, d = query.shape
    r = n_q // st.num_kv_heads
    if not np.isfinite(query).all():
        raise OracleError("NumericError", "non-finite query")
    out = np.empty((n_q, d))
    rows = []
    for h in range(st.num_kv_heads):
        if st.ctx[seq][layer, h] < 1:
            raise OracleError("EmptyContextError", f"head {h} has no live KVs")
        f = st.live_slots(seq, layer, h)
        qg = query[h * r : (h + 1) * r]
        s = qg @ st.keys[f].T / math.sqrt(d)
        p = np.exp(s - s.max(axis=1, keepdims=True))
        p /= p.sum(axis=1, keepdims=True)
        out[h * r : (h + 1) * r] = p @ st.values[f]
        rows.append(p)
    return out, rows


def agg(x: np.ndarray, aggregation: str) -> np.ndarray:
    """f(x) = x (L1) or x^2 (L2) (metrics.py:46-47)."""
    return x * x if aggregation == "L2" else x


def accumulate(st: OracleState, seq, layer, rows, aggregation="L2") -> None:
    """metric[slot_j] += sum over the group of f(p_hj) (metrics.py:189-211)."""
    for h, p in enumerate(rows):
        f = st.live_slots(seq, layer, h)
        if p.shape[-1] != f.size:
            raise ValueError("row length does not match the live KV count")
        st.metric[f] += agg(p, aggregation).sum(axis=0)


def decode_step_layer(st, seq, layer, q, k_new, v_new, aggregation="L2"):
    """Engine decode for one (seq, layer): append all heads, attend, fold
    the rows into the metrics (engine.py:426-444)."""
    for h in range(st.num_kv_heads):
        append(st, seq, layer, h, k_new[h], v_new[h], fresh=True)
    out, rows = paged_decode(st, q, seq, layer)
    accumulate(st, seq, layer, rows, aggregation)
    return out, rows


def clear_fresh(st: OracleState) -> None:
    st.fresh[:] = False


# ---------------------------------------------------------------------------
# Prefill metrics (window-rows-only restatement)
# ---------------------------------------------------------------------------


def pool_max(x: np.ndarray, pool: int) -> np.ndarray:
    """Centred max-pool of odd width, truncated at the edges (metrics.py:57-65)."""
    half = pool // 2
    n = x.shape[-1]
    out = x.copy()
    for off in range(1, half + 1):
        if off >= n:
            break
        out[..., off:] = np.maximum(out[..., off:], x[..., :-off])
        out[..., :-off] = np.maximum(out[..., :-off], x[..., off:])
    return out


def window_metric(q_win, k, num_kv_heads, window=8, pool=7, aggregation="L2",
                  protect_window=True):
    """Observation-window metric of one layer from the last w query rows.

    q_win: (n_q, w', d) the last w' = min(w, L) prompt queries; k: (H, L, d).
    Row i of the window is prompt position start+i and sees keys 0..start+i
    (causal softmax of gqa_attention, attention.py:62-89).  Returns
    (metrics (H, L), protected (L,)) like window_metrics (metrics.py:68-89).
    """
    n_q, wq, d = q_win.shape
    H, L, _ = k.shape
    r = n_q // num_kv_heads
    start = max(L - window, 0)
    assert wq == L - start
    raw = np.zeros((H, L))
    for h in range(H):
        s = q_win[h * r : (h + 1) * r] @ k[h].T / math.sqrt(d)  # (r, w', L)
        causal = np.arange(L)[None, :] <= (start + np.arange(wq))[:, None]
        s = np.where(causal[None], s, -np.inf)
        p = np.exp(s - s.max(axis=2, keepdims=True))
        p /= p.sum(axis=2, keepdims=True)
        raw[h] = agg(p, aggregation).sum(axis=(0, 1))
    protected = np.arange(L) >= start
    if not protect_window:
        protected[:] = False
    return pool_max(raw, pool), protected


def full_metric(q, k, num_kv_heads, excluded=10, aggregation="L2"):
    """Full-range metric: key j aggregates queries i >= j + v (metrics.py:92-109)."""
    n_q, L, d = q.shape
    r = n_q // num_kv_heads
    out = np.zeros((num_kv_heads, L))
    # query rows in blocks (each row's causal softmax is independent), so the
    # (r, rows, L) tensors stay small at long prompts; same arithmetic
    rb = max(1, min(L, (1 << 22) // max(1, r * L)))
    cols = np.arange(L)[None, :]
    for h in range(num_kv_heads):
        for i0 in range(0, L, rb):
            rows = np.arange(i0, min(L, i0 + rb))[:, None]
            s = q[h * r : (h + 1) * r, i0 : i0 + rb] @ k[h].T / math.sqrt(d)
            s = np.where((cols <= rows)[None], s, -np.inf)
            p = np.exp(s - s.max(axis=2, keepdims=True))
            p /= p.sum(axis=2, keepdims=True)
            c = agg(p, aggregation).sum(axis=0)  # (rows, L_k)
            out[h] += np.where(rows >= cols + excluded, c, 0.0).sum(axis=0)
    return out


def write_prompt(st: OracleState, seq, layer, metrics, protected) -> None:
    """Install prefill metrics for all heads of a layer (metrics.py:160-175)."""
    for h in range(st.num_kv_heads):
        f = st.live_slots(seq, layer, h)
        c = f.size
        st.metric[f] = metrics[h, :c]
        st.logical[f] = np.arange(c)
        st.protected[f] = protected[:c]
        st.fresh[f] = False


def prefill(st: OracleState, seq, q, k, v, window=8, pool=7, aggregation="L2",
            protect_window=True, mode="window", excluded=10):
    """Engine prefill (engine.py:335-353): allocate, scatter K/V, metric."""
    L = k.shape[2]
    alloc_prefill(st, seq, L)
    for m in range(st.num_layers):
        for h in range(st.num_kv_heads):
            st.ctx[seq][m, h] = L
            f = st.live_slots(seq, m, h)
            st.keys[f] = k[m, h]
            st.values[f] = v[m, h]
        if mode == "window":
            start = max(L - window, 0)
            met, prot = window_metric(q[m][:, start:], k[m], st.num_kv_heads, window,
                                      pool, aggregation, protect_window)
        else:
            met = full_metric(q[m], k[m], st.num_kv_heads, excluded, aggregation)
            prot = np.zeros(L, dtype=bool)
        write_prompt(st, seq, m, met, prot)


# ---------------------------------------------------------------------------
# Eviction scheduling and compaction (compression.py)
# ---------------------------------------------------------------------------


@dataclass
class HeadPlan:
    layer: int
    head: int
    blocks: list
    slots: np.ndarray
    ctx: int
    occupied: np.ndarray
    key: np.ndarray  # effective metric: 0 empty, +inf shielded
    logical: np.ndarray
    cap: int
    perm: np.ndarray = None
    thresholds: np.ndarray = None


def head_plans(st: OracleState, seq: int) -> list:
    """Per-head M1 snapshot with effective metric and cap (compression.py:122-149)."""
    b = st.block_size
    plans = []
    for m, h in st.head_order():
        slots = st.head_slots(seq, m, h)
        c = int(st.ctx[seq][m, h])
        occ = np.arange(slots.size) < c
        shield = (st.protected[slots] | st.fresh[slots]) & occ
        key = np.where(shield, np.inf, np.where(occ, st.metric[slots], 0.0))
        nb = len(st.tables[seq][m][h])
        cap = max(0, nb - max(1, -(-int(shield.sum()) // b)))
        plans.append(HeadPlan(m, h, list(st.tables[seq][m][h]), slots, c, occ, key,
                              st.logical[slots].copy(), cap))
    return plans


def sort_head(plan: HeadPlan) -> np.ndarray:
    """Stable order by (key, occupied, logical-or--1, position)
    (compression.py:156-166), via one argsort over a structured record."""
    rec = np.zeros(plan.slots.size, dtype=[("k", "f8"), ("o", "i1"), ("l", "i8"), ("p", "i8")])
    rec["k"] = plan.key
    rec["o"] = plan.occupied
    rec["l"] = np.where(plan.occupied, plan.logical, -1)
    rec["p"] = np.arange(plan.slots.size)
    return np.argsort(rec, order=("k", "o", "l", "p"), kind="stable")


def thresholds_of(plan: HeadPlan, b: int) -> np.ndarray:
    """th[e-1] = (b*e)-th smallest effective metric (compression.py:169-177)."""
    return plan.key[plan.perm][b - 1 :: b]


def select_rows(plans: list, budget: int) -> list:
    """Take the first `budget` eligible rows in (threshold, head_idx, row)
    order; rows at or beyond a head's cap are skipped (compression.py:180-231).
    Returns per-head evicted block counts."""
    total_cap = sum(p.cap for p in plans)
    if budget > total_cap:
        raise OracleError("BudgetError", f"budget {budget} exceeds {total_cap}")
    cand = [
        (float(th), hi, ri)
        for hi, p in enumerate(plans)
        for ri, th in enumerate(p.thresholds)
        if ri < p.cap
    ]
    cand.sort()
    counts = [0] * len(plans)
    for _, hi, _ in cand[:budget]:
        counts[hi] += 1
    return counts


def compact_head(st: OracleState, plan: HeadPlan, evict: int, mask=None) -> list:
    """Two-cursor MoveCache walk for one head (compression.py:234-280).

    Holes are marked or empty slots.  Survivors inside the last evict*b
    slots move, scanning the range downward, into the lowest remaining hole
    below it; K, V, metric, logical and both flags travel together.
    """
    b = st.block_size
    n = plan.slots.size
    span = evict * b
    if span == 0:
        return []
    if span > n:
        raise OracleError("ScheduleCorruptionError", "eviction range exceeds the head")
    if mask is None:
        mask = np.zeros(n, dtype=bool)
        mask[plan.perm[:span]] = True
    hole = mask | (st.logical[plan.slots] < 0)
    end = n - span
    dsts = [i for i in range(end) if hole[i]]
    srcs = [j for j in range(n - 1, end - 1, -1) if not hole[j]]
    if len(srcs) > len(dsts):
        raise OracleError("ScheduleCorruptionError", "no hole left outside the range")
    moves = []
    for j, i in zip(srcs, dsts):
        src, dst = int(plan.slots[j]), int(plan.slots[i])
        for arr in (st.keys, st.values, st.metric, st.logical, st.protected, st.fresh):
            arr[dst] = arr[src]
        moves.append((src, dst))
    return moves


def compress(st: OracleState, budgets: dict) -> dict:
    """Full round (compression.py:312-355) -> the CompressionSchedule.to_dict
    payload (compression.py:95-119), plus per-head counts for all heads."""
    b = st.block_size
    out = {"freed_blocks": 0, "evicted_kvs": 0, "sequences": []}
    for seq, requested in budgets.items():
        plans = head_plans(st, seq)
        budget = min(requested, sum(p.cap for p in plans))
        srec = {"seq_id": seq, "requested_budget": requested, "budget": budget, "heads": []}
        out["sequences"].append(srec)
        if budget <= 0:
            continue
        for p in plans:
            p.perm = sort_head(p)
            p.thresholds = thresholds_of(p, b)
        counts = select_rows(plans, budget)
        for p, e in zip(plans, counts):
            if e == 0:
                continue
            mask = np.zeros(p.slots.size, dtype=bool)
            mask[p.perm[: e * b]] = True
            moves = compact_head(st, p, e)
            freed = p.blocks[len(p.blocks) - e :]
            srec["heads"].append({
                "layer": p.layer, "head": p.head, "evicted_blocks": e,
                "evicted_kvs": int((mask & p.occupied).sum()),
                "freed": [int(x) for x in freed],
                "moves": [[s, d] for s, d in moves],
            })
        # free + renumber (compression.py:283-309)
        for hrec in srec["heads"]:
            m, h = hrec["layer"], hrec["head"]
            free_blocks(st, hrec["freed"])
            clear_blocks(st, hrec["freed"])
            f = st.live_slots(seq, m, h)
            order = np.argsort(st.logical[f], kind="stable")
            ranks = np.empty(f.size, dtype=np.int64)
            ranks[order] = np.arange(f.size)
            st.logical[f] = ranks
            out["freed_blocks"] += len(hrec["freed"])
            out["evicted_kvs"] += hrec["evicted_kvs"]
    return out


def evict_counts(st: OracleState, seq: int, budget: int):
    """(clamped budget, per-head evicted blocks in head_idx order) without
    mutating anything: the schedule_evictions half of ``compress``."""
    plans = head_plans(st, seq)
    budget = min(budget, sum(p.cap for p in plans))
    if budget <= 0:
        return budget, [0] * len(plans), plans
    for p in plans:
        p.perm = sort_head(p)
        p.thresholds = thresholds_of(p, st.block_size)
    return budget, select_rows(plans, budget), plans


# ---------------------------------------------------------------------------
# Budgets (engine.py:96-129)
# ---------------------------------------------------------------------------


def per_sequence_budget(prompt_len, rate, floor_tokens=128, mode="min") -> int:
    if rate < 1:
        raise ValueError("rate must be >= 1")
    if rate == 1:
        return prompt_len
    pick = min if mode == "min" else max
    return int(math.floor(pick(float(floor_tokens), prompt_len / rate)))


def budget_to_blocks(budget_tokens, layers, heads, b, allocated_blocks) -> int:
    target = budget_tokens * layers * heads
    return max(0, allocated_blocks - (-(-target // b)))
