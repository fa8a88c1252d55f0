"""Per-sequence eviction budgets (host integer arithmetic feeding K3).

Same functions and semantics as pkg/src/pagedkv/engine.py:96-129.
"""

from __future__ import annotations

import math


def per_sequence_budget(prompt_len: int, rate: float, floor_tokens: int = 128, mode: str = "min") -> int:
    """Target cache tokens for a sequence compressed at ``rate``.

    Default combines the floor and prompt_len/rate with min(); mode="max"
    selects the floor reading instead.  rate == 1 returns prompt_len so no
    eviction ever triggers (engine.py:96-113).
    """
    if rate < 1:
        raise ValueError("rate must be >= 1")
    if rate == 1:
        return prompt_len
    combine = min if mode == "min" else max
    return int(math.floor(combine(float(floor_tokens), prompt_len / rate)))


def budget_to_blocks(budget_tokens: int, num_layers: int, num_kv_heads: int, block_size: int,
                     allocated_blocks: int) -> int:
    """Blocks to evict so the kept KVs fit the token budget (engine.py:116-129)."""
    target_kvs = budget_tokens * num_layers * num_kv_heads
    return max(0, allocated_blocks - (-(-target_kvs // block_size)))
