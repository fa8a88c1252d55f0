"""Deterministic synthetic token source shared by the reference engine
(golden generation, make_engine_golden.py) and the device Engine test.

Activations are rounded to bf16 so the device cache stores them exactly;
token i of a request is a pure function of (request key, i)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def bf16_round(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32).astype(np.float64)


@dataclass(frozen=True)
class Tok:
    q: np.ndarray
    k: np.ndarray
    v: np.ndarray


class HashTokens:
    def __init__(self, key: int, prompt_len: int, output_tokens: int, layers: int, n_q: int, n_k: int, d: int):
        self.key, self.prompt_len, self.output_tokens = key, prompt_len, output_tokens
        self.shape = (layers, n_q, n_k, d)

    def token(self, i: int) -> Tok:
        layers, n_q, n_k, d = self.shape
        rng = np.random.default_rng([self.key, i])
        return Tok(bf16_round(rng.standard_normal((layers, n_q, d))),
                   bf16_round(rng.standard_normal((layers, n_k, d))),
                   bf16_round(rng.standard_normal((layers, n_k, d))))


# (name, engine kwargs, requests [(prompt_len, output_tokens)])
SHAPE = dict(layers=2, n_q=8, n_k=4, d=64, block_size=16)
CASES = [
    ("prefill-preempt", dict(policy="prefill-preempt", num_blocks=170, rate=4.0, budget_floor=64),
     [(150, 30), (90, 40), (260, 8), (60, 45), (200, 15), (120, 30), (300, 6), (75, 38)]),
    ("every-step", dict(policy="every-step", num_blocks=400, rate=8.0, budget_floor=8),
     [(120, 10), (220, 14), (64, 20), (180, 9), (99, 16)]),
    ("no-compression-preemption", dict(policy="none", num_blocks=70, rate=1.0, budget_floor=128),
     [(64, 20), (64, 10), (48, 6)]),
    # f4 policy coverage (engine.py:132-156, 282-289, 388-410):
    # every-step rounds truncated by kv_limit (staleness order, stop at the
    # first sequence that would exceed the limit)
    ("kv-limit", dict(policy=dict(on_prefill=True, on_preempt=True, every_c=1, kv_limit=2000), num_blocks=400,
                      rate=8.0, budget_floor=8),
     [(120, 10), (220, 14), (64, 20), (180, 9), (99, 16)]),
    # rounds triggered only by the uncompressed-token threshold
    ("token-threshold", dict(policy=dict(on_prefill=False, on_preempt=False, token_threshold=30), num_blocks=400,
                             rate=8.0, budget_floor=8),
     [(120, 10), (220, 14), (64, 20), (180, 9), (99, 16)]),
    # decode allocation runs dry: compress first, then preempt when that is
    # not enough (same step)
    ("decode-compress-then-preempt", dict(policy="prefill-preempt", num_blocks=52, rate=2.0, budget_floor=16),
     [(40, 25), (45, 20), (50, 30), (35, 25)]),
]

# multi-GPU: request i of a case runs on rank i % SHARD_WORLD (sharding.owner_of)
SHARD_WORLD = 2


def make_policy(mod, spec):
    """Preset name or CompressionPolicy kwargs -> the module's policy object."""
    return mod.POLICY_PRESETS[spec] if isinstance(spec, str) else mod.CompressionPolicy(**spec)


def shard(reqs, rank, world=SHARD_WORLD):
    """(global index, request) pairs rank `rank` owns."""
    return [(i, r) for i, r in enumerate(reqs) if i % world == rank]
