"""B200-native KV-Compress hot path: variable-head-rate paged KV on sm_100a.

Drop-in for the reference ``pagedkv`` package's hot path (cache config,
block allocator, per-head block tables, metric update, eviction scheduling,
cache moves, paged decode attention); see DESIGN.md.  The compute runs in
libkvc.so (hand-written CUDA, C ABI in include/kvc.h); there is no CPU
fallback.
"""

from .attention import AttentionConfig, dense_attention, gqa_attention, paged_attention, paged_decode
from .block_manager import BlockManager, blocks_needed_prefill
from .budget import budget_to_blocks, per_sequence_budget
from .cache import (
    BlockTables,
    SlotHandle,
    UnifiedKVCache,
    append_kv,
    fragmentation,
    lookup_kv,
)
from .compression import (
    CompressionSchedule,
    EvictionPlan,
    compress,
    execute_cache_moves,
    schedule_evictions,
)
from .metrics import MetricConfig, MetricsStore, accumulate_decode, full_metrics, prompt_metrics, window_metrics
from .engine import (POLICY_PRESETS, CompressionPolicy, Engine, SequenceState, StepRecord, preempt_select,
                     select_compression_batch)
from .graph import DecodeStepGraph
from .prefill import full_metrics_qk, prefill_compress_sequence, prefill_sequence, window_metrics_qk
from .sharding import ShardedEngine, gather_counts, gather_round_counts, owner_of, shard_sequences

__version__ = "0.1.0"

__all__ = [
    "AttentionConfig",
    "dense_attention",
    "gqa_attention",
    "preempt_select",
    "SequenceState",
    "BlockManager",
    "BlockTables",
    "CompressionSchedule",
    "EvictionPlan",
    "MetricConfig",
    "MetricsStore",
    "SlotHandle",
    "UnifiedKVCache",
    "accumulate_decode",
    "append_kv",
    "blocks_needed_prefill",
    "budget_to_blocks",
    "compress",
    "execute_cache_moves",
    "fragmentation",
    "lookup_kv",
    "paged_attention",
    "paged_decode",
    "DecodeStepGraph",
    "Engine",
    "CompressionPolicy",
    "POLICY_PRESETS",
    "StepRecord",
    "select_compression_batch",
    "per_sequence_budget",
    "prefill_compress_sequence",
    "prefill_sequence",
    "full_metrics",
    "schedule_evictions",
    "window_metrics",
    "window_metrics_qk",
    "full_metrics_qk",
    "prompt_metrics",
    "ShardedEngine",
    "gather_counts",
    "gather_round_counts",
    "owner_of",
    "shard_sequences",
]
