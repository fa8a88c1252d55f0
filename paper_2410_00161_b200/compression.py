"""Eviction scheduling (K3) and compaction (K4) -- under construction."""

from __future__ import annotations


class CompressionSchedule:  # placeholder, replaced below
    pass


class EvictionPlan:
    pass


def schedule_evictions(*a, **k):
    raise NotImplementedError


def execute_cache_moves(*a, **k):
    raise NotImplementedError


def compress(*a, **k):
    raise NotImplementedError
