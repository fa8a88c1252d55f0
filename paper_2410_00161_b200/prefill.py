"""Prefill write path + observation-window metric (K2) -- under construction."""


def window_metrics(*a, **k):
    raise NotImplementedError


def prefill_sequence(*a, **k):
    raise NotImplementedError
