"""Loader for the golden JSON fixtures written by tests/golden/make_golden.py."""

from __future__ import annotations

import base64
import functools
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def dec(rec):
    """Inverse of make_golden.enc."""
    raw = base64.b64decode(rec["b64"])
    return np.frombuffer(raw, dtype=np.dtype(rec["dtype"])).reshape(rec["shape"]).copy()


@functools.lru_cache(maxsize=None)
def load(name: str):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def slot_index(blocks, block_size):
    """Flat slot ids covered by a snapshot's `blocks` list, in snapshot order."""
    return (np.asarray(blocks, dtype=np.int64)[:, None] * block_size
            + np.arange(block_size)).reshape(-1)
