"""Build oracle states from golden snapshots (test helper)."""

from __future__ import annotations

import numpy as np

from golden_io import dec, slot_index
from oracle import kvc_oracle as O


def state_from_snapshot(snap, num_blocks, block_size, head_dim, layers, heads):
    st = O.OracleState(num_blocks, block_size, head_dim, layers, heads)
    idx = slot_index(snap["blocks"], block_size)
    st.metric[idx] = dec(snap["metric"])
    st.logical[idx] = dec(snap["logical"])
    st.protected[idx] = np.asarray(snap["protected"], dtype=bool)
    st.fresh[idx] = np.asarray(snap["fresh"], dtype=bool)
    if "keys" in snap:
        st.keys[idx] = dec(snap["keys"])
        st.values[idx] = dec(snap["values"])
    st.free[:] = False
    st.free[snap["free"]] = True
    for s, rows in snap["tables"].items():
        st.tables[int(s)] = [[list(t) for t in row] for row in rows]
        st.ctx[int(s)] = np.asarray(snap["ctx"][s], dtype=np.int64)
    return st


def check_state(st, snap, block_size, kv=True):
    """Assert the oracle state equals a golden snapshot exactly."""
    idx = slot_index(snap["blocks"], block_size)
    assert np.array_equal(st.metric[idx], dec(snap["metric"]))
    assert np.array_equal(st.logical[idx], dec(snap["logical"]))
    assert np.array_equal(st.protected[idx], np.asarray(snap["protected"], dtype=bool))
    assert np.array_equal(st.fresh[idx], np.asarray(snap["fresh"], dtype=bool))
    if kv and "keys" in snap:
        assert np.array_equal(st.keys[idx], dec(snap["keys"]))
        assert np.array_equal(st.values[idx], dec(snap["values"]))
    assert sorted(np.flatnonzero(st.free).tolist()) == snap["free"]
    assert {str(s): rows for s, rows in st.tables.items()} == snap["tables"]
    assert {str(s): c.tolist() for s, c in st.ctx.items()} == snap["ctx"]
