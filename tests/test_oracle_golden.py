"""Pin the CPU oracle before trusting it (CPU-only).

(a) The reference test suite's known-answer tests, re-expressed on the
    oracle (pkg/tests/test_compression.py, test_block_manager.py,
    test_metrics.py, test_engine.py, test_cache.py).
(b) Golden vectors produced by the reference itself
    (tests/golden/make_golden.py): compression rounds, decode attention,
    window/full metrics and allocator traces must match exactly (integers)
    or to 1e-12 (float64).
"""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import dec, load, slot_index
from oracle import kvc_oracle as O
from oracle_rig import check_state, state_from_snapshot

FIG_HEAD0 = [0.1, 0.2, 0.3, 0.4, 0.9]  # tests/test_compression.py:42
FIG_HEAD1 = [0.5, 0.6]  # tests/test_compression.py:43


def one_seq_state(metric_lists, b=2, protected=None, layers=1, d=4, rng=None):
    """One sequence, one layer, one head per metric list (test_compression.py:23-36)."""
    heads = len(metric_lists) // layers
    st = O.OracleState(256, b, d, layers, heads)
    st.tables[0] = [[[] for _ in range(heads)] for _ in range(layers)]
    st.ctx[0] = np.zeros((layers, heads), dtype=np.int64)
    rng = rng or np.random.default_rng(0)
    for i, metrics in enumerate(metric_lists):
        m, h = divmod(i, heads)
        nb = -(-len(metrics) // b)
        st.tables[0][m][h].extend(int(x) for x in O._take_smallest(st, nb))
        for j, val in enumerate(metrics):
            f = O.append(st, 0, m, h, rng.standard_normal(d), rng.standard_normal(d), fresh=False)
            st.metric[f] = val
            if protected is not None and protected[i][j]:
                st.protected[f] = True
    return st


def plans_of(st, b=2):
    plans = O.head_plans(st, 0)
    for p in plans:
        p.perm = O.sort_head(p)
        p.thresholds = O.thresholds_of(p, b)
    return plans


class TestKnownAnswers:
    def test_thresholds_hand_example(self):  # test_compression.py:76-81
        p = plans_of(one_seq_state([[0.3, 0.1, 0.5, 0.2, 0.4]]))[0]
        assert np.allclose(p.thresholds, [0.1, 0.3, 0.5])
        assert not p.occupied[p.perm[0]]  # empty slot first (:52-56)

    def test_ties_by_logical(self):  # :64-68
        p = plans_of(one_seq_state([[0.5] * 4]))[0]
        assert p.logical[p.perm].tolist() == [0, 1, 2, 3]

    def test_candidate_order(self):  # :127-141
        plans = plans_of(one_seq_state([FIG_HEAD0, FIG_HEAD1]))
        cand = sorted((th, hi, ri) for hi, p in enumerate(plans) for ri, th in enumerate(p.thresholds))
        assert [(h, r) for _, h, r in cand][:3] == [(0, 0), (0, 1), (1, 0)]

    def test_budget_two(self):  # :161-169
        plans = plans_of(one_seq_state([FIG_HEAD0, FIG_HEAD1]))
        assert O.select_rows(plans, 2) == [2, 0]
        assert O.select_rows(plans, 0) == [0, 0]

    def test_lone_block_never_marked(self):  # :171-175
        plans = plans_of(one_seq_state([[0.9] * 6, [0.0, 0.0]]))
        assert O.select_rows(plans, 2) == [2, 0]

    def test_budget_error(self):  # :177-185
        plans = plans_of(one_seq_state([FIG_HEAD0, FIG_HEAD1]))
        assert sum(p.cap for p in plans) == 2
        with pytest.raises(O.OracleError) as exc:
            O.select_rows(plans, 3)
        assert exc.value.kind == "BudgetError"

    def test_hand_traced_move(self):  # :212-223
        st = one_seq_state([[0.5, 0.1, 0.6, 0.2, 0.7]])
        p = O.head_plans(st, 0)[0]
        # mask positions 1 and 3 (metrics 0.1, 0.2) plus nothing else
        mask = np.array([False, True, False, True, False, False])
        moves = O.compact_head(st, p, 1, mask=mask)
        assert moves == [(int(p.slots[4]), int(p.slots[1]))]
        assert st.metric[p.slots[1]] == 0.7 and st.logical[p.slots[1]] == 4

    def test_move_without_holes_raises(self):  # :225-230
        st = one_seq_state([[0.5, 0.1, 0.6, 0.2, 0.7, 0.8]])
        p = O.head_plans(st, 0)[0]
        with pytest.raises(O.OracleError) as exc:
            O.compact_head(st, p, 1, mask=np.zeros(6, dtype=bool))
        assert exc.value.kind == "ScheduleCorruptionError"

    def test_end_state(self):  # :251-261
        st = one_seq_state([FIG_HEAD0, FIG_HEAD1])
        sched = O.compress(st, {0: 2})
        assert sched["freed_blocks"] == 2
        assert st.ctx[0].tolist() == [[2, 2]]
        assert len(st.tables[0][0][0]) == 1
        f = st.live_slots(0, 0, 0)
        order = np.argsort(st.logical[f])
        assert [round(x, 3) for x in st.metric[f][order]] == [0.4, 0.9]
        assert sorted(st.logical[f].tolist()) == [0, 1]

    def test_budget_clamp(self):  # :263-266
        st = one_seq_state([FIG_HEAD0, FIG_HEAD1])
        sched = O.compress(st, {0: 99})
        assert sched["sequences"][0]["budget"] == 2 and sched["freed_blocks"] == 2

    def test_protected_and_fresh_survive(self):  # :319-335
        metrics = [0.01, 0.02, 0.03, 0.04, 0.9, 0.8, 0.7, 0.6, 0.5, 0.4]
        st = one_seq_state([metrics], protected=[[True] * 4 + [False] * 6])
        O.compress(st, {0: 99})
        assert {0.01, 0.02, 0.03, 0.04} <= set(st.metric[st.live_slots(0, 0, 0)].tolist())
        st = one_seq_state([[0.9, 0.8, 0.7, 0.6]])
        f = st.head_slots(0, 0, 0)
        st.fresh[f[2]] = st.fresh[f[3]] = True
        O.compress(st, {0: 99})
        assert {0.7, 0.6} <= set(st.metric[st.live_slots(0, 0, 0)].tolist())

    def test_block_and_budget_arithmetic(self):
        assert O.blocks_needed_prefill(100, 32, 8, 16) == 1792  # test_block_manager.py:33-34
        assert O.per_sequence_budget(6000, 64) == 93  # test_engine.py:27-35
        assert O.per_sequence_budget(256, 2) == 128
        assert O.per_sequence_budget(64, 8, mode="max") == 128
        assert O.per_sequence_budget(6000, 8, mode="max") == 750
        assert O.budget_to_blocks(2, 2, 2, 2, 8) == 4  # test_engine.py:46-65
        assert O.budget_to_blocks(100, 2, 2, 2, 8) == 0

    def test_pooling_edges(self):  # test_metrics.py:62-68
        x = np.array([[0.4, 0.1, 0.2, 0.3]])
        assert np.allclose(O.pool_max(x, 3), [[0.4, 0.4, 0.3, 0.3]])

    def test_single_token_metric(self):  # test_metrics.py:29-35
        for agg in ("L1", "L2"):
            m, prot = O.window_metric(np.ones((1, 1, 4)), np.ones((1, 1, 4)), 1, 8, 7, agg)
            assert m[0, 0] == 1.0 and prot[0]

    def test_fragmentation_hand(self):  # test_cache.py:115-122
        st = O.OracleState(64, 4, 4, 2, 2)
        O.alloc_prefill(st, 0, 5)
        st.ctx[0][:] = 5
        assert st.fragmentation() == 12

    def test_allocation_kats(self):  # test_block_manager.py:62-68, 159-165
        st = O.OracleState(3, 4, 4, 2, 2)
        with pytest.raises(O.OraclePreemption) as exc:
            O.alloc_prefill(st, 0, 1)
        assert exc.value.shortfall == 1 and st.free_count == 3
        st = O.OracleState(4, 4, 4, 1, 1)
        O.alloc_prefill(st, 0, 16)
        freed = O.free_sequence(st, 0)
        O.alloc_prefill(st, 1, 1)
        assert st.tables[1][0][0][0] == min(freed)


# ---------------------------------------------------------------------------
# Golden vectors from the reference itself
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("i", range(len(load("compress_cases.json"))))
def test_compress_golden(i):
    case = load("compress_cases.json")[i]
    st = state_from_snapshot(case["before"], case["num_blocks"], case["block_size"],
                             case["head_dim"], case["layers"], case["heads"])
    sched = O.compress(st, {int(s): int(e) for s, e in case["budgets"]})
    assert sched == case["schedule"]
    check_state(st, case["after"], case["block_size"])


@pytest.mark.parametrize("i", range(len(load("decode_cases.json"))))
def test_decode_golden(i):
    case = load("decode_cases.json")[i]
    st = state_from_snapshot(case["before"], case["num_blocks"], case["block_size"],
                             case["head_dim"], case["layers"], case["heads"])
    out, rows = O.paged_decode(st, dec(case["query"]), case["seq"], case["layer"])
    assert np.abs(out - dec(case["out"])).max() <= 1e-12
    for row, ref in zip(rows, case["rows"]):
        assert np.abs(row - dec(ref)).max() <= 1e-12
    O.accumulate(st, case["seq"], case["layer"], rows, case["aggregation"])
    idx = slot_index(case["before"]["blocks"], case["block_size"])
    assert np.abs(st.metric[idx] - dec(case["metric_after"])).max() <= 1e-12


@pytest.mark.parametrize("i", range(len(load("metric_cases.json"))))
def test_metric_golden(i):
    case = load("metric_cases.json")[i]
    q, k = dec(case["q"]), dec(case["k"])
    L = case["L"]
    start = max(L - case["window"], 0)
    wm, prot = O.window_metric(q[:, start:], k, case["heads"], case["window"], case["pool"],
                               case["aggregation"])
    assert np.abs(wm - dec(case["window_metrics"])).max() <= 1e-12
    assert prot.astype(int).tolist() == case["protected"]
    fm = O.full_metric(q, k, case["heads"], case["excluded"], case["aggregation"])
    assert np.abs(fm - dec(case["full_metrics"])).max() <= 1e-12


@pytest.mark.parametrize("i", range(len(load("alloc_cases.json"))))
def test_alloc_golden(i):
    case = load("alloc_cases.json")[i]
    st = O.OracleState(case["num_blocks"], case["block_size"], 1, case["layers"], case["heads"])
    for op in case["ops"]:
        if op["op"] == "prefill":
            try:
                O.alloc_prefill(st, op["seq"], op["tokens"])
                st.ctx[op["seq"]][:] = op["tokens"]
                assert op["ok"]
            except O.OraclePreemption as exc:
                assert not op["ok"] and exc.shortfall == op["shortfall"]
        elif op["op"] == "decode":
            try:
                counts = O.alloc_decode(st, op["seqs"])
                for s in op["seqs"]:
                    st.ctx[s] += 1
                assert op["ok"] and [[k, v] for k, v in counts.items()] == op["counts"]
            except O.OraclePreemption as exc:
                assert not op["ok"] and exc.shortfall == op["shortfall"]
        else:
            assert O.free_sequence(st, op["seq"]) == op["freed"]
        assert {str(s): rows for s, rows in st.tables.items()} == op["tables"]
        assert st.free_count == op["free_count"]
