"""Planner split mode (an extension of the reference's
binary choice, migration.py:155-169).  Off by default: then plan_hybrid is the
reference's bit for bit (the golden fixtures).  On: a single-request move whose
KV does not fit the link budget may be split into a KV prefix (link budget)
and a re-prefilled suffix (destination compute budget), with s chosen from the
reference's own linear cost terms."""
import random

import pytest
from hypothesis import given, settings, strategies as st

from paper_2501_06709_b200.planner import (DEFERRED, FORCED_KV_TRANSFER, KV_TRANSFER, SPLIT_TRANSFER,
                                           TOKEN_TRANSFER, Boundaries, PendingMove, Topology, check_budgets,
                                           load_boundaries, plan_hybrid, split_suffix)
from test_planner import _bounds, _plan_json, _topo


def test_split_off_is_the_reference(golden):
    for c in golden("planner_cases.json"):
        topo, bounds = _topo(c["topology"]), _bounds(c["boundaries"])
        moves = [PendingMove(*m) for m in c["moves"]]
        defer = {k: v for k, v in c["defer_counts"]}
        plan = plan_hybrid(moves, bounds, topo, defer_counts=defer, max_defer=c["max_defer"], split=False)
        assert _plan_json(plan) == c["plan"]
        assert all(p.suffix_tokens == 0 for p in plan.assignments)


def test_balanced_split_point():
    """13B, 8k tokens, 770 GB/s link, re-prefill at the QKV proxy's ~206k tok/s:
    the suffix balances (n - s) * bpt / BW against s / rate, prefix whole blocks."""
    bpt, n, bw, rate = 819_200, 8192, 770e9, 206_000.0
    s = split_suffix(n, n * bpt, bw, rate, link_left=1e30, comp_left=1e30)
    ideal = n * (bpt / bw) / (bpt / bw + 1 / rate)
    assert (n - s) % 16 == 0 and abs(s - ideal) <= 8
    lat_x, lat_c = (n - s) * bpt / bw, s / rate
    assert abs(lat_x - lat_c) / max(lat_x, lat_c) < 0.02


def test_split_respects_both_budgets():
    bpt, n = 524_288, 4096
    # the link fits 1000 tokens' worth of bytes, the destination 3500 tokens
    s = split_suffix(n, n * bpt, 900e9, 50_000.0, link_left=1000 * bpt + 5, comp_left=3500)
    assert n - s <= 1000 and (n - s) % 16 == 0 and s <= 3500
    # neither the link nor the compute budget can take its share: no split
    assert split_suffix(n, n * bpt, 900e9, 50_000.0, link_left=100 * bpt, comp_left=3000) is None
    # bytes per token not exact (a mixed-model group's aggregate): no split
    assert split_suffix(n, n * bpt + 1, 900e9, 50_000.0, link_left=1e30, comp_left=1e30) is None


def test_split_only_when_kv_does_not_fit():
    topo = Topology(gpus_per_machine=8, intra_bandwidth_bytes_per_s=900e9, prefill_tokens_per_s=200_000.0)
    bounds = load_boundaries(topo, 0.05, 0.2)   # 9e9 B link, 2000 tokens compute per epoch
    bpt = 524_288
    fits = [PendingMove(1, 0, 1, 1024 * bpt, 1024), PendingMove(2, 0, 2, 12288 * bpt, 12288)]  # 7.0 GB together
    assert _plan_json(plan_hybrid(fits, bounds, topo, split=True)) == _plan_json(plan_hybrid(fits, bounds, topo))
    # consensus order puts the 9.4 GB move first: it cannot fit, so it is split and its prefix
    # takes link budget the smaller moves would otherwise have used
    huge = PendingMove(3, 0, 3, 18000 * bpt, 18000)    # 9.4 GB > 9e9
    plan = plan_hybrid(fits + [huge], bounds, topo, split=True)
    assert plan.assignments[0].move.item == 3 and plan.assignments[0].mode == SPLIT_TRANSFER
    assert check_budgets(plan, bounds) == []


def test_split_wins_over_deferral_and_charges_both_ledgers():
    topo = Topology(gpus_per_machine=8, intra_bandwidth_bytes_per_s=900e9, prefill_tokens_per_s=200_000.0)
    bpt, n = 819_200, 8192
    bounds = Boundaries(comm_budget={}, comp_budget=2000.0, intra_comm_budget=0.8 * n * bpt,
                        inter_comm_budget=1e9)
    mv = PendingMove(7, 0, 1, n * bpt, n)
    ref = plan_hybrid([mv], bounds, topo)
    assert ref.assignments[0].mode == DEFERRED            # the reference waits
    plan = plan_hybrid([mv], bounds, topo, split=True)
    p = plan.assignments[0]
    assert p.mode == SPLIT_TRANSFER and 0 < p.suffix_tokens <= 2000 and (n - p.suffix_tokens) % 16 == 0
    assert plan.link_bytes[("intra", 0)] == (n - p.suffix_tokens) * bpt
    assert plan.dest_tokens[1] == p.suffix_tokens
    assert p.latency_s == max((n - p.suffix_tokens) * bpt / 900e9, p.suffix_tokens / 200_000.0)
    assert plan.executed == [p] and check_budgets(plan, bounds) == []


def test_groups_keep_the_binary_choice():
    topo = Topology(gpus_per_machine=8, intra_bandwidth_bytes_per_s=900e9, prefill_tokens_per_s=200_000.0)
    bounds = Boundaries(comm_budget={}, comp_budget=2000.0, intra_comm_budget=1e9, inter_comm_budget=1e9)
    plan = plan_hybrid([PendingMove(-3, 0, 1, 8192 * 819_200, 8192)], bounds, topo, split=True)
    assert plan.assignments[0].mode == DEFERRED


@settings(max_examples=300, deadline=None)
@given(st.lists(st.tuples(st.integers(-10, 40), st.integers(0, 15), st.integers(0, 15),
                          st.integers(1, 20000), st.sampled_from([100, 524_288, 819_200, 327_680])),
                max_size=25, unique_by=lambda t: t[0]),
       st.floats(1e6, 3e10), st.floats(0, 5e4), st.integers(0, 4))
def test_split_plans_never_exceed_budgets(specs, comm, comp, max_defer):
    topo = Topology(gpus_per_machine=8, intra_bandwidth_bytes_per_s=900e9, prefill_tokens_per_s=100_000.0)
    bounds = Boundaries(comm_budget={}, comp_budget=comp, intra_comm_budget=comm, inter_comm_budget=comm / 10)
    moves = [PendingMove(i, s, d, tok * bpt, tok) for i, s, d, tok, bpt in specs]
    plan = plan_hybrid(moves, bounds, topo, max_defer=max_defer, split=True)
    assert check_budgets(plan, bounds) == []
    ref = plan_hybrid(moves, bounds, topo, max_defer=max_defer)
    assert [p.move.item for p in plan.assignments] == [p.move.item for p in ref.assignments]
    for p, r in zip(plan.assignments, ref.assignments):
        if p.mode == SPLIT_TRANSFER:
            assert p.move.item >= 0 and 0 < p.suffix_tokens < p.move.tokens
            assert (p.move.tokens - p.suffix_tokens) % 16 == 0
        else:
            assert p.suffix_tokens == 0
        if r.mode == KV_TRANSFER and p.mode != KV_TRANSFER:
            # a split earlier in the order may have used the link budget this move had
            assert any(q.mode == SPLIT_TRANSFER for q in plan.assignments)
