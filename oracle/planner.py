"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain-Python restatement of the reference migration planner
(/root/reference/pkg/src/kvpack/migration.py), used as the checker for the
product planner in paper_2501_06709_b200.migration on boxes where the
reference is not mounted.  Pinned against tests/golden/planner_cases.json and
tests/golden/boundaries.json, which tests/golden/make_golden.py produced by
running the reference itself (parity pinned).

Each function cites the reference lines it restates.  Deliberately naive:
tuples and dicts, no classes beyond what the comparison needs.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

KV, TOKEN, DEFER, FORCED = "kv_transfer", "token_transfer", "deferred", "forced_kv_transfer"


def link_of(gpm: int, src: int, dst: int) -> tuple:
    """migration.py:46-53 — machine = gpu // gpus_per_machine."""
    ms, md = src // gpm, dst // gpm
    return ("intra", ms) if ms == md else ("inter",)


def load_boundaries(intra_bw: float, inter_bw: float, prefill: float,
                    epoch_seconds: float, fraction: float) -> Tuple[float, float, float]:
    """migration.py:77-91 — (comp, intra_comm, inter_comm), left-to-right float64."""
    if epoch_seconds <= 0 or not 0.0 < fraction <= 1.0:
        raise ValueError("bad epoch/fraction")
    return (prefill * epoch_seconds * fraction,
            intra_bw * epoch_seconds * fraction,
            inter_bw * epoch_seconds * fraction)


def consensus_order(moves: Sequence[tuple]) -> List[tuple]:
    """migration.py:128-134 — moves are (item, src, dst, kv_bytes, tokens)."""
    return sorted(moves, key=lambda m: (-m[3], m[0]))


def plan_hybrid(moves: Sequence[tuple], *, gpm: int, intra_bw: float, inter_bw: float,
                prefill: float, comp_budget: float, intra_comm: float, inter_comm: float,
                comm_override: Optional[Dict[tuple, float]] = None,
                defer_counts: Optional[Dict[int, int]] = None, max_defer: int = 3) -> dict:
    """migration.py:137-170 — greedy two-budget assignment.

    Returns {"assignments": [(item, mode, latency)], "link_bytes": {...},
    "dest_tokens": {...}, "forced": [item, ...]} with dict insertion order
    identical to the reference's.
    """
    defer_counts = defer_counts or {}
    comm_override = comm_override or {}
    out = {"assignments": [], "link_bytes": {}, "dest_tokens": {}, "forced": []}
    for m in consensus_order(moves):
        item, src, dst, kvb, tok = m
        link = link_of(gpm, src, dst)
        used_link = out["link_bytes"].get(link, 0.0)
        used_dest = out["dest_tokens"].get(dst, 0.0)
        bw = intra_bw if link[0] == "intra" else inter_bw
        budget = comm_override[link] if link in comm_override else (
            intra_comm if link[0] == "intra" else inter_comm)       # :70-74
        if used_link + kvb <= budget:                                 # :155
            out["link_bytes"][link] = used_link + kvb
            out["assignments"].append((item, KV, kvb / bw))
        elif used_dest + tok <= comp_budget:                          # :159
            out["dest_tokens"][dst] = used_dest + tok
            out["assignments"].append((item, TOKEN, tok / prefill))
        elif defer_counts.get(item, 0) >= max_defer:                  # :164
            out["forced"].append(item)
            out["assignments"].append((item, FORCED, kvb / bw))
        else:
            out["assignments"].append((item, DEFER, 0.0))
    return out


def check_budgets(plan: dict, *, comp_budget: float, intra_comm: float, inter_comm: float,
                  comm_override: Optional[Dict[tuple, float]] = None) -> List[str]:
    """migration.py:173-182 — 1e-9 slack, forced transfers exempt."""
    comm_override = comm_override or {}
    problems = []
    for link, used in plan["link_bytes"].items():
        budget = comm_override[link] if link in comm_override else (
            intra_comm if link[0] == "intra" else inter_comm)
        if used > budget + 1e-9:
            problems.append(f"link {link} over comm budget: {used}")
    for dst, used in plan["dest_tokens"].items():
        if used > comp_budget + 1e-9:
            problems.append(f"gpu {dst} over comp budget: {used}")
    return problems
