"""Differential driver: the native MellScheduler vs the reference's, in lockstep.

Test infrastructure only (imported by tests/test_scheduler_native.py and
tools/bench_scheduler.py).  Both schedulers receive identical step_epoch
inputs produced by a slot loop shaped like the reference's sim.run
(sim.py:151-205: growth, completions, arrivals, rejections and aborts drop
requests); after every epoch the EpochResults and the full cluster state
(placement, sizes, groups, GPUs with residents and activation sequence,
request->group map, id counters, scheduled_class) must be identical.
"""
from __future__ import annotations

import math
import os
import random
import sys

REF = "/root/reference/pkg/src"


def kvpack():
    """The reference package, or None when /root/reference is not mounted."""
    if not os.path.isdir(REF):
        return None
    if REF not in sys.path:
        sys.path.append(REF)
    import kvpack as k
    return k


def result_key(res):
    return ([(log.kind, log.request_id, [(m.item, m.src, m.dst, m.reason) for m in log.moves],
              [tuple(e) for e in log.events]) for log in res.logs], list(res.terminated), bool(res.batched))


def state_key(cluster, sched, native: bool):
    gpus = [(g, st.machine_id, st.activation_seq, sorted(st.residents)) for g, st in cluster.gpus.items()]
    groups = [(gid, sorted(gr.members), gr.aggregate_bytes) for gid, gr in cluster.groups.items()]
    if native:
        snap = cluster._snap()
        counters = (snap.next_activation_seq, snap.next_group_id, snap.next_gpu_id, sorted(snap.free_ids))
        sc = {k: v.value for k, v in sched.scheduled_class.items()}
    else:
        counters = (cluster.next_activation_seq, cluster._next_group_id, cluster._next_gpu_id,
                    sorted(cluster._free_gpu_ids))
        sc = {k: v.value for k, v in sched.scheduled_class.items()}
    return (sorted(gpus), list(cluster.placement.items()), list(cluster.sizes.items()), sorted(groups),
            sorted(cluster.request_group.items()), counters, sorted(sc.items()))


def random_trace(rng: random.Random, n: int, slots: int, max_prompt: int, max_resp: int):
    recs = []
    for rid in range(n):
        recs.append((rid, rng.randrange(slots), rng.randint(1, max_prompt), rng.randint(1, max_resp)))
    return recs


def lockstep(ref_mod, ours_mod, recs, *, capacity, gpm, prio, batching, bpt, tps, epoch_slots=1,
             check_state_every=1, on_mismatch=None):
    """Drive both schedulers over `recs`; returns the number of epochs compared.
    Raises AssertionError at the first divergence."""
    rc = ref_mod.ClusterState(capacity, gpus_per_machine=gpm)
    rs = ref_mod.MellScheduler(rc, priority_cfg=ref_mod.PriorityConfig(*prio), batching=batching)
    oc = ours_mod.ClusterState(capacity, gpus_per_machine=gpm)
    os_ = ours_mod.MellScheduler(oc, priority_cfg=ours_mod.PriorityConfig(*prio), batching=batching)
    by_slot, by_id = {}, {r[0]: r for r in recs}
    for r in recs:
        by_slot.setdefault(r[1], []).append(r)
    horizon = max((r[1] for r in recs), default=-1) + 1
    running, buffered = {}, []
    slot = 0
    while slot < horizon or running or buffered:
        growths, completions = {}, []
        for rid, (_, arr, prompt, resp) in running.items():
            if arr + math.ceil(resp / tps) <= slot:
                completions.append(rid)
            else:
                growths[rid] = (prompt + min(resp, tps * (slot - arr))) * bpt
        for rec in by_slot.get(slot, []):
            buffered.append((rec[0], rec[2] * bpt))
        if slot % epoch_slots == 0:
            arrivals, buffered = buffered, []
        else:
            arrivals = []
        a = rs.step_epoch(arrivals, completions, growths=growths)
        b = os_.step_epoch(arrivals, completions, growths=growths)
        ka, kb = result_key(a), result_key(b)
        if ka != kb:
            if on_mismatch:
                on_mismatch(slot, ka, kb)
            raise AssertionError(f"slot {slot}: epoch results differ\nref : {ka}\nours: {kb}")
        if slot % check_state_every == 0:
            sa, sb = state_key(rc, rs, False), state_key(oc, os_, True)
            assert sa == sb, f"slot {slot}: cluster state differs\nref : {sa}\nours: {sb}"
        assert rs.epoch_migration_counts == os_.epoch_migration_counts
        gone = set(completions)
        for log in a.logs:
            for kind, *detail in log.events:
                if kind in ("rejected", "aborted"):
                    gone.add(int(detail[0]))
        for rid in gone:
            running.pop(rid, None)
        for rid, _ in arrivals:
            if rid not in gone:
                running[rid] = by_id[rid]
        slot += 1
        if slot > horizon + 100000:
            raise RuntimeError("did not drain")
    return slot
