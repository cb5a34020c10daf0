"""plan_hybrid cost: Python drop-in vs native kvm_plan_hybrid (host CPU, no GPU).

SURVEY.md §6 measured the reference at 1.1 / 4.3 / 32.8 / 569 us for n = 1 / 8 / 64 / 1024.
"""
import ctypes
import json
import os
import random
import sys
import timeit

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2501_06709_b200 import _native  # noqa: E402
from paper_2501_06709_b200.planner import (PendingMove, Topology, load_boundaries, plan_hybrid,  # noqa: E402
                                           plan_hybrid_native)


def main():
    rng = random.Random(0)
    topo = Topology(gpus_per_machine=8, intra_bandwidth_bytes_per_s=900e9)
    bounds = load_boundaries(topo, 0.05, 0.2)
    out = {}
    for n in (1, 8, 64, 1024):
        moves = [PendingMove(i, rng.randrange(16), rng.randrange(16), rng.randint(1, 4 * 10 ** 9),
                             rng.randint(1, 8000)) for i in range(n)]
        defer = {i: rng.randint(0, 4) for i in range(0, n, 3)}
        reps = max(20, 20000 // n)
        py = min(timeit.repeat(lambda: plan_hybrid(moves, bounds, topo, defer), number=reps, repeat=5)) / reps
        nat = min(timeit.repeat(lambda: plan_hybrid_native(moves, bounds, topo, defer), number=reps,
                                repeat=5)) / reps
        assert plan_hybrid(moves, bounds, topo, defer) == plan_hybrid_native(moves, bounds, topo, defer)
        # the C ABI call alone, arguments pre-marshalled (what a C/C++ host pays)
        arr = (_native.Pending * n)(*[_native.Pending(m.item, m.src, m.dst, m.kv_bytes, m.tokens,
                                                      defer.get(m.item, 0)) for m in moves])
        pp = _native.PlanParams(8, 3, 900e9, 1.25e9, 10_000.0, bounds.comp_budget, bounds.intra_comm_budget,
                                bounds.inter_comm_budget, 0, 0, None, None)
        res = (_native.Planned * n)()
        fn = _native.lib().kvm_plan_hybrid
        c_only = min(timeit.repeat(lambda: fn(arr, n, ctypes.byref(pp), res, None), number=reps,
                                   repeat=5)) / reps
        out[n] = {"python_us": round(py * 1e6, 2), "native_from_python_us": round(nat * 1e6, 2),
                  "native_call_us": round(c_only * 1e6, 2)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
