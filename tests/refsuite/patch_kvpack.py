"""pytest plugin: swap this repo's planner into the REFERENCE package before the
reference's own tests import it, so /root/reference/pkg/tests/test_migration.py
and test_sim.py exercise paper_2501_06709_b200.planner (and its ConfigError)
instead of kvpack.migration.  Loaded with `-p patch_kvpack` by
tests/test_reference_suite.py; never imported by the product."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import kvpack  # noqa: E402  (the reference, via PYTHONPATH)
import kvpack.migration as ref_migration  # noqa: E402
import kvpack.sim as ref_sim  # noqa: E402
import kvpack.verification as ref_verif  # noqa: E402

import paper_2501_06709_b200.errors as ours_errors  # noqa: E402
import paper_2501_06709_b200.planner as ours  # noqa: E402

NAMES = ["Topology", "Boundaries", "load_boundaries", "PendingMove", "PlannedMove", "MigrationPlan",
         "consensus_order", "plan_hybrid", "check_budgets", "KV_TRANSFER", "TOKEN_TRANSFER", "DEFERRED",
         "FORCED_KV_TRANSFER"]
for name in NAMES:
    setattr(ref_migration, name, getattr(ours, name))
    if hasattr(kvpack, name):
        setattr(kvpack, name, getattr(ours, name))
    for mod in (ref_sim, ref_verif):
        if hasattr(mod, name):
            setattr(mod, name, getattr(ours, name))
# the reference tests catch kvpack.ConfigError; ours must be that class for them
kvpack.ConfigError = ours_errors.ConfigError
ref_migration.ConfigError = ours_errors.ConfigError
os.environ["KVPACK_PLANNER_UNDER_TEST"] = ours.__file__
