"""Interop with the reference package itself (CPU; skipped where
/root/reference is absent, e.g. on the GPU box): our SimTarget served by the
reference's own run_update gives the reference simulator's timeline."""
from __future__ import annotations

import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference package not present")


@pytest.fixture(scope="module")
def R():
    sys.path.insert(0, str(REF))
    import optistate

    return optistate


def test_reference_engine_drives_our_target(R):
    import paper_2410_21316_b200 as D

    for stride in (1, 2, 3, R.ALL_CPU):
        rplan = R.build_plan(10, stride, 0.2)
        ours = D.SimTarget(D.get_profile("h100-node"), rplan, 10**8)
        got = R.run_update(rplan, ours)
        want = R.simulate_update_phase(rplan, R.get_profile("h100-node"), 10**8).events
        assert [(e.action.id, e.start_ns, e.end_ns, e.bytes) for e in got] == \
               [(e.action.id, e.start_ns, e.end_ns, e.bytes) for e in want]


def test_plan_descs_accept_reference_plans(R):
    from paper_2410_21316_b200.device import plan_descs
    from paper_2410_21316_b200.plan import KIND_CODE

    rplan = R.build_plan(9, 3, 0.25)
    ours = __import__("paper_2410_21316_b200").build_plan(9, 3, 0.25)
    a, b = plan_descs(rplan).descs, plan_descs(ours).descs
    for i in range(len(ours.actions)):
        assert (a[i].kind, a[i].lane, a[i].subgroup, a[i].is_static, a[i].num_deps) == \
               (b[i].kind, b[i].lane, b[i].subgroup, b[i].is_static, b[i].num_deps)
    assert set(KIND_CODE.values()) == set(range(12))
