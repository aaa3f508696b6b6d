"""Sparse host pool + per-subgroup HBM homes on the B200: a shard whose
static residents never touch host memory runs the update phase bit-exactly
against the oracle, the phase commits no host memory, and the static set can
shrink and grow between steps (subgroups move home one at a time)."""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import optistate_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2410_21316_b200 as D  # noqa: E402
from paper_2410_21316_b200 import Placement  # noqa: E402

HYPER = D.AdamHyper()


def sparse_shard(total, sg, seed, lowp, static_set):
    """The oracle's seeded shard, loaded with its static residents homed in
    HBM only (D.load_shard: sparse pinned pool)."""
    want = O.initialize(total, sg, seed, lowp)
    opt = D.load_shard(want["p"], want["m"], want["v"], want["g"], want["w"], sg, lowp=lowp, static_set=static_set)
    return opt, want


def assert_matches(opt, want):
    assert np.array_equal(opt.params32.view(np.uint32), want["p"].view(np.uint32))
    assert np.array_equal(opt.momentum32.view(np.uint32), want["m"].view(np.uint32))
    assert np.array_equal(opt.variance32.view(np.uint32), want["v"].view(np.uint32))
    assert np.array_equal(opt.model16.view(np.uint16), want["w"].view(np.uint16))


@pytest.mark.parametrize("lowp", ["bf16", "fp16"])
@pytest.mark.parametrize("placement", list(Placement))
@pytest.mark.parametrize("stride", [1, 2, 3])
def test_sparse_static_phase_matches_oracle(h100, lowp, placement, stride):
    total, sg = 10 * (1 << 20) + 12345, 1 << 20  # 11 subgroups, ragged tail, 4 MiB fp32 pieces
    plan = D.build_plan(11, stride, static_ratio=0.5, placement=placement)
    opt, want = sparse_shard(total, sg, 5, lowp, plan.static_set)
    committed = opt.host_bytes
    assert committed < 16 * total
    for _ in range(2):
        D.execute_plan(opt, plan, h100, HYPER)
        O.sequential_oracle(want)
    assert opt.host_bytes == committed  # the phase itself commits nothing
    assert_matches(opt, want)


def test_static_set_shrinks_and_grows_between_steps(h100):
    total, sg = 12 * (1 << 20), 1 << 20
    ratios = (0.5, 0.25, 0.75, 0.0, 1.0, 0.5)
    first = D.build_plan(12, 2, static_ratio=ratios[0])
    opt, want = sparse_shard(total, sg, 8, "bf16", first.static_set)
    for r in ratios:
        plan = D.build_plan(12, 2, static_ratio=r, placement=Placement.STATIC_LAST)
        D.execute_plan(opt, plan, h100, HYPER)
        O.sequential_oracle(want)
        assert opt.residency.static_set == plan.static_set
        assert set(opt.residency.static_sg) == set(plan.static_set)
    assert_matches(opt, want)


@pytest.mark.parametrize("placement", list(Placement))
def test_sparse_host_io_commits_grads_and_matches(h100, placement):
    """host_io reads every subgroup's grads from the host image: the target
    commits the half-precision ranges of the static residents first.  With
    STATIC_FIRST the residents' grads are shipped just ahead of the fast lane
    (host_io_ahead), with STATIC_LAST all at phase start."""
    total, sg = 8 * (1 << 20), 1 << 20
    plan = D.build_plan(8, 2, static_ratio=0.5, placement=placement)
    opt, want = sparse_shard(total, sg, 2, "bf16", plan.static_set)
    D.execute_plan(opt, plan, h100, HYPER)  # device grads
    O.sequential_oracle(want)
    opt.grads16[:] = want["g"]  # the next step's grads arrive on the host
    D.execute_plan(opt, plan, h100, HYPER, host_io=True)
    O.sequential_oracle(want)
    assert_matches(opt, want)


def test_host_side_oracle_on_a_sparse_shard(h100):
    """A host-side pass (sequential_oracle / adam_step_subgroup) over a shard
    whose residents live only in HBM first pulls them to the host, so the
    host update sees their real state and the re-upload keeps it."""
    total, sg = 6 * (1 << 20), 1 << 20
    plan = D.build_plan(6, 2, static_ratio=0.5, placement=Placement.STATIC_FIRST)
    opt, want = sparse_shard(total, sg, 4, "bf16", plan.static_set)
    D.sequential_oracle(opt, HYPER)
    O.sequential_oracle(want)
    D.execute_plan(opt, plan, h100, HYPER)  # the residents' HBM homes were refreshed from the host pass
    O.sequential_oracle(want)
    assert_matches(opt, want)
