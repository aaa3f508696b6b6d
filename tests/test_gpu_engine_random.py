"""Randomised engine options, bit-exact against the oracle on the B200:
stride, static ratio/placement, one or two HBM windows, host_io,
in-phase grad flush, fused/unfused downscale, fp16/bf16, ragged sizes,
dense or sparse pinned pool, two consecutive steps with re-planning in
between."""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest

from oracle import optistate_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2410_21316_b200 as D  # noqa: E402


def _instance(rng):
    n = int(rng.integers(1, 24))
    sg = int(rng.integers(8, 30_000))
    total = (n - 1) * sg + int(rng.integers(1, sg + 1))
    lowp = ["fp16", "bf16"][int(rng.integers(0, 2))]
    hyper = dict(lr=float(10 ** rng.uniform(-4, -2)), beta1=float(rng.uniform(0.8, 0.95)),
                 beta2=float(rng.uniform(0.95, 0.9995)), eps=float(10 ** rng.uniform(-9, -6)),
                 weight_decay=float(rng.choice([0.0, 0.0, 0.01])))
    steps = []
    for _ in range(2):
        stride = [1, 2, 3, 4, 5, D.ALL_CPU][int(rng.integers(0, 6))]
        mode = ["plain", "host_io", "flush"][int(rng.integers(0, 3))]
        steps.append(dict(stride=stride, ratio=float(rng.choice([0.0, 0.2, 0.5])),
                          placement=list(D.Placement)[int(rng.integers(0, 2))],
                          windows=int(rng.integers(1, 3)), mode=mode, fuse=bool(rng.integers(0, 2))))
    return total, sg, lowp, hyper, steps


def _plan(n, s):
    if s["ratio"] * n >= n - 1e-9 and s["stride"] is not D.ALL_CPU:
        return D.build_plan(n, s["stride"])
    return D.build_plan(n, s["stride"], s["ratio"], s["placement"])


def _sparse(total, sg, seed, lowp, static):
    """The oracle's shard in a sparse pool: residents homed in HBM only."""
    ref = O.initialize(total, sg, seed, lowp)
    return D.load_shard(ref["p"], ref["m"], ref["v"], ref["g"], ref["w"], sg, lowp=lowp, static_set=static)


def test_random_engine_options_match_oracle(h100):
    rng = np.random.default_rng(20261017)
    for case in range(48):
        total, sg, lowp, hyper, steps = _instance(rng)
        seed = int(rng.integers(0, 2**31))
        n = -(-total // sg)
        if rng.integers(0, 3) == 0:  # a third of the cases in a sparse pinned pool
            opt = _sparse(total, sg, seed, lowp, _plan(n, steps[0]).static_set)
        else:
            opt = D.ShardedOptimizer.initialize(total, sg, seed=seed, lowp=lowp)
            opt.to_device()
        ref = O.initialize(total, sg, seed, lowp)
        for s in steps:
            plan = _plan(n, s)
            cap = s["windows"] * 12 * sg
            prof = dataclasses.replace(h100, fast_capacity_bytes=cap)
            D.execute_plan(opt, plan, prof, D.AdamHyper(**hyper), host_io=s["mode"] == "host_io",
                           flush_grads=s["mode"] == "flush", fuse_downscale=s["fuse"])
            O.sequential_oracle(ref, **hyper)
        got = (opt.params32, opt.momentum32, opt.variance32, opt.model16)
        want = (ref["p"], ref["m"], ref["v"], ref["w"])
        for name, a, b in zip("pmvw", got, want):
            assert a.tobytes() == b.tobytes(), (case, name, total, sg, lowp, steps)
