"""State container, partitioner and the host-side step entry points."""
from __future__ import annotations

import json
import math
from pathlib import Path

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2410_21316_b200 as D
from oracle import optistate_oracle as O

STATES = json.loads((Path(__file__).resolve().parent / "golden" / "states.json").read_text())


def digest(opt) -> str:
    import hashlib

    h = hashlib.sha256()
    for a in (opt.params32, opt.momentum32, opt.variance32, opt.model16, opt.grads16):
        h.update(a.tobytes())
    return h.hexdigest()


def test_subgroup_and_shard():
    sg = D.Subgroup(index=2, start=200, size=100)
    assert (sg.stop, sg.slice, sg.state_bytes()) == (300, slice(200, 300), 1200)
    for kw in (dict(index=0, start=0, size=0), dict(index=0, start=-1, size=4)):
        with pytest.raises(ValueError):
            D.Subgroup(**kw)
    ranks = D.shard(1000, 3, 128)
    assert [sum(g.size for g in r) for r in ranks] == [334, 334, 332]
    assert [g.size for g in ranks[2]] == [128, 128, 76]
    for args in ((0, 1, 10), (10, 0, 10), (10, 1, 0)):
        with pytest.raises(ValueError):
            D.shard(*args)


@given(total=st.integers(1, 10_000), ranks=st.integers(1, 8), size=st.integers(1, 512))
@settings(max_examples=150, deadline=None)
def test_shard_properties(total, ranks, size):
    out = D.shard(total, ranks, size)
    assert len(out) == ranks and sum(g.size for r in out for g in r) == total
    for groups in out:
        off = 0
        for i, g in enumerate(groups):
            assert (g.index, g.start) == (i, off) and 0 < g.size <= size
            off = g.stop
        assert all(g.size == size for g in groups[:-1])
        assert sum(g.size for g in groups) <= math.ceil(total / ranks)


def test_footprint_and_profile_validation():
    rep = D.footprint(6_000_000_000, 100_000_000)
    assert (rep.fast_resident_bytes, rep.optimizer32_bytes, rep.per_subgroup_state_bytes, rep.num_subgroups) == (
        24_000_000_000, 96_000_000_000, 1_200_000_000, 60)
    base = dict(name="t", channel_params_per_s=1e9, fast_update_params_per_s=1e10, cpu_update_params_per_s=1e9,
                cpu_downscale_params_per_s=1e9, fast_convert_bytes_per_s=1e12, host_convert_bytes_per_s=1e10,
                host_alloc_bytes_per_s=1e9, pageable_d2h_bytes_per_s=1e9, pageable_h2d_bytes_per_s=1e9)
    for bad in (dict(channel_params_per_s=0.0), dict(cpu_update_params_per_s=-1.0), dict(host_contention=0.5)):
        with pytest.raises(ValueError):
            D.SystemProfile(**{**base, **bad})
    assert D.Precision.FP16.itemsize == 2 and D.Precision.FP32.itemsize == 4 and D.Precision.BF16.itemsize == 2


def test_initialize_matches_reference_draws_and_is_pinned():
    for key in [k for k in STATES["oracle"] if k.endswith("|init")]:
        total, sg, seed, _ = key.split("|")
        opt = D.ShardedOptimizer.initialize(int(total), int(sg), seed=int(seed))
        assert digest(opt) == STATES["oracle"][key]
    opt = D.ShardedOptimizer.initialize(1000, 128, seed=3)
    assert opt.params32.ctypes.data % 4096 == 0  # pinned-pool view, page aligned
    assert len(opt.subgroups) == 8 and opt.subgroups[-1].size == 1000 - 7 * 128


def test_validation_and_copy():
    groups = D.shard(100, 1, 32)[0]
    z32, z16 = np.zeros(100, np.float32), np.zeros(100, np.float16)
    with pytest.raises(TypeError):
        D.ShardedOptimizer(groups, z32.astype(np.float64), z32, z32, z16, z16)
    with pytest.raises(ValueError):
        D.ShardedOptimizer(groups, z32[:99], z32, z32, z16, z16)
    with pytest.raises(TypeError):
        D.ShardedOptimizer(groups, z32, z32, z32, z32.copy(), z16)
    a = D.ShardedOptimizer.initialize(256, 64, seed=1)
    b = a.copy()
    assert a.state_equal(b)
    b.params32[0] += np.float32(1.0)
    assert not a.state_equal(b)


@pytest.mark.parametrize("key", sorted(k for k in STATES["oracle"] if not k.endswith("|init")))
def test_host_sequential_oracle_matches_reference_digests(key):
    total, sg, seed, steps = key.split("|")
    opt = D.ShardedOptimizer.initialize(int(total), int(sg), seed=int(seed))
    for _ in range(int(steps)):
        D.sequential_oracle(opt, D.AdamHyper())
    assert opt.step == int(steps)
    assert digest(opt) == STATES["oracle"][key]


def test_host_sequential_oracle_acceptance_instances():
    for inst in STATES["acceptance"]:
        opt = D.ShardedOptimizer.initialize(inst["total"], inst["sg"], seed=inst["seed"])
        D.sequential_oracle(opt, D.AdamHyper(**inst["hyper"]))
        assert digest(opt) == inst["digest"], inst


def test_adam_step_subgroup_leaves_model16_stale():
    opt = D.ShardedOptimizer.initialize(512, 256, seed=1)
    before = opt.model16.copy()
    D.adam_step_subgroup(opt, 0, D.AdamHyper())
    assert opt.model16.tobytes() == before.tobytes() and opt.step == 0


def test_bf16_shard_host_oracle():
    opt = D.ShardedOptimizer.initialize(50_000, 7_000, seed=2, lowp="bf16")
    ref = O.initialize(50_000, 7_000, seed=2, lowp="bf16")
    assert opt.grads16.tobytes() == ref["g"].tobytes()
    D.sequential_oracle(opt, D.AdamHyper(lr=3e-4))
    O.sequential_oracle(ref, lr=3e-4)
    assert opt.params32.tobytes() == ref["p"].tobytes() and opt.model16.tobytes() == ref["w"].tobytes()


def test_hyper_validation():
    for kw in (dict(beta1=1.0), dict(beta2=-0.1), dict(lr=0.0), dict(eps=0.0), dict(weight_decay=-1.0)):
        with pytest.raises(ValueError):
            D.AdamHyper(**kw)


def test_flush_gradients_host_exact(h100):
    opt = D.ShardedOptimizer.initialize(3000, 1024, seed=6)
    want = opt.grads16.astype(np.float32)
    for strat in D.GradFlushStrategy:
        for chunk in (2, 130, 1 << 22):
            out, rec = D.flush_gradients(opt, h100, strat, chunk_bytes=chunk)
            assert out.tobytes() == want.tobytes() and rec.payload_bytes == 6000
    with pytest.raises(ValueError):
        D.flush_gradients(opt, h100, D.GradFlushStrategy.FP16_HOST_UPSCALE, chunk_bytes=1)


def test_execute_plan_needs_a_gpu(h100):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    opt = D.ShardedOptimizer.initialize(1024, 256, seed=0)
    with pytest.raises(ValueError):
        D.execute_plan(opt, D.build_plan(3, 2), h100, D.AdamHyper())
    with pytest.raises(RuntimeError, match="CUDA"):
        D.execute_plan(opt, D.build_plan(4, 2), h100, D.AdamHyper())


def test_emulated_device_ledger():
    dev = D.EmulatedDevice()
    dev.stage(0, "m", np.zeros(4, np.float32))
    with pytest.raises(AssertionError):
        dev.stage(0, "m", np.zeros(4, np.float32))
    dev.stage(0, "v", np.zeros(4, np.float32))
    with pytest.raises(AssertionError):
        dev.require_triplet(0)
    dev.stage(0, "p", np.zeros(4, np.float32))
    assert set(dev.require_triplet(0)) == {"m", "v", "p"}
    with pytest.raises(AssertionError):
        dev.unstage(3, "p")
    with pytest.raises(AssertionError):
        dev.assert_drained()
    for piece in "mvp":
        dev.unstage(0, piece)
    dev.assert_drained()


def test_sparse_pool_commits_only_host_homed_subgroups():
    """allocate(host_homed=...) reserves the shard but commits host memory
    only for the listed subgroups (2 MB granularity); the rest read as zeros
    and are committed on demand."""
    SG = 1 << 20  # 4 MiB of fp32 per subgroup piece
    opt = D.ShardedOptimizer.allocate(8 * SG, SG, lowp="bf16", host_homed=[0, 1, 5])
    assert opt.host_runs("state") == [(0, 2 * SG), (5 * SG, 6 * SG)]
    assert opt.host_runs("lowp") == [(0, 2 * SG), (5 * SG, 6 * SG)]
    assert [opt.host_committed(i) for i in range(8)] == [True, True, False, False, False, True, False, False]
    full = 8 * SG * 16
    assert opt.host_bytes == 3 * SG * 16 < full
    opt._p[: 2 * SG] = 1.5
    assert float(opt._p[3 * SG]) == 0.0  # uncommitted range reads as zeros
    opt.ensure_host([2, 3], "state")
    assert opt.host_runs("state") == [(0, 4 * SG), (5 * SG, 6 * SG)]
    assert float(opt._p[0]) == 1.5  # merging runs keeps committed contents
    opt.ensure_host([2, 3], "state")  # idempotent
    assert opt.params32.shape == (8 * SG,)  # a full-array read materialises every range
    assert opt.host_runs("state") == [(0, 8 * SG)]
    assert all(opt.host_committed(i) for i in range(8))
    assert float(opt.params32[SG - 1]) == 1.5 and float(opt.params32[7 * SG]) == 0.0


def test_sparse_pool_matches_dense_host_oracle():
    """A sparse shard, fully committed on demand, runs the host oracle to the
    same digest as a dense one."""
    dense = D.ShardedOptimizer.initialize(5000, 1024, seed=3, lowp="bf16")
    sparse = D.ShardedOptimizer.allocate(5000, 1024, lowp="bf16", host_homed=[1, 3])
    for name in ("params32", "momentum32", "variance32", "model16", "grads16"):
        getattr(sparse, name)[:] = getattr(dense, name)
    hyper = D.AdamHyper()
    D.sequential_oracle(dense, hyper)
    D.sequential_oracle(sparse, hyper)
    assert sparse.state_equal(dense)
    with pytest.raises(ValueError):
        D.ShardedOptimizer.allocate(5000, 1024, host_homed=[5])


def test_sparse_pool_abi_errors():
    from paper_2410_21316_b200 import _native as N

    hb = N.HostBuffer(1 << 22, sparse=True)
    assert hb.committed_bytes == 0
    hb.commit(100, 10)
    assert hb.committed_bytes == 2 << 20
    with pytest.raises(ValueError):
        hb.commit(1 << 22, 1)
    with pytest.raises(ValueError):
        N.check(N.lib().dos_host_commit(12345, 0, 1))


def test_host_membw_probe():
    import ctypes

    from paper_2410_21316_b200 import _native as N

    a, b = N.HostBuffer(1 << 22, register_cuda=False), N.HostBuffer(1 << 22, register_cuda=False)
    secs = ctypes.c_double()
    for mode in (0, 1):
        N.check(N.lib().dos_host_membw(a.address, b.address, 1 << 22, mode, 0, ctypes.byref(secs)))
        assert secs.value > 0
    a.array(np.uint8, 1 << 22)[:] = 7
    N.check(N.lib().dos_host_membw(a.address, b.address, 1 << 22, 1, 0, ctypes.byref(secs)))
    assert (b.array(np.uint8, 1 << 22) == 7).all()  # the copy pass really copies
    for bad in ((a.address, b.address, 1 << 22, 2), (a.address, None, 1 << 22, 1), (None, b.address, 64, 0)):
        with pytest.raises(ValueError):
            N.check(N.lib().dos_host_membw(*bad, 0, ctypes.byref(secs)))


def test_load_shard_validates_before_touching_a_device():
    from paper_2410_21316_b200.device import load_shard

    n = 1000
    f32, u16 = np.zeros(n, np.float32), np.zeros(n, np.uint16)
    with pytest.raises(TypeError):
        load_shard(f32, f32, f32, f32, u16, 100)  # grads must be bf16 bits
    with pytest.raises(ValueError):
        load_shard(f32, f32[:-1], f32, u16, u16, 100)
    with pytest.raises(ValueError):
        load_shard(f32, f32, f32, u16, u16, 100, static_set={10})
