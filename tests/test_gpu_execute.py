"""execute_plan on the B200: every plan shape reproduces the reference's
sequential update bit for bit (fp16 kind: against the reference's own
digests; bf16 kind: against the oracle), with the measured timeline audited."""
from __future__ import annotations

import dataclasses
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import optistate_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2410_21316_b200 as D  # noqa: E402
from paper_2410_21316_b200 import ALL_CPU, Placement  # noqa: E402

STATES = json.loads((Path(__file__).resolve().parent / "golden" / "states.json").read_text())
HYPER = D.AdamHyper()


def digest(opt) -> str:
    h = hashlib.sha256()
    for a in (opt.params32, opt.momentum32, opt.variance32, opt.model16, opt.grads16):
        h.update(a.tobytes())
    return h.hexdigest()


def oracle_digest(total, sg, seed, lowp="fp16", steps=1, **hyper):
    st = O.initialize(total, sg, seed, lowp)
    for _ in range(steps):
        O.sequential_oracle(st, **hyper)
    return O.state_digest(st)


@pytest.mark.parametrize("stride", [1, 2, 3, ALL_CPU])
@pytest.mark.parametrize("ratio", [0.0, 0.25])
@pytest.mark.parametrize("placement", list(Placement))
def test_any_plan_matches_oracle(h100, stride, ratio, placement):
    opt = D.ShardedOptimizer.initialize(10 * 1024, 1024, seed=11)
    plan = D.build_plan(10, stride, static_ratio=ratio, placement=placement)
    res = D.execute_plan(opt, plan, h100, HYPER, check_coherence=True)
    assert res.step == 1 and opt.step == 1
    assert digest(opt) == STATES["oracle"]["10240|1024|11|1"]
    assert res.measured is not None and len(res.measured.events) == len(plan.actions)


def test_acceptance_instances_on_b200(h100):
    """The reference's 236 schedule-independence instances (test_acceptance.py:121-175)."""
    for inst in STATES["acceptance"]:
        opt = D.ShardedOptimizer.initialize(inst["total"], inst["sg"], seed=inst["seed"])
        plan = D.build_plan(len(opt.subgroups), inst["stride"], static_ratio=inst["ratio"],
                            placement=Placement(inst["placement"]))
        D.execute_plan(opt, plan, h100, D.AdamHyper(**inst["hyper"]))
        assert digest(opt) == inst["digest"], inst
    for stride in range(1, 7):
        for ratio in (0.0, 0.25, 0.5):
            for pl in Placement:
                opt = D.ShardedOptimizer.initialize(12 * 257, 257, seed=4242)
                D.execute_plan(opt, D.build_plan(12, stride, ratio, pl), h100, HYPER)
                assert digest(opt) == STATES["fixed_4242"]


def test_ragged_consecutive_and_replanned_steps(h100):
    opt = D.ShardedOptimizer.initialize(5000, 1024, seed=5)
    D.execute_plan(opt, D.build_plan(5, 2), h100, HYPER)
    assert digest(opt) == oracle_digest(5000, 1024, 5)
    opt = D.ShardedOptimizer.initialize(2048, 512, seed=2)
    D.execute_plan(opt, D.build_plan(4, 2), h100, HYPER)
    D.execute_plan(opt, D.build_plan(4, 3, 0.25), h100, HYPER)  # re-plan: subgroups change tier
    assert opt.step == 2 and digest(opt) == STATES["oracle"]["2048|512|2|2"]


def test_custom_hyper_and_bf16_kind(h100):
    hyper = D.AdamHyper(lr=3e-4, beta1=0.8, beta2=0.95, eps=1e-6)
    opt = D.ShardedOptimizer.initialize(1536, 256, seed=8)
    D.execute_plan(opt, D.build_plan(6, 3, static_ratio=0.3, placement=Placement.STATIC_FIRST), h100, hyper)
    assert digest(opt) == oracle_digest(1536, 256, 8, lr=3e-4, beta1=0.8, beta2=0.95, eps=1e-6)
    for stride in (1, 2, 3, ALL_CPU):
        opt = D.ShardedOptimizer.initialize(70_000, 7_000, seed=3, lowp="bf16")
        D.execute_plan(opt, D.build_plan(10, stride, 0.2), h100, HYPER)
        D.execute_plan(opt, D.build_plan(10, stride, 0.2), h100, HYPER)
        assert digest(opt) == oracle_digest(70_000, 7_000, 3, "bf16", steps=2)


def test_adamw_matches_oracle(h100):
    hyper = D.AdamHyper(weight_decay=0.01)
    opt = D.ShardedOptimizer.initialize(40_000, 4_000, seed=4, lowp="bf16")
    D.execute_plan(opt, D.build_plan(10, 2, 0.2), h100, hyper)
    assert digest(opt) == oracle_digest(40_000, 4_000, 4, "bf16", weight_decay=0.01)


def test_predicted_timeline_equals_simulator_and_measured_validates(h100):
    opt = D.ShardedOptimizer.initialize(8 * 256, 256, seed=4)
    plan = D.build_plan(8, 2, static_ratio=0.25)
    sim = D.simulate_update_phase(plan, h100, [g.size for g in opt.subgroups])
    res = D.execute_plan(opt, plan, h100, HYPER)
    assert res.timeline.events == sim.events and res.timeline.makespan_ns == sim.makespan_ns
    m = res.measured
    assert m.makespan_ns > 0 and m.span_ns >= m.makespan_ns
    assert {e.action.id for e in m.events} == set(range(len(plan.actions)))


def test_single_window_capacity(h100):
    prof = dataclasses.replace(h100, fast_capacity_bytes=12 * 1000)
    opt = D.ShardedOptimizer.initialize(8000, 1000, seed=9)
    res = D.execute_plan(opt, D.build_plan(8, 1), prof, HYPER)
    assert digest(opt) == oracle_digest(8000, 1000, 9)
    with pytest.raises(D.InfeasibleConfigError):
        D.execute_plan(D.ShardedOptimizer.initialize(8000, 1000, seed=9), D.build_plan(8, 1),
                       dataclasses.replace(h100, fast_capacity_bytes=11_999), HYPER)
    assert res.measured is not None


def test_large_subgroups_sampled(h100):
    """Four 25M-param subgroups, bf16, stride 2: property check at size."""
    total, sg = 100_000_000, 25_000_000
    opt = D.ShardedOptimizer.initialize(total, sg, seed=1, lowp="bf16")
    want = O.initialize(total, sg, 1, "bf16")
    D.execute_plan(opt, D.build_plan(4, 2), h100, HYPER)
    O.sequential_oracle(want)
    assert np.array_equal(opt.params32.view(np.uint32), want["p"].view(np.uint32))
    assert np.array_equal(opt.variance32.view(np.uint32), want["v"].view(np.uint32))
    assert np.array_equal(opt.model16, want["w"])


def test_flush_gradients_device_path(h100):
    opt = D.ShardedOptimizer.initialize(300_000, 70_000, seed=6, lowp="bf16")
    opt.to_device()
    out, rec = D.flush_gradients(opt, h100, D.GradFlushStrategy.GPU_UPSCALE_FP32, chunk_bytes=1 << 16)
    assert out.tobytes() == O.f32_from_bf16(opt.grads16).tobytes()


def test_load_grads_from_device_tensor(h100):
    opt = D.ShardedOptimizer.initialize(20_000, 5_000, seed=2, lowp="bf16")
    res = opt.to_device()
    g = torch.randn(20_000, device="cuda").to(torch.bfloat16)
    opt.load_grads(g)
    assert np.array_equal(opt.grads16, g.view(torch.int16).cpu().numpy().view(np.uint16))
    want = O.initialize(20_000, 5_000, 2, "bf16")
    want["g"] = opt.grads16.copy()
    D.execute_plan(opt, D.build_plan(4, 2), h100, HYPER)
    O.sequential_oracle(want)
    assert opt.params32.tobytes() == want["p"].tobytes() and res.model16.view(torch.int16).cpu().numpy().view(
        np.uint16).tobytes() == want["w"].tobytes()


def test_host_io_mode_reads_host_grads_and_mirrors_working_copy(h100):
    opt = D.ShardedOptimizer.initialize(90_000, 10_000, seed=12, lowp="bf16")
    res = opt.to_device()
    res.grads.zero_()  # device grads are stale: host_io must ship the host image
    plan = D.build_plan(9, 2, static_ratio=0.25)
    D.execute_plan(opt, plan, h100, HYPER, host_io=True)
    assert "_w" not in res.host_stale  # mirrored inside the phase
    want = O.sequential_oracle(O.initialize(90_000, 10_000, 12, "bf16"))
    assert opt._w.tobytes() == want["w"].tobytes()
    assert opt.params32.tobytes() == want["p"].tobytes()
    assert res.model16.view(torch.int16).cpu().numpy().view(np.uint16).tobytes() == want["w"].tobytes()


def test_b200_policy_refit_and_choice(h100):
    from paper_2410_21316_b200 import policy

    opt = D.ShardedOptimizer.initialize(400_000, 40_000, seed=1, lowp="bf16")
    sizes = [g.size for g in opt.subgroups]
    r = D.execute_plan(opt, D.build_plan(10, 2), h100, HYPER)
    prof = policy.refit_profile(h100, r.measured, sizes)
    assert prof.channel_params_per_s > 0 and prof.fast_update_params_per_s > 0
    k, spans = policy.choose_stride(prof, sizes)
    assert k in spans and spans[k] == min(spans.values())


def _tampered(plan, actions):
    import dataclasses as dc

    return dc.replace(plan, actions=tuple(actions))


def test_engine_rejects_structural_violations(h100):
    """The native engine enforces EmulatedDevice's rules on real HBM slots
    (executor.py:134-171): a fast update without its triplet, a flush of a
    piece never staged and a double stage all raise, and the engine stays
    usable afterwards."""
    from paper_2410_21316_b200.plan import Action, ActionKind

    opt = D.ShardedOptimizer.initialize(40_000, 10_000, seed=2, lowp="bf16")
    plan = D.build_plan(4, 1)
    acts = list(plan.actions)
    # drop subgroup 0's PREFETCH_V: GPU_UPDATE 0 finds an incomplete window
    bad = [a for a in acts if not (a.kind is ActionKind.PREFETCH_V and a.subgroup == 0)]
    bad = [Action(i, a.kind, a.subgroup, a.lane, a.stream, a.batch,
                  tuple(d if d < 1 else d - 1 for d in a.deps if d != 1)) for i, a in enumerate(bad)]
    with pytest.raises(AssertionError):
        D.execute_plan(opt, _tampered(plan, bad), h100, HYPER, validate_measured=False)
    # double stage: PREFETCH_M of subgroup 0 twice
    dup = acts[:1] + [Action(1, ActionKind.PREFETCH_M, 0, acts[0].lane, acts[0].stream)]
    with pytest.raises(AssertionError):
        D.execute_plan(opt, _tampered(plan, dup), h100, HYPER, validate_measured=False)
    # the engine recovers: a valid phase on a fresh shard still matches the oracle
    ok = D.ShardedOptimizer.initialize(40_000, 10_000, seed=2, lowp="bf16")
    ok.residency = None
    D.execute_plan(ok, plan, h100, HYPER)
    assert digest(ok) == oracle_digest(40_000, 10_000, 2, "bf16")


def test_throttled_mode_paces_but_matches(h100):
    import time

    opt = D.ShardedOptimizer.initialize(512, 256, seed=3)
    t0 = time.perf_counter()
    res = D.execute_plan(opt, D.build_plan(2, 2), h100, HYPER, mode=D.ExecMode.THROTTLED, throttle_scale=1e-7)
    assert time.perf_counter() - t0 < 5.0 and res.mode is D.ExecMode.THROTTLED
    assert digest(opt) == oracle_digest(512, 256, 3)
    with pytest.raises(ValueError):
        D.execute_plan(opt, D.build_plan(2, 2), h100, HYPER, mode=D.ExecMode.THROTTLED, throttle_scale=0.0)


@pytest.mark.parametrize("name,nsub,tail", [
    ("7B/1", 70, 1.0), ("13B/1", 130, 1.0), ("13B/2", 65, 1.0), ("20B/4", 50, 1.0), ("20B/8", 25, 1.0),
    ("70B/8", 88, 0.5),
])
def test_baseline_config_shapes(name, nsub, tail):
    """Each BASELINE config's per-rank shard shape (subgroup count, ragged
    last subgroup) at a scaled-down subgroup size, with the planner's measured
    B200 profile and the policy's stride, bit-exact against the oracle."""
    from paper_2410_21316_b200 import policy

    sg = 20_000
    total = (nsub - 1) * sg + int(tail * sg)
    prof = D.get_profile("b200-node")
    sizes = [sg] * (nsub - 1) + [int(tail * sg)]
    stride, _ = policy.choose_stride(prof, sizes, range(1, 7), 0.2)
    for ratio, k in ((0.0, stride), (0.2, stride), (0.0, D.optimal_stride(prof, nsub, sg).k)):
        opt = D.ShardedOptimizer.initialize(total, sg, seed=nsub, lowp="bf16")
        D.execute_plan(opt, D.build_plan(nsub, k, static_ratio=ratio), prof, HYPER)
        assert digest(opt) == oracle_digest(total, sg, nsub, "bf16"), (name, ratio, k)


@pytest.mark.parametrize("stride,ratio", [(2, 0.0), (3, 0.25), (D.ALL_CPU, 0.0), (1, 0.0)])
def test_in_phase_grad_flush(h100, stride, ratio):
    """flush_grads=True: the device grads are the only source; the host lane
    reads each subgroup's grads after its own in-phase D2H copy."""
    opt = D.ShardedOptimizer.initialize(60_000, 6_000, seed=21, lowp="bf16")
    want_g = opt.grads16.copy()
    res = opt.to_device()
    opt._g[:] = 0x7FC0  # poison the host image: only the in-phase flush can repair it
    plan = D.build_plan(10, stride, ratio)
    D.execute_plan(opt, plan, h100, HYPER, flush_grads=True)
    cpu = [sg for i, sg in enumerate(opt.subgroups) if plan.devices[i] is D.Device.CPU]
    for sg in cpu:
        assert opt.grads16[sg.slice].tobytes() == want_g[sg.slice].tobytes()
    ref = O.initialize(60_000, 6_000, 21, "bf16")
    O.sequential_oracle(ref)
    assert opt.params32.tobytes() == ref["p"].tobytes()
    assert opt.model16.tobytes() == ref["w"].tobytes()
    with pytest.raises(ValueError):
        D.execute_plan(opt, plan, h100, HYPER, flush_grads=True, host_io=True)
    assert res is opt.residency


@pytest.mark.parametrize("stride", [2, 3, D.ALL_CPU])
def test_unfused_cpu_downscale_matches(h100, stride):
    """fuse_downscale=False: CPU_DOWNSCALE does its own pass over each batch
    (the reference's separate action, executor.py:228-231)."""
    opt = D.ShardedOptimizer.initialize(50_000, 5_000, seed=31, lowp="fp16")
    D.execute_plan(opt, D.build_plan(10, stride, 0.2), h100, HYPER, fuse_downscale=False)
    assert digest(opt) == oracle_digest(50_000, 5_000, 31)


@pytest.mark.parametrize("host_io", [False, True])
def test_post_phase_coherence_is_asserted_by_default(h100, host_io):
    """The reference asserts model16 == downscale_rne(params32) after every
    phase (executor.py:271-282); so does execute_plan by default: a corrupted
    working copy of a static resident, of a host-homed subgroup at a sampled
    window, or (``"full"``) anywhere raises AssertionError."""
    from paper_2410_21316_b200.executor import COHERENCE_WINDOW, check_coherence_after_phase

    sg = 4 * COHERENCE_WINDOW * 16  # larger than the sample: "sampled" reads a part of each subgroup
    opt = D.ShardedOptimizer.initialize(6 * sg + 1234, sg, seed=17, lowp="bf16")
    plan = D.build_plan(7, 2, static_ratio=0.3, placement=Placement.STATIC_FIRST)
    D.execute_plan(opt, plan, h100, HYPER, host_io=host_io)  # coherent: passes with the default check
    res = opt.residency
    static = min(plan.static_set)
    host = next(i for i in range(7) if i not in plan.static_set)
    w = res.model16.view(torch.int16)
    check_coherence_after_phase(opt, res, "full", host_io)
    for sgi, off, modes in ((static, 12345, ("sampled", "full")),  # residents: always the whole subgroup
                            (host, 5, ("sampled", "full")),  # first window of a host-homed subgroup
                            (host, opt.subgroups[host].size - 1, ("sampled", "full")),  # last window
                            (host, 3 * COHERENCE_WINDOW // 2 + 7, ("full",))):  # between windows
        i = opt.subgroups[sgi].start + off
        keep = w[i].clone()
        w[i] ^= 1
        for mode in modes:
            with pytest.raises(AssertionError, match=f"subgroup {sgi}"):
                check_coherence_after_phase(opt, res, mode, host_io)
        if modes == ("full",):
            check_coherence_after_phase(opt, res, "sampled", host_io)
        w[i] = keep
    if host_io:  # the host mirror is checked too
        j = opt.subgroups[host].start + 3
        opt._w[j] ^= 1
        with pytest.raises(AssertionError, match="host model16 mirror"):
            check_coherence_after_phase(opt, res, "sampled", True)
        opt._w[j] ^= 1
    check_coherence_after_phase(opt, res, "full", host_io)
    # the host-side variant (for host arrays the device cannot read) agrees
    from paper_2410_21316_b200.executor import _coherence_on_host

    _coherence_on_host(opt, res, False, host_io)
    w[opt.subgroups[host].start] ^= 1
    with pytest.raises(AssertionError, match=f"subgroup {host}"):
        _coherence_on_host(opt, res, False, host_io)
    w[opt.subgroups[host].start] ^= 1
    with pytest.raises(ValueError):
        D.execute_plan(opt, plan, h100, HYPER, check_coherence="sometimes")
