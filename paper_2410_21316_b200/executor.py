"""Step entry points of the update phase (reference: pkg/src/optistate/executor.py).

* ``execute_plan`` runs one optimizer step of a plan on the B200 and its host
  (``B200Target``): fast subgroups stream through HBM windows and K1, host
  subgroups run H1 on the host team, the half-precision working copy ends in
  HBM.  It returns the *predicted* timeline (identical to
  ``simulate_update_phase``, as the reference guarantees,
  pkg/tests/test_executor.py:79-86) and the *measured* one.
* ``sequential_oracle`` / ``adam_step_subgroup`` are the reference's plain
  in-order host update (executor.py:77-117), executed by H1.
* ``flush_gradients`` materialises fp32 grads on the host (executor.py:317-349).
"""

from __future__ import annotations

import ctypes as C
import enum
import math
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .device import B200Target
from .engine import run_update, validate_schedule
from .plan import UpdatePlan
from .state import GRADS16_BYTES_PER_PARAM, ShardedOptimizer, SystemProfile, bias_corrections, lowp_downscale
from .timing import GradFlushStrategy, Timeline, build_timeline, grad_flush_throughput

# Cross-clock slack when auditing measured timelines: host-lane events are
# stamped with the host clock aligned to the phase's t0 CUDA event, device
# events with the GPU clock.
MEASURED_CLOCK_SLACK_NS = 200_000


@dataclass(frozen=True)
class AdamHyper:
    """Adam hyperparameters (executor.py:45-56) plus optional decoupled
    weight decay (AdamW; no reference pin)."""

    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0

    def __post_init__(self) -> None:
        if not (0.0 <= self.beta1 < 1.0 and 0.0 <= self.beta2 < 1.0):
            raise ValueError("betas must be in [0, 1)")
        if self.lr <= 0 or self.eps <= 0:
            raise ValueError("lr and eps must be positive")
        if self.weight_decay < 0:
            raise ValueError("weight_decay must be >= 0")

    def scalars(self, step: int) -> N.dos_adam_scalars:
        bc1, bc2 = bias_corrections(self.beta1, self.beta2, step)
        return N.scalars(self.lr, self.beta1, self.beta2, self.eps, bc1, bc2, self.weight_decay)


class ExecMode(str, enum.Enum):
    VIRTUAL = "virtual"
    THROTTLED = "throttled"


def _host_update(opt: ShardedOptimizer, sg_index: int, hyper: AdamHyper, step: int, refresh_lowp: bool) -> None:
    sg = opt.subgroups[sg_index]
    a, n = sg.start, sg.size
    p, m, v, g, w = opt._p, opt._m, opt._v, opt._g, opt._w
    item16 = g.itemsize
    lp = N.ptr(w) + item16 * a if refresh_lowp else None
    sc = hyper.scalars(step)
    N.check(N.lib().dos_adam_step_host(N.ptr(p) + 4 * a, N.ptr(m) + 4 * a, N.ptr(v) + 4 * a, N.ptr(g) + item16 * a,
                                       opt.lowp_code, lp, opt.lowp_code if refresh_lowp else N.DOS_NONE, n, sc, 0))


def _host_authoritative(opt: ShardedOptimizer):
    res = opt.residency
    if res is not None:
        res.sync_all_host()
    return res


def adam_step_subgroup(optimizer: ShardedOptimizer, subgroup: int, hyper: AdamHyper, step: int | None = None) -> None:
    """Fused Adam on one subgroup's master state, in place, on the host.

    Grads are widened from the half-precision copy inside H1.  ``model16`` is
    left stale (the refresh is a separate action); the caller owns the step
    bump (executor.py:77-100).
    """
    res = _host_authoritative(optimizer)
    _host_update(optimizer, subgroup, hyper, optimizer.step + 1 if step is None else step, refresh_lowp=False)
    if res is not None:
        res.push_host()


def sequential_oracle(optimizer: ShardedOptimizer, hyper: AdamHyper) -> ShardedOptimizer:
    """Every subgroup in order on the host: Adam, then the working-copy
    refresh (fused into the same H1 pass); bumps ``step`` (executor.py:103-117)."""
    res = _host_authoritative(optimizer)
    step = optimizer.step + 1
    for sg in optimizer.subgroups:
        _host_update(optimizer, sg.index, hyper, step, refresh_lowp=True)
    optimizer.step = step
    if res is not None:
        res.push_host()
    return optimizer


class EmulatedDevice:
    """Structural staging ledger (executor.py:120-171): double stages,
    incomplete triplets and undrained windows are schedule bugs.  The native
    engine enforces the same rules on the real HBM slots; this class keeps
    the reference's pure-Python form for planners and tests."""

    PIECES = ("m", "v", "p")

    def __init__(self) -> None:
        self.staging: dict[int, dict[str, np.ndarray]] = {}
        self.model16_valid: set[int] = set()

    def stage(self, subgroup: int, piece: str, data: np.ndarray) -> None:
        slot = self.staging.setdefault(subgroup, {})
        if piece in slot:
            raise AssertionError(f"subgroup {subgroup} piece {piece!r} staged twice")
        slot[piece] = data

    def staged(self, subgroup: int, piece: str) -> np.ndarray:
        slot = self.staging.get(subgroup, {})
        if piece not in slot:
            raise AssertionError(f"subgroup {subgroup} piece {piece!r} not resident on device")
        return slot[piece]

    def require_triplet(self, subgroup: int) -> dict[str, np.ndarray]:
        slot = self.staging.get(subgroup, {})
        missing = [p for p in self.PIECES if p not in slot]
        if missing:
            raise AssertionError(f"fast update of subgroup {subgroup} with missing pieces {missing}")
        return slot

    def unstage(self, subgroup: int, piece: str) -> np.ndarray:
        data = self.staged(subgroup, piece)
        slot = self.staging[subgroup]
        del slot[piece]
        if not slot:
            del self.staging[subgroup]
        return data

    def assert_drained(self) -> None:
        if self.staging:
            raise AssertionError(f"staging store not drained: subgroups {sorted(self.staging)}")


@dataclass(frozen=True)
class ExecutionResult:
    optimizer: ShardedOptimizer
    timeline: Timeline  # predicted (== simulate_update_phase of the same plan/profile/sizes)
    step: int
    mode: ExecMode
    measured: Timeline | None = None  # wall-clock timeline of the B200 run


def _under_profiler() -> bool:
    """Nsight Compute (ncu) injects itself through CUDA_INJECTION64_PATH and
    replays each kernel: CUDA-event timestamps around a replayed kernel are
    not a timeline, so the measured-timeline audit is skipped under it (the
    numeric results are unaffected; ncu runs are never timing runs)."""
    import os

    return bool(os.environ.get("CUDA_INJECTION64_PATH")) or any(k.startswith("NV_NSIGHT") for k in os.environ)


def execute_plan(
    optimizer: ShardedOptimizer,
    plan: UpdatePlan,
    profile: SystemProfile,
    hyper: AdamHyper,
    mode: ExecMode = ExecMode.VIRTUAL,
    throttle_scale: float = 1e-3,
    *,
    host_threads: int = 0,
    host_io: bool = False,
    check_coherence: bool | str = "sampled",
    validate_measured: bool = True,
    on_submitted=None,
    peers=None,
    flush_grads: bool = False,
    fuse_downscale: bool = True,
    grad_sources=None,
) -> ExecutionResult:
    """Run one optimizer step of ``plan`` on the B200; mutates ``optimizer``.

    Same contract as executor.py:246-293: raises ValueError on a plan/shard
    size mismatch, audits the schedule, requires the staging windows to
    drain, bumps ``step``, and asserts — as the reference always does
    (executor.py:271-282) — that every subgroup's working copy equals the
    downscaled fp32 params (``check_coherence_after_phase``; AssertionError
    otherwise).  ``check_coherence``: ``"sampled"`` (default: HBM-homed
    state compared in full on the device, host-homed state in evenly spread
    windows of every subgroup read over the link), ``"full"`` / ``True``
    (every element of every subgroup), ``"off"`` / ``False``.

    ``host_io=True`` is the host-buffer mode: this step's gradients are read
    from the host image (``grads16``) for every subgroup — fast subgroups
    ship theirs H2D inside their prefetch — and the working copy is mirrored
    into the host ``model16`` inside the flushes, so both host images are
    coherent when the call returns.

    ``flush_grads=True`` moves the gradient flush into
    the phase: the device grads of each host-updated subgroup are copied D2H
    on their own stream in subgroup order and each CPU_UPDATE waits only for
    its own subgroup (the upcast stays fused in H1).  ``peers`` enables the
    fused all-gather (``distributed.PeerTargets``); ``grad_sources`` (a
    ``distributed.GradSources``, with ``flush_grads=True``) the fused
    reduce-scatter: this step's grads are the rank-order sum of every rank's
    grads for this shard, reduced inside K1 (fast subgroups) or right before
    the flush (host subgroups) and left in the device grads like a
    reduce-scatter would.  ``on_submitted(target)`` runs after the last
    submit, before the wait.
    """
    if plan.num_subgroups != len(optimizer.subgroups):
        raise ValueError(f"plan covers {plan.num_subgroups} subgroups, optimizer has {len(optimizer.subgroups)}")
    if mode is ExecMode.THROTTLED and throttle_scale <= 0:
        raise ValueError("throttle_scale must be positive")
    coherence = _coherence_mode(check_coherence)
    step = optimizer.step + 1
    target = B200Target(profile, plan, optimizer, hyper, step, host_threads=host_threads, host_io=host_io,
                        peers=peers, flush_grads=flush_grads, fuse_downscale=fuse_downscale,
                        grad_sources=grad_sources)
    sizes = target.sizes
    try:
        events = run_update(plan, target)
        if on_submitted is not None:  # e.g. chain per-subgroup collectives onto engine events
            on_submitted(target)
        # the predicted timeline's audit and summary need no device results:
        # done while the phase runs
        validate_schedule(plan, events, target)
        timeline = build_timeline(plan, events, sizes)
    except BaseException:
        target.finish(raise_errors=False)
        raise
    measured_events = target.finish()
    target.residency.after_phase(host_io, flush_grads)
    measured = build_timeline(plan, measured_events, sizes) if measured_events else None
    if validate_measured and measured_events and not _under_profiler():
        validate_schedule(plan, measured_events, target, check_streams=False, max_windows=target.num_slots,
                          tolerance_ns=MEASURED_CLOCK_SLACK_NS)
    optimizer.step = step
    check_coherence_after_phase(optimizer, target.residency, coherence, host_io)
    if mode is ExecMode.THROTTLED:
        _pace_replay(timeline, throttle_scale)
    return ExecutionResult(optimizer=optimizer, timeline=timeline, step=step, mode=mode, measured=measured)


# host-homed subgroups: this many windows of this many elements each, spread
# from the first element to the last (ragged tails included), per subgroup
COHERENCE_WINDOW = 2048
COHERENCE_WINDOWS = 16
COHERENCE_FULL_WINDOW = 1 << 16  # whole-subgroup checks: one CTA per 64K elements


def _coherence_mode(check) -> str:
    if check is True:
        return "full"
    if check is False or check is None:
        return "off"
    if check not in ("full", "sampled", "off"):
        raise ValueError(f"check_coherence must be 'sampled', 'full', 'off' or a bool, got {check!r}")
    return check


def check_coherence_after_phase(opt: ShardedOptimizer, res, mode: str = "sampled", host_io: bool = False) -> None:
    """The reference's post-phase assertion (executor.py:271-282): for every
    subgroup, model16 == downscale_rne(params32), bit for bit, else
    AssertionError naming the first incoherent subgroup.

    One device kernel (``dos_coherence_cuda``) reads each subgroup where its
    state lives: the authoritative working copy in HBM against the fp32
    params in HBM (static residents: always the whole subgroup, 6 B/param at
    HBM speed) or in the pinned host pool (everyone else, read over the
    link: sampled windows, or everything in ``"full"`` mode).  With
    ``host_io`` the host ``model16`` mirror is checked against the host
    params the same way.  Host arrays the device cannot read (plain,
    unregistered numpy memory) are compared on the host instead."""
    if mode == "off":
        return
    torch = __import__("torch")
    full = mode == "full"
    lowp = opt.lowp_code
    w_dev = res.model16
    esz = w_dev.element_size()
    ranges, names = [], []

    def add(p_ptr: int, w_ptr: int, n: int, whole: bool, what: str):
        win = COHERENCE_FULL_WINDOW if whole else COHERENCE_WINDOW
        nwin = -(-n // win) if whole else COHERENCE_WINDOWS
        ranges.append(N.dos_coh_range(p_ptr, w_ptr, n, win, nwin))
        names.append(what)

    for sg in opt.subgroups:
        w_ptr = w_dev.data_ptr() + sg.start * esz
        if sg.index in res.static_sg:
            add(res.static_sg[sg.index][0].data_ptr(), w_ptr, sg.size, True, f"subgroup {sg.index}")
        else:
            add(opt._p.ctypes.data + 4 * sg.start, w_ptr, sg.size, full, f"subgroup {sg.index}")
            if host_io:
                add(opt._p.ctypes.data + 4 * sg.start, opt._w.ctypes.data + 2 * sg.start, sg.size, full,
                    f"subgroup {sg.index} (host model16 mirror)")
    if not ranges:
        return
    arr = (N.dos_coh_range * len(ranges))(*ranges)
    with torch.cuda.device(res.device):
        out = torch.tensor([0, -1], dtype=torch.int64, device=res.device)
        stream = torch.cuda.current_stream(res.device)
        rc = N.lib().dos_coherence_cuda(arr, len(ranges), lowp,
                                        C.cast(out.data_ptr(), C.POINTER(C.c_ulonglong)), stream.cuda_stream)
        if rc == N.DOS_EINVAL and b"device-accessible" in N.lib().dos_last_error():
            return _coherence_on_host(opt, res, full, host_io)
        N.check(rc)
        bad, key = (int(x) for x in out.cpu().tolist())
    if bad:
        key &= (1 << 64) - 1
        r, i = key >> 40, key & ((1 << 40) - 1)
        raise AssertionError(f"model16 of {names[r]} incoherent with params32 ({bad} elements checked differ, "
                             f"first at offset {i})")


def _coherence_on_host(opt: ShardedOptimizer, res, full: bool, host_io: bool) -> None:
    torch = __import__("torch")
    i16 = res.model16.view(torch.int16)
    for sg in opt.subgroups:
        if sg.index in res.static_sg:
            p = res.static_sg[sg.index][0].cpu().numpy()
            sel = slice(0, sg.size)
        else:
            p = opt._p[sg.slice]
            if full or sg.size <= COHERENCE_WINDOW * COHERENCE_WINDOWS:
                sel = slice(0, sg.size)
            else:  # the device kernel's sample: first, last and evenly spread windows
                starts = [k * (sg.size - COHERENCE_WINDOW) // (COHERENCE_WINDOWS - 1) for k in range(COHERENCE_WINDOWS)]
                sel = np.concatenate([np.arange(a, a + COHERENCE_WINDOW) for a in starts])
        want = lowp_downscale(np.ascontiguousarray(p[sel]), opt.lowp).view(np.int16)
        idx = torch.as_tensor(np.arange(sg.size)[sel] + sg.start, device=res.device)
        got = i16[idx].cpu().numpy()
        mirrors = [("", got)]
        if host_io and sg.index not in res.static_sg:
            mirrors.append((" (host model16 mirror)", opt._w[sg.slice][sel].view(np.int16)))
        for tag, have in mirrors:
            if want.tobytes() != np.ascontiguousarray(have).tobytes():
                raise AssertionError(f"model16 of subgroup {sg.index}{tag} incoherent with params32")


def _pace_replay(timeline: Timeline, scale: float) -> None:
    if scale <= 0:
        raise ValueError("throttle_scale must be positive")
    t0 = time.perf_counter()
    for ev in sorted(timeline.events, key=lambda e: e.start_ns):
        wait = t0 + ev.start_ns * 1e-9 * scale - time.perf_counter()
        if wait > 0:
            time.sleep(wait)


@dataclass(frozen=True)
class GradFlushRecord:
    strategy: GradFlushStrategy
    payload_bytes: int
    chunk_bytes: int
    throughput_bytes_per_s: float
    cost_ns: int


def flush_gradients(optimizer: ShardedOptimizer, profile: SystemProfile, strategy: GradFlushStrategy,
                    chunk_bytes: int = 1 << 22) -> tuple[np.ndarray, GradFlushRecord]:
    """fp32 host gradients plus the modelled cost of the strategy.

    Numerically the exact widening of the half-precision grads, identical for
    every strategy and chunk size (executor.py:317-349).  With a B200
    residency the GPU_UPSCALE_FP32 leg runs on the device (dos_upscale_cuda)
    followed by a pinned D2H; otherwise H1 widens the host image.
    """
    if chunk_bytes < 2:
        raise ValueError("chunk_bytes must hold at least one fp16 element")
    P = optimizer.total_params
    elems = chunk_bytes // 2
    res = optimizer.residency
    if res is not None and strategy is GradFlushStrategy.GPU_UPSCALE_FP32:
        # chunk-wise on-device upcast double-buffered against
        # the pinned fp32 D2H: chunk k+1 converts while chunk k crosses the link
        import torch

        from .state import pinned_empty

        out = pinned_empty(P, np.float32)
        host = torch.from_numpy(out)
        n_buf = min(elems, P)
        bufs = [torch.empty(n_buf, dtype=torch.float32, device=res.device) for _ in range(2)]
        conv = torch.cuda.current_stream(res.device)
        copy = torch.cuda.Stream(device=res.device)
        done = [None, None]
        for k, lo in enumerate(range(0, P, elems)):
            hi = min(lo + elems, P)
            b = bufs[k % 2]
            if done[k % 2] is not None:
                conv.wait_event(done[k % 2])  # the D2H that last read this buffer has finished
            N.check(N.lib().dos_upscale_cuda(res.grads.data_ptr() + 2 * lo, optimizer.lowp_code, b.data_ptr(),
                                             hi - lo, conv.cuda_stream))
            copy.wait_stream(conv)
            with torch.cuda.stream(copy):
                host[lo:hi].copy_(b[:hi - lo], non_blocking=True)
                done[k % 2] = torch.cuda.Event()
                done[k % 2].record(copy)
        copy.synchronize()
    else:
        g = optimizer.grads16
        out = np.empty(P, dtype=np.float32)
        for lo in range(0, P, elems):
            hi = min(lo + elems, P)
            N.check(N.lib().dos_upscale_host(N.ptr(g) + 2 * lo, optimizer.lowp_code, N.ptr(out) + 4 * lo, hi - lo, 0))
    payload = GRADS16_BYTES_PER_PARAM * P
    rate = grad_flush_throughput(strategy, profile, payload)
    rec = GradFlushRecord(strategy=strategy, payload_bytes=payload, chunk_bytes=chunk_bytes,
                          throughput_bytes_per_s=rate, cost_ns=math.ceil(payload / rate * 1e9))
    return out, rec
