"""The list-scheduling engine and the plugin seam (``UpdateTarget``).

``run_update(plan, target)`` serves a plan exactly like the reference
(pkg/src/optistate/scheduler.py:402-466): every action starts at the
earliest time allowed by its dependencies, its lane's FIFO, its state
stream's FIFO and — for a dynamic subgroup's window-opening PREFETCH_M —
the fast-tier capacity gate; ``target.apply`` is called once per action in
emission order after its interval is fixed.  Durations come from the
target, so the same engine yields the simulator's prediction and drives
``B200Target``, whose ``apply`` enqueues the real work without waiting.

``validate_schedule`` is the reference's structural audit
(scheduler.py:484-591).  It runs on predicted timelines unchanged, and on
*measured* B200 timelines with ``check_streams=False`` (the B200 stages
windows in separate HBM slots, so the one-buffer-per-stream FIFO of the
model is intentionally not a hardware constraint) and ``max_windows`` set
to the number of physical slots.
"""

from __future__ import annotations

from typing import Iterable, Protocol

from ._native import InfeasibleConfigError
from .plan import (
    FLUSH_STATE_KINDS,
    PREFETCH_KINDS,
    Action,
    ActionKind,
    Device,
    Lane,
    ScheduledAction,
    Stream,
    UpdatePlan,
)


class UpdateTarget(Protocol):
    """Duration / side-effect provider driven by ``run_update``."""

    fast_capacity_bytes: int | None

    def duration_ns(self, action: Action) -> int: ...

    def bytes_of(self, action: Action) -> int: ...

    def window_bytes(self, subgroup: int) -> int: ...

    def apply(self, action: Action, start_ns: int, end_ns: int) -> None: ...


def _gate(t0: int, need: int, capacity: int, closed: list[tuple[int, int]]) -> int:
    """Earliest t >= t0 where windows still open at t plus ``need`` fit."""
    for t in [t0, *sorted(c for c, _ in closed if c > t0)]:
        if sum(b for c, b in closed if c > t) + need <= capacity:
            return t
    raise InfeasibleConfigError(f"capacity gate cannot admit a {need} B window within {capacity} B")


def run_update(plan: UpdatePlan, target: UpdateTarget) -> tuple[ScheduledAction, ...]:
    capacity = target.fast_capacity_bytes
    dynamic = set(plan.dynamic_fast)
    if capacity is not None and dynamic:
        worst = max(target.window_bytes(sg) for sg in dynamic)
        if worst > capacity:
            raise InfeasibleConfigError(
                f"fast tier capacity {capacity} B cannot hold one in-flight subgroup window of {worst} B")
    lane_free = dict.fromkeys(Lane, 0)
    stream_free = dict.fromkeys(Stream, 0)
    finish: list[int] = []
    closed: list[tuple[int, int]] = []  # (close time, bytes) of windows whose flush is scheduled
    opened: set[int] = set()
    out: list[ScheduledAction] = []
    for a in plan.actions:
        t = max([lane_free[a.lane], *(finish[d] for d in a.deps)])
        if a.stream is not None:
            t = max(t, stream_free[a.stream])
        if capacity is not None and a.kind is ActionKind.PREFETCH_M and a.subgroup in dynamic:
            t = _gate(t, target.window_bytes(a.subgroup), capacity, closed)
            opened.add(a.subgroup)
        end = t + target.duration_ns(a)
        finish.append(end)
        lane_free[a.lane] = end
        if a.stream is not None:
            stream_free[a.stream] = end
        if a.kind is ActionKind.FLUSH_OUT_P and a.subgroup in opened:
            opened.discard(a.subgroup)
            closed.append((end, target.window_bytes(a.subgroup)))
        out.append(ScheduledAction(action=a, start_ns=t, end_ns=end, bytes=target.bytes_of(a)))
        target.apply(a, t, end)
    return tuple(out)


def validate_schedule(plan: UpdatePlan, schedule: Iterable[ScheduledAction], target: UpdateTarget, *,
                      check_streams: bool = True, max_windows: int = 2, tolerance_ns: int = 0) -> None:
    """Structural audit; raises AssertionError (scheduler.py:484-591).

    ``tolerance_ns`` relaxes dependency edges only; it exists for measured
    timelines whose host and device events come from two clocks.
    """
    events = list(schedule)
    by_id = {ev.action.id: ev for ev in events}
    lane_last: dict[Lane, ScheduledAction] = {}
    stream_last: dict[Stream, ScheduledAction] = {}
    for ev in events:
        a = ev.action
        assert 0 <= ev.start_ns <= ev.end_ns, f"bad interval on action {a.id}"
        prev = lane_last.get(a.lane)
        assert prev is None or ev.start_ns >= prev.end_ns, (
            f"lane {a.lane.value} overlap: action {a.id} starts at {ev.start_ns} before {prev.action.id} "
            f"ends {prev.end_ns}")
        lane_last[a.lane] = ev
        if check_streams and a.stream is not None:
            sprev = stream_last.get(a.stream)
            assert sprev is None or ev.start_ns >= sprev.end_ns, (
                f"stream {a.stream.value} FIFO violated by action {a.id}")
            stream_last[a.stream] = ev
        for d in a.deps:
            assert by_id[d].end_ns <= ev.start_ns + tolerance_ns, f"action {a.id} starts before dep {d} ends"

    n_updates: dict[int, int] = {}
    n_down: dict[int, int] = {}
    kinds: dict[int, list[ActionKind]] = {}
    for ev in events:
        a = ev.action
        if a.kind in (ActionKind.CPU_UPDATE, ActionKind.GPU_UPDATE):
            n_updates[a.subgroup] = n_updates.get(a.subgroup, 0) + 1
        if a.kind is ActionKind.CPU_DOWNSCALE:
            for j in a.batch:
                n_down[j] = n_down.get(j, 0) + 1
        kinds.setdefault(a.subgroup, []).append(a.kind)
    for i in range(plan.num_subgroups):
        assert n_updates.get(i, 0) == 1, f"subgroup {i} has {n_updates.get(i, 0)} updates"
        ks = kinds.get(i, [])
        if plan.devices[i] is Device.CPU:
            assert n_down.get(i, 0) == 1, f"subgroup {i} missing downscale"
            assert ks.count(ActionKind.H2D_PARAMS16) == 1, f"subgroup {i} missing half-width params H2D"
            assert not any(k in PREFETCH_KINDS for k in ks), f"CPU subgroup {i} has prefetch actions"
        elif i in plan.static_set:
            assert ks.count(ActionKind.FLUSH_OUT_MODEL16) == 1
            assert not any(k in PREFETCH_KINDS or k in FLUSH_STATE_KINDS for k in ks), (
                f"static subgroup {i} moves optimizer state")
        else:
            for k in PREFETCH_KINDS + FLUSH_STATE_KINDS:
                assert ks.count(k) == 1, f"dynamic fast subgroup {i} missing {k.value}"
            assert ks.count(ActionKind.FLUSH_OUT_MODEL16) == 1

    open_at: dict[int, int] = {}
    close_at: dict[int, int] = {}
    upd: dict[int, ScheduledAction] = {}
    for ev in events:
        a = ev.action
        if a.kind is ActionKind.PREFETCH_M:
            open_at[a.subgroup] = ev.start_ns
        elif a.kind is ActionKind.FLUSH_OUT_P:
            close_at[a.subgroup] = ev.end_ns
        elif a.kind is ActionKind.GPU_UPDATE:
            upd[a.subgroup] = ev
    windows = []
    for sg, t0 in open_at.items():
        t1 = close_at.get(sg)
        assert t1 is not None and t1 > t0, f"window of subgroup {sg} never closes"
        windows.append((t0, t1, target.window_bytes(sg)))
        u = upd[sg]
        assert t0 <= u.start_ns and u.end_ns <= t1, f"fast update of subgroup {sg} escapes its residency window"
    if windows:
        cap = target.fast_capacity_bytes
        for t in sorted({x for t0, t1, _ in windows for x in (t0, t1)}):
            live = [w for w in windows if w[0] <= t < w[1]]
            assert len(live) <= max_windows, (
                f"{len(live)} dynamic windows overlap at t={t}; pipelining bound is {max_windows}")
            if cap is not None:
                used = sum(w[2] for w in live)
                assert used <= cap, f"dynamic window occupancy {used} exceeds capacity {cap} at t={t}"
