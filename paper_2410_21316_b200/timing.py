"""Profile-derived durations, timelines and the fast-tier memory trace.

Restates the update-phase part of pkg/src/optistate/sim.py (SimTarget
:64-133, Timeline/_build_timeline :136-171, simulate_update_phase :174-183,
memory_trace :186-223 and the grad-flush rate model :226-268) with identical
integer-ns arithmetic, so predicted timelines match the reference's frozen
makespans exactly.  The reference's offline analysis drivers (sweep_stride,
simulate_iteration, compare_approaches, sim.py:271-550) are out of scope.

Makespan is the last end over the compute lanes; transfers after it (the
final half-precision H2D) are ``spillover``.  The B200 report states both
makespan and span, because the next iteration needs the last H2D.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass
from typing import Iterable, Sequence

from .engine import run_update, validate_schedule
from .perfmodel import ALL_CPU
from .plan import COMPUTE_LANES, Action, ActionKind, Lane, ScheduledAction, UpdatePlan
from .state import (
    GRADS16_BYTES_PER_PARAM,
    MODEL16_BYTES_PER_PARAM,
    SUBGROUP_STATE_BYTES_PER_PARAM,
    SystemProfile,
)

_STATE_MOVES = frozenset({
    ActionKind.PREFETCH_M, ActionKind.PREFETCH_V, ActionKind.PREFETCH_P,
    ActionKind.FLUSH_OUT_M, ActionKind.FLUSH_OUT_V, ActionKind.FLUSH_OUT_P,
})


def kind_of(action) -> ActionKind:
    """The action's kind as this package's enum — also for Action objects
    built by the reference package (same string values, another enum class)."""
    k = action.kind
    return k if type(k) is ActionKind else ActionKind(k.value)


def normalize_sizes(plan: UpdatePlan, subgroup_size: "int | Sequence[int]") -> tuple[int, ...]:
    if isinstance(subgroup_size, int):
        return (subgroup_size,) * plan.num_subgroups
    sizes = tuple(int(s) for s in subgroup_size)
    if len(sizes) != plan.num_subgroups:
        raise ValueError(f"got {len(sizes)} subgroup sizes for {plan.num_subgroups} subgroups")
    return sizes


def ceil_ns(seconds: float) -> int:
    return math.ceil(seconds * 1e9)


class SimTarget:
    """Timing-only UpdateTarget: durations and bytes from a profile."""

    def __init__(self, profile: SystemProfile, plan: UpdatePlan, subgroup_size: "int | Sequence[int]") -> None:
        self.profile = profile
        self.plan = plan
        self.sizes = normalize_sizes(plan, subgroup_size)
        self.fast_capacity_bytes = profile.fast_capacity_bytes
        # host work only contends with link traffic when the plan overlaps them
        self._cpu_scale = 1.0 if plan.blocking else profile.host_contention

    def _params(self, a: Action) -> int:
        if kind_of(a) is ActionKind.CPU_DOWNSCALE:
            return sum(self.sizes[j] for j in a.batch)
        return self.sizes[a.subgroup]

    def duration_ns(self, action: Action) -> int:
        p, s, k = self.profile, self._params(action), kind_of(action)
        if k is ActionKind.CPU_UPDATE:
            return ceil_ns(s / p.cpu_update_params_per_s * self._cpu_scale)
        if k is ActionKind.GPU_UPDATE:
            return ceil_ns(s / p.fast_update_params_per_s)
        if k is ActionKind.CPU_DOWNSCALE:
            return ceil_ns(s / p.cpu_downscale_params_per_s * self._cpu_scale)
        if k in _STATE_MOVES:
            return ceil_ns(s / p.channel_params_per_s)
        if k is ActionKind.H2D_PARAMS16:
            return ceil_ns(s / (2.0 * p.channel_params_per_s))
        if k is ActionKind.FLUSH_OUT_MODEL16:
            return ceil_ns(MODEL16_BYTES_PER_PARAM * s / p.fast_convert_bytes_per_s)
        raise ValueError(f"unexpected action kind in update plan: {k}")

    def bytes_of(self, action: Action) -> int:
        """Algorithmic link bytes: 4 B/param per fp32 piece, 2 B for halves."""
        k = kind_of(action)
        if k in _STATE_MOVES:
            return 4 * self._params(action)
        if k in (ActionKind.H2D_PARAMS16, ActionKind.FLUSH_OUT_MODEL16):
            return 2 * self._params(action)
        return 0

    def window_bytes(self, subgroup: int) -> int:
        return SUBGROUP_STATE_BYTES_PER_PARAM * self.sizes[subgroup]

    def apply(self, action: Action, start_ns: int, end_ns: int) -> None:
        return None


@dataclass(frozen=True)
class Timeline:
    events: tuple[ScheduledAction, ...]
    makespan_ns: int
    span_ns: int
    spillover_ns: int
    peak_fast_bytes: int
    lane_busy_ns: dict[Lane, int]

    def makespan_per_subgroup(self, num_subgroups: int) -> float:
        return self.makespan_ns / num_subgroups if num_subgroups else 0.0


def build_timeline(plan: UpdatePlan, events: tuple[ScheduledAction, ...], sizes: tuple[int, ...]) -> Timeline:
    busy = dict.fromkeys(Lane, 0)
    span = makespan = 0
    for ev in events:
        busy[ev.action.lane] += ev.duration_ns
        span = max(span, ev.end_ns)
        if ev.action.lane in COMPUTE_LANES:
            makespan = max(makespan, ev.end_ns)
    peak = max((level for _, level in memory_trace(events, plan, sizes)), default=0)
    return Timeline(events=events, makespan_ns=makespan, span_ns=span, spillover_ns=span - makespan,
                    peak_fast_bytes=peak, lane_busy_ns=busy)


def simulate_update_phase(plan: UpdatePlan, profile: SystemProfile,
                          subgroup_size: "int | Sequence[int]") -> Timeline:
    target = SimTarget(profile, plan, subgroup_size)
    events = run_update(plan, target)
    validate_schedule(plan, events, target)
    return build_timeline(plan, events, target.sizes)


def memory_trace(events: Iterable[ScheduledAction], plan: UpdatePlan,
                 subgroup_size: "int | Sequence[int]") -> list[tuple[int, int]]:
    """Fast-tier bytes over time: lowp model + grads for the whole shard,
    static residents' fp32 state, and each dynamic window from its
    PREFETCH_M start to its FLUSH_OUT_P end."""
    sizes = normalize_sizes(plan, subgroup_size)
    level = (MODEL16_BYTES_PER_PARAM + GRADS16_BYTES_PER_PARAM) * sum(sizes)
    level += sum(SUBGROUP_STATE_BYTES_PER_PARAM * sizes[i] for i in plan.static_set)
    steps: dict[int, int] = {0: 0}
    started: dict[int, int] = {}
    for ev in events:
        a = ev.action
        if a.kind is ActionKind.PREFETCH_M:
            started[a.subgroup] = ev.start_ns
        elif a.kind is ActionKind.FLUSH_OUT_P:
            w = SUBGROUP_STATE_BYTES_PER_PARAM * sizes[a.subgroup]
            t0 = started.pop(a.subgroup)
            steps[t0] = steps.get(t0, 0) + w
            steps[ev.end_ns] = steps.get(ev.end_ns, 0) - w
    if started:
        raise AssertionError(f"unclosed residency windows: {sorted(started)}")
    trace = []
    for t in sorted(steps):
        level += steps[t]
        trace.append((t, level))
    return trace


TRACE_HEADER = ("event_id", "lane", "kind", "subgroup", "start_ns", "end_ns", "bytes")


def write_trace_csv(timeline: Timeline, stream) -> None:
    """Timeline as CSV in the reference's trace schema (cli.py:49,250-264);
    works for predicted and measured timelines alike."""
    import csv

    w = csv.writer(stream)
    w.writerow(TRACE_HEADER)
    for ev in timeline.events:
        a = ev.action
        w.writerow((a.id, a.lane.value, a.kind.value, a.subgroup, ev.start_ns, ev.end_ns, ev.bytes))


class GradFlushStrategy(str, enum.Enum):
    """How half-precision grads reach the host as fp32 (sim.py:226-243)."""

    FP16_HOST_UPSCALE = "fp16_host_upscale"
    GPU_UPSCALE_FP32 = "gpu_upscale_fp32"


def grad_flush_throughput(strategy: GradFlushStrategy, profile: SystemProfile,
                          grad_bytes: int | None = None) -> float:
    """Effective flush rate in half-precision payload bytes/s (size-free)."""
    del grad_bytes
    if strategy is GradFlushStrategy.FP16_HOST_UPSCALE:
        return 1.0 / (1.0 / profile.host_alloc_bytes_per_s + 1.0 / profile.pageable_d2h_bytes_per_s
                      + 1.0 / profile.host_convert_bytes_per_s)
    if strategy is GradFlushStrategy.GPU_UPSCALE_FP32:
        pinned = 4.0 * profile.channel_params_per_s
        return 1.0 / (1.0 / profile.fast_convert_bytes_per_s + 2.0 / pinned)
    raise ValueError(f"unknown strategy {strategy!r}")


__all__ = [
    "ALL_CPU", "GradFlushStrategy", "SimTarget", "Timeline", "build_timeline",
    "grad_flush_throughput", "memory_trace", "normalize_sizes", "simulate_update_phase",
    "GRADS16_BYTES_PER_PARAM",
]
