"""Algorithm 1: device assignment and the action list.

Produces plans bit-identical to the reference's ``build_plan``
(pkg/src/optistate/scheduler.py:322-385): same ``devices``, ``static_set``,
``dynamic_fast`` and the same ``actions`` tuple (ids, kinds, lanes, streams,
batches, deps), so any UpdateTarget — simulator, reference executor or
``B200Target`` — sees the same program.

Interleaved plans put subgroup i on the fast tier iff it is a static
resident or ``(i + 1) % stride == 0``.  While a fast subgroup's state is in
flight the host walks the subgroups in between; a host slot with
``i % stride == 0`` (a cycle start) flushes the previous fast subgroup and
prefetches the next one.  Host-updated params collect in a downscale batch
that drains at the next fast slot, each member then shipping its
half-precision params to the device.  ``ALL_CPU`` plans are the serialized
baseline: every action depends on its predecessor.
"""

from __future__ import annotations

import bisect
import enum
import math
import warnings
from dataclasses import dataclass

from ._native import InfeasibleConfigError  # noqa: F401  (re-exported)
from .perfmodel import ALL_CPU, _AllCpuType


class Device(enum.Enum):
    CPU = "cpu"
    FAST = "fast"


class Lane(str, enum.Enum):
    CPU_COMPUTE = "cpu_compute"
    FAST_COMPUTE = "fast_compute"
    H2D = "h2d"
    D2H = "d2h"


COMPUTE_LANES = (Lane.CPU_COMPUTE, Lane.FAST_COMPUTE)


class Stream(str, enum.Enum):
    PARAM = "param"
    MOMENTUM = "momentum"
    VARIANCE = "variance"


class ActionKind(str, enum.Enum):
    CPU_UPDATE = "cpu_update"
    GPU_UPDATE = "gpu_update"
    CPU_DOWNSCALE = "cpu_downscale"
    H2D_PARAMS16 = "h2d_params16"
    FLUSH_OUT_MODEL16 = "flush_out_model16"
    FLUSH_OUT_M = "flush_out_m"
    FLUSH_OUT_V = "flush_out_v"
    FLUSH_OUT_P = "flush_out_p"
    PREFETCH_M = "prefetch_m"
    PREFETCH_V = "prefetch_v"
    PREFETCH_P = "prefetch_p"
    GRAD_FLUSH = "grad_flush"


# position in the enum == the C-ABI code (include/dos.h dos_action_kind)
KIND_CODE = {k: i for i, k in enumerate(ActionKind)}
LANE_CODE = {Lane.CPU_COMPUTE: 0, Lane.FAST_COMPUTE: 1, Lane.H2D: 2, Lane.D2H: 3}

PREFETCH_KINDS = (ActionKind.PREFETCH_M, ActionKind.PREFETCH_V, ActionKind.PREFETCH_P)
FLUSH_STATE_KINDS = (ActionKind.FLUSH_OUT_M, ActionKind.FLUSH_OUT_V, ActionKind.FLUSH_OUT_P)


class Placement(str, enum.Enum):
    STATIC_FIRST = "static_first"
    STATIC_LAST = "static_last"


@dataclass(frozen=True)
class Action:
    """One schedulable unit; ``subgroup == -1`` for a batched CPU_DOWNSCALE."""

    id: int
    kind: ActionKind
    subgroup: int
    lane: Lane
    stream: Stream | None = None
    batch: tuple[int, ...] = ()
    deps: tuple[int, ...] = ()


@dataclass(frozen=True)
class ScheduledAction:
    action: Action
    start_ns: int
    end_ns: int
    bytes: int

    @property
    def duration_ns(self) -> int:
        return self.end_ns - self.start_ns


@dataclass(frozen=True)
class UpdatePlan:
    num_subgroups: int
    stride: "int | _AllCpuType"
    static_ratio: float
    placement: Placement
    static_set: frozenset[int]
    devices: tuple[Device, ...]
    dynamic_fast: tuple[int, ...]
    blocking: bool
    actions: tuple[Action, ...]

    @property
    def static_count(self) -> int:
        return len(self.static_set)

    def device_of(self, subgroup: int) -> Device:
        return self.devices[subgroup]

    def is_static(self, subgroup: int) -> bool:
        return subgroup in self.static_set


def prev_on_gpu(plan: UpdatePlan, subgroup: int) -> int | None:
    """Closest dynamic fast subgroup strictly before ``subgroup``."""
    k = bisect.bisect_left(plan.dynamic_fast, subgroup)
    return plan.dynamic_fast[k - 1] if k else None


def next_on_gpu(plan: UpdatePlan, subgroup: int) -> int | None:
    """Closest dynamic fast subgroup strictly after ``subgroup``."""
    k = bisect.bisect_right(plan.dynamic_fast, subgroup)
    return plan.dynamic_fast[k] if k < len(plan.dynamic_fast) else None


def _pinned(num_subgroups: int, static_ratio: float, placement: Placement) -> frozenset[int]:
    # floor with a 1e-9 guard against one-ulp products (scheduler.py:161-168)
    count = min(num_subgroups, math.floor(static_ratio * num_subgroups + 1e-9))
    if placement is Placement.STATIC_FIRST:
        return frozenset(range(count))
    return frozenset(range(num_subgroups - count, num_subgroups))


class _ActionLog:
    """Append-only action list; ``serial`` chains each action to the last."""

    def __init__(self, serial: bool = False) -> None:
        self.items: list[Action] = []
        self.serial = serial

    def add(self, kind: ActionKind, sg: int, lane: Lane, stream: Stream | None = None,
            batch: tuple[int, ...] = (), deps: tuple[int, ...] = ()) -> int:
        if self.serial and self.items and self.items[-1].id not in deps:
            deps = (*deps, self.items[-1].id)
        aid = len(self.items)
        self.items.append(Action(aid, kind, sg, lane, stream, batch, deps))
        return aid


def _interleaved(n: int, stride: int, devices: tuple[Device, ...], dynamic: tuple[int, ...]) -> list[Action]:
    log = _ActionLog()
    dyn = frozenset(dynamic)
    updated: dict[int, int] = {}  # subgroup -> id of its update action
    fetched: dict[int, tuple[int, ...]] = {}  # subgroup -> ids of its three prefetches
    batch: list[int] = []  # host-updated subgroups awaiting downscale
    in_flight: int | None = None  # fast subgroup whose flush is deferred

    def fetch(sg: int) -> None:
        fetched[sg] = (
            log.add(ActionKind.PREFETCH_M, sg, Lane.H2D, Stream.MOMENTUM),
            log.add(ActionKind.PREFETCH_V, sg, Lane.H2D, Stream.VARIANCE),
            log.add(ActionKind.PREFETCH_P, sg, Lane.H2D, Stream.PARAM),
        )

    def flush(sg: int) -> None:
        after = (updated[sg],)
        log.add(ActionKind.FLUSH_OUT_MODEL16, sg, Lane.FAST_COMPUTE, Stream.PARAM, deps=after)
        log.add(ActionKind.FLUSH_OUT_M, sg, Lane.D2H, Stream.MOMENTUM, deps=after)
        log.add(ActionKind.FLUSH_OUT_V, sg, Lane.D2H, Stream.VARIANCE, deps=after)
        log.add(ActionKind.FLUSH_OUT_P, sg, Lane.D2H, Stream.PARAM, deps=after)

    def drain() -> None:
        if not batch:
            return
        members = tuple(batch)
        d = log.add(ActionKind.CPU_DOWNSCALE, -1, Lane.CPU_COMPUTE, batch=members,
                    deps=tuple(updated[j] for j in members))
        for j in members:
            log.add(ActionKind.H2D_PARAMS16, j, Lane.H2D, Stream.PARAM, deps=(d,))
        batch.clear()

    def following(i: int) -> int | None:
        k = bisect.bisect_right(dynamic, i)
        return dynamic[k] if k < len(dynamic) else None

    def cycle_start_between(lo: int, hi: int) -> bool:
        return any(devices[c] is Device.CPU and c % stride == 0 for c in range(lo + 1, hi))

    for i, dev in enumerate(devices):
        if dev is Device.CPU:
            if i % stride == 0:
                if in_flight is not None:
                    flush(in_flight)
                    in_flight = None
                nxt = following(i)
                if nxt is not None and nxt not in fetched:
                    fetch(nxt)
            updated[i] = log.add(ActionKind.CPU_UPDATE, i, Lane.CPU_COMPUTE)
            batch.append(i)
            continue
        drain()
        if i not in dyn:  # static resident: update in place, refresh the working copy
            updated[i] = log.add(ActionKind.GPU_UPDATE, i, Lane.FAST_COMPUTE)
            log.add(ActionKind.FLUSH_OUT_MODEL16, i, Lane.FAST_COMPUTE, Stream.PARAM, deps=(updated[i],))
            continue
        if i not in fetched:  # nothing pumped it (all-fast plan, or statics lead)
            fetch(i)
        updated[i] = log.add(ActionKind.GPU_UPDATE, i, Lane.FAST_COMPUTE, deps=fetched[i])
        in_flight = i
        nxt = following(i)
        if nxt is not None and not cycle_start_between(i, nxt):
            flush(i)
            in_flight = None
            if nxt not in fetched:
                fetch(nxt)
    if in_flight is not None:
        flush(in_flight)
    drain()
    return log.items


def _serialized(devices: tuple[Device, ...]) -> list[Action]:
    log = _ActionLog(serial=True)
    for i, dev in enumerate(devices):
        if dev is Device.FAST:
            u = log.add(ActionKind.GPU_UPDATE, i, Lane.FAST_COMPUTE)
            log.add(ActionKind.FLUSH_OUT_MODEL16, i, Lane.FAST_COMPUTE, Stream.PARAM, deps=(u,))
        else:
            u = log.add(ActionKind.CPU_UPDATE, i, Lane.CPU_COMPUTE)
            d = log.add(ActionKind.CPU_DOWNSCALE, -1, Lane.CPU_COMPUTE, batch=(i,), deps=(u,))
            log.add(ActionKind.H2D_PARAMS16, i, Lane.H2D, Stream.PARAM, deps=(d,))
    return log.items


def build_plan(num_subgroups: int, stride: "int | _AllCpuType", static_ratio: float = 0.0,
               placement: Placement = Placement.STATIC_LAST) -> UpdatePlan:
    """Assign devices and emit the phase's actions (scheduler.py:322-385)."""
    if num_subgroups < 0:
        raise ValueError("num_subgroups must be >= 0")
    if not 0.0 <= static_ratio <= 1.0:
        raise ValueError(f"static_ratio must be in [0, 1], got {static_ratio}")
    if stride is not ALL_CPU and (not isinstance(stride, int) or stride < 1):
        raise ValueError(f"stride must be an int >= 1 or ALL_CPU, got {stride!r}")
    statics = _pinned(num_subgroups, static_ratio, placement)
    blocking = stride is ALL_CPU
    if not blocking and num_subgroups > 0 and len(statics) == num_subgroups:
        warnings.warn("static_ratio pins every subgroup: the plan degenerates to all-static and the stride "
                      "never applies", UserWarning, stacklevel=2)
    devices = tuple(
        Device.FAST if (i in statics or (not blocking and (i + 1) % stride == 0)) else Device.CPU
        for i in range(num_subgroups)
    )
    dynamic = tuple(i for i, d in enumerate(devices) if d is Device.FAST and i not in statics)
    actions = _serialized(devices) if blocking else _interleaved(num_subgroups, stride, devices, dynamic)
    return UpdatePlan(
        num_subgroups=num_subgroups,
        stride=stride,
        static_ratio=static_ratio,
        placement=placement,
        static_set=statics,
        devices=devices,
        dynamic_fast=dynamic,
        blocking=blocking,
        actions=tuple(actions),
    )
