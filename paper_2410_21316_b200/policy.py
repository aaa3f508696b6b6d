"""Per-iteration re-fit of the performance model and the B200 stride policy.

The reference's planner (``optimal_stride``, perfmodel.py:155-179) is kept
bit-identical in ``perfmodel``; this module adds what the north star asks of
the B200 build: constants re-derived from the *measured* timeline of the
previous iteration, and a split chosen per iteration.

``simulate_b200_phase`` is the reference list scheduler (scheduler.py:
402-466) with the two rules the B200 engine changes: state streams are not
FIFO across directions (each in-flight window has its own HBM slot), and a
window opens only when the window ``num_slots`` earlier has fully flushed.
FLUSH_OUT_MODEL16 and CPU_DOWNSCALE cost nothing (fused into K1 / H1).
``choose_stride`` takes the candidate with the smallest predicted span.
"""

from __future__ import annotations

import dataclasses
from typing import Iterable, Sequence

from .perfmodel import ALL_CPU
from .plan import ActionKind, Device, Lane, Placement, ScheduledAction, UpdatePlan, build_plan
from .state import SystemProfile
from .timing import SimTarget, Timeline, build_timeline, normalize_sizes

_H2D_STATE = (ActionKind.PREFETCH_M, ActionKind.PREFETCH_V, ActionKind.PREFETCH_P)
_D2H_STATE = (ActionKind.FLUSH_OUT_M, ActionKind.FLUSH_OUT_V, ActionKind.FLUSH_OUT_P)


def refit_profile(profile: SystemProfile, measured: Timeline, sizes: Sequence[int]) -> SystemProfile:
    """Rates observed in a measured phase, folded into ``profile``.

    link: bytes / busy time of each direction's fp32 state copies (slower
    direction); K1: params / GPU_UPDATE time; host: params / CPU_UPDATE time,
    which was measured *under* link traffic, so the uncontended rate stored
    is that times ``host_contention``.
    """
    acc = {"h2d": [0, 0], "d2h": [0, 0], "gpu": [0, 0], "cpu": [0, 0]}
    for ev in measured.events:
        a, d = ev.action, ev.duration_ns
        if d <= 0:
            continue
        if a.kind in _H2D_STATE:
            acc["h2d"][0] += sizes[a.subgroup]
            acc["h2d"][1] += d
        elif a.kind in _D2H_STATE:
            acc["d2h"][0] += sizes[a.subgroup]
            acc["d2h"][1] += d
        elif a.kind is ActionKind.GPU_UPDATE:
            acc["gpu"][0] += sizes[a.subgroup]
            acc["gpu"][1] += d
        elif a.kind is ActionKind.CPU_UPDATE:
            acc["cpu"][0] += sizes[a.subgroup]
            acc["cpu"][1] += d
    rate = {k: (n / (t * 1e-9) if t else None) for k, (n, t) in acc.items()}
    upd = {}
    links = [r for r in (rate["h2d"], rate["d2h"]) if r]
    if links:
        upd["channel_params_per_s"] = min(links)
    if rate["gpu"]:
        upd["fast_update_params_per_s"] = rate["gpu"]
    if rate["cpu"]:
        upd["cpu_update_params_per_s"] = rate["cpu"] * profile.host_contention
    return dataclasses.replace(profile, **upd)


def _quiet_plan(n: int, stride, static_ratio: float, placement: Placement = Placement.STATIC_LAST) -> UpdatePlan:
    """build_plan without the all-static warning (the policy sweeps ratios
    up to 1.0 on purpose; the stride is then irrelevant, not a mistake)."""
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return build_plan(n, stride, static_ratio=static_ratio, placement=placement)


_LINK_KINDS = frozenset({ActionKind.PREFETCH_M, ActionKind.PREFETCH_V, ActionKind.PREFETCH_P,
                         ActionKind.FLUSH_OUT_M, ActionKind.FLUSH_OUT_V, ActionKind.FLUSH_OUT_P,
                         ActionKind.H2D_PARAMS16})


class _B200Durations(SimTarget):
    """SimTarget durations with the B200's fused actions made free and the
    host link slowed while the host team competes for host DRAM.

    ``link_slowdown`` is the measured duplex-link ratio alone / under H1
    (profile_b200.measure_link_under_h1); it applies in proportion to the
    share of the plan's params the host updates (0 for an all-fast plan)."""

    def __init__(self, profile, plan, sizes, link_slowdown: float = 1.0) -> None:
        super().__init__(profile, plan, sizes)
        total = sum(self.sizes) or 1
        host = sum(s for i, s in enumerate(self.sizes) if plan.devices[i] is Device.CPU)
        self._link_scale = 1.0 + (max(1.0, link_slowdown) - 1.0) * host / total

    def duration_ns(self, action) -> int:
        if action.kind in (ActionKind.FLUSH_OUT_MODEL16, ActionKind.CPU_DOWNSCALE):
            return 0
        d = super().duration_ns(action)
        return int(d * self._link_scale) if action.kind in _LINK_KINDS else d


def simulate_b200_phase(plan: UpdatePlan, profile: SystemProfile, subgroup_size: "int | Sequence[int]",
                        num_slots: int = 2, link_slowdown: float = 1.0) -> Timeline:
    """Predicted timeline of ``plan`` on the B200 engine (see module doc)."""
    sizes = normalize_sizes(plan, subgroup_size)
    t = _B200Durations(profile, plan, sizes, link_slowdown)
    lane_free = dict.fromkeys(Lane, 0)
    finish: list[int] = []
    closes: list[int] = []  # window close times, in opening order
    window_of: dict[int, int] = {}  # subgroup -> index of its window in `closes`
    dyn = set(plan.dynamic_fast)
    out = []
    for a in plan.actions:
        start = max([lane_free[a.lane], *(finish[d] for d in a.deps)])
        if a.kind is ActionKind.PREFETCH_M and a.subgroup in dyn:
            opened = len(closes)
            if opened >= num_slots:  # the slot frees when the window num_slots back closes
                start = max(start, closes[opened - num_slots])
            closes.append(-1)  # filled at its FLUSH_OUT_P
            window_of[a.subgroup] = opened
        end = start + t.duration_ns(a)
        finish.append(end)
        lane_free[a.lane] = end
        if a.kind is ActionKind.FLUSH_OUT_P and a.subgroup in dyn:
            closes[window_of[a.subgroup]] = end
        out.append(ScheduledAction(action=a, start_ns=start, end_ns=end, bytes=t.bytes_of(a)))
    return build_timeline(plan, tuple(out), sizes)


def choose_stride(profile: SystemProfile, sizes: Sequence[int], candidates: Iterable = range(1, 7),
                  static_ratio: float = 0.0, num_slots: int = 2, link_slowdown: float = 1.0):
    """Stride with the smallest predicted B200 span; returns (stride, {stride: span_ns})."""
    n = len(sizes)
    spans = {}
    for k in candidates:
        plan = _quiet_plan(n, k, static_ratio)
        spans[k] = simulate_b200_phase(plan, profile, list(sizes), num_slots, link_slowdown).span_ns
    best = min(spans, key=lambda k: (spans[k], 0 if k is ALL_CPU else k))
    return best, spans


class StrideTuner:
    """Explore-then-exploit stride selection by *measured* phase time.

    Every optimizer step is a real step whatever the stride (all plans are
    bit-identical in effect), so exploration costs nothing in correctness:
    the first steps each try one candidate (model-predicted best first), the
    measured spans are kept, and from then on the fastest measured stride is
    used.  This captures what the closed-form and simulated models do not —
    on a host whose DRAM is shared by the H1 threads and the copy engines,
    host traffic slows the DMA (measured on the B200 box: 50 -> 29-35 GB/s).

    With ``hill_climb`` the exploration does not stop at the predicted
    candidates: while the fastest measured stride has an unmeasured
    neighbour (stride ± 1, within 1..number of subgroups), that neighbour is
    tried next, so the tuner ends on a measured local minimum even when the
    model's ranking is off by more than the explored set.  Decisions depend
    only on the recorded spans, so ranks that record the same (max-over-
    ranks) spans stay in lockstep.

    ``placement`` is the plan's static placement (scheduler.py:161-168).
    With host buffers (``execute_plan(host_io=True)``) the residents' grads
    stream in from the host at the start of the phase, so STATIC_FIRST lets
    their updates — and the working-copy D2H behind them — lead the fast lane
    instead of queueing behind the streamed subgroups' prefetches.
    """

    def __init__(self, profile: SystemProfile, sizes: Sequence[int], candidates: Iterable = range(1, 7),
                 static_ratio: float = 0.0, explore: int = 4, num_slots: int = 2,
                 link_slowdown: float = 1.0, hill_climb: bool = True,
                 placement: Placement = Placement.STATIC_LAST, refine: bool = True) -> None:
        self.sizes = list(sizes)
        self.static_ratio = static_ratio
        self.placement = placement
        best, spans = choose_stride(profile, self.sizes, candidates, static_ratio, num_slots, link_slowdown)
        ranked = sorted(spans, key=lambda k: spans[k])
        self.queue = ranked[:max(1, explore)]
        self.predicted = spans
        self.measured: dict = {}
        self.hill_climb = hill_climb
        self.refine = refine

    def next_stride(self):
        if self.queue:
            return self.queue[0]
        return min(self.measured, key=lambda k: self.measured[k])

    def record(self, stride, span_ns: int) -> None:
        self.measured[stride] = min(span_ns, self.measured.get(stride, span_ns))
        if self.queue and self.queue[0] == stride:
            self.queue.pop(0)
        if self.hill_climb and not self.queue:
            best = min(self.measured, key=lambda k: self.measured[k])
            if best is not ALL_CPU:
                top = max(1, len(self.sizes))
                self.queue = [k for k in (best + 1, best - 1) if 1 <= k <= top and k not in self.measured][:1]
        if not self.queue and self.refine and len(self.measured) > 1:
            # one more sample of the two fastest (spans are kept as the min
            # over samples), so a single noisy step does not pick the stride
            self.refine = False
            self.queue = sorted(self.measured, key=lambda k: self.measured[k])[:2]

    @property
    def exploring(self) -> bool:
        return bool(self.queue)

    def plan(self) -> UpdatePlan:
        return self.plan_for(self.next_stride())

    def plan_for(self, stride) -> UpdatePlan:
        return _quiet_plan(len(self.sizes), stride, self.static_ratio, self.placement)


def fast_fraction(plan: UpdatePlan, sizes: Sequence[int]) -> float:
    tot = sum(sizes)
    return sum(s for i, s in enumerate(sizes) if plan.devices[i] is Device.FAST) / tot if tot else 0.0


def capacity_static_ratio(sizes: Sequence[int], free_hbm_bytes: int, *, lowp_bytes_per_param: int = 4,
                          windows: int = 2, headroom_bytes: int = 4 << 30) -> float:
    """SURVEY §8(f) row 2, capacity-aware: the largest TwinFlow static ratio
    whose residents fit in the HBM left after the half-precision grads and
    working copy (``lowp_bytes_per_param`` for the whole shard), ``windows``
    in-flight subgroup windows and a headroom.  Residents are counted at the
    largest subgroup size (placement may take the ragged tail or not), and the
    returned ratio reproduces the count exactly through the reference rule
    ``floor(ratio * N + 1e-9)`` (scheduler.py:161-168)."""
    n = len(sizes)
    if n == 0:
        return 0.0
    big = max(sizes)
    budget = free_hbm_bytes - headroom_bytes - lowp_bytes_per_param * sum(sizes)
    budget -= windows * 12 * big
    count = max(0, min(n, budget // (12 * big)))
    if count == n:  # nothing streams: no windows needed
        count = n if free_hbm_bytes - headroom_bytes - (lowp_bytes_per_param + 12) * sum(sizes) >= 0 else n - 1
    return count / n
