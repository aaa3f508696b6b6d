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
``simulate_b200_fluid`` adds what the list scheduler cannot express: the
host DRAM is shared by the host team and the copy engines, so their rates
are fluid (scaled together whenever their joint host-memory traffic exceeds
the measured peak); with measured ``HostRates`` it is the predictor.
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


@dataclasses.dataclass(frozen=True)
class HostRates:
    """Measured rates for ``simulate_b200_fluid`` (bytes/s, params/s)."""

    link_bytes_per_s: float       # pinned copy per direction, duplex
    host_params_per_s: float      # H1 alone (uncontended)
    fast_params_per_s: float      # K1
    host_dram_bytes_per_s: float  # best measured host-memory throughput


def choose_stride(profile: SystemProfile, sizes: Sequence[int], candidates: Iterable = range(1, 7),
                  static_ratio: float = 0.0, num_slots: int = 2, link_slowdown: float = 1.0,
                  rates: "HostRates | None" = None, placement: Placement = Placement.STATIC_LAST):
    """Stride with the smallest predicted B200 span; returns (stride, {stride: span_ns}).
    With measured ``rates`` the prediction is the fluid host-DRAM model
    (``simulate_b200_fluid``), else the list-scheduled ``simulate_b200_phase``."""
    n = len(sizes)
    spans = {}
    for k in candidates:
        plan = _quiet_plan(n, k, static_ratio, placement)
        if rates is not None:
            spans[k] = simulate_b200_fluid(plan, list(sizes), link_bytes_per_s=rates.link_bytes_per_s,
                                           host_params_per_s=rates.host_params_per_s,
                                           fast_params_per_s=rates.fast_params_per_s,
                                           host_dram_bytes_per_s=rates.host_dram_bytes_per_s, num_slots=num_slots)
        else:
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
                 placement: Placement = Placement.STATIC_LAST, refine: bool = True,
                 rates: "HostRates | None" = None) -> None:
        self.sizes = list(sizes)
        self.static_ratio = static_ratio
        self.placement = placement
        best, spans = choose_stride(profile, self.sizes, candidates, static_ratio, num_slots, link_slowdown,
                                    rates, placement)
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


def simulate_b200_fluid(plan: UpdatePlan, sizes: Sequence[int], *, link_bytes_per_s: float,
                        host_params_per_s: float, fast_params_per_s: float, host_dram_bytes_per_s: float,
                        num_slots: int = 2) -> int:
    """Predicted span (ns) of ``plan`` on the B200 engine with the host DRAM
    modelled as a shared resource.

    Same lanes, FIFO order, dependencies and window gating as
    ``simulate_b200_phase``, but rates are fluid: every action runs at its
    own cap (the link per direction for copies, the uncontended H1 rate for
    host updates, K1 for GPU updates) unless the host-DRAM traffic of the
    actions running together exceeds the measured host-DRAM peak, in which
    case every DRAM consumer is slowed by the same factor (what the probes
    measure: under duplex DMA both H1 and the copy engines drop to ~0.6 of
    their solo rates).  Host bytes per param: 12 per fp32 piece moved over
    the link (4 per piece), 2 per half-precision copy, 28 per host update
    (fused working-copy store)."""
    sizes = list(sizes)
    acts = plan.actions
    n = len(acts)
    dyn = set(plan.dynamic_fast)
    # per action: lane, work units, cap (units/s), host DRAM bytes per unit
    work, cap, dram = [0.0] * n, [1.0] * n, [0.0] * n
    for a in acts:
        k, s = a.kind, (sizes[a.subgroup] if a.subgroup >= 0 else 0)
        if k in _H2D_STATE or k in _D2H_STATE:
            work[a.id], cap[a.id], dram[a.id] = 4.0 * s, link_bytes_per_s, 1.0
        elif k is ActionKind.H2D_PARAMS16:
            work[a.id], cap[a.id], dram[a.id] = 2.0 * s, link_bytes_per_s, 1.0
        elif k is ActionKind.CPU_UPDATE:
            work[a.id], cap[a.id], dram[a.id] = float(s), host_params_per_s, 28.0
        elif k is ActionKind.GPU_UPDATE:
            work[a.id], cap[a.id] = float(s), fast_params_per_s
    queues: dict = {lane: [] for lane in Lane}
    for a in acts:
        queues[a.lane].append(a.id)
    head = dict.fromkeys(Lane, 0)
    finish: list = [None] * n
    window_no: dict[int, int] = {}  # subgroup -> index of its window, in opening order
    closes: list = []               # finish time of each window's FLUSH_OUT_P (None until it happens)
    running: dict = {}              # lane -> [action id, remaining work]
    t = 0.0
    done = 0
    while done < n:
        progressed = True
        while progressed:  # start every lane head whose deps and window are satisfied (zero-work ones finish now)
            progressed = False
            for lane, q in queues.items():
                if lane in running or head[lane] >= len(q):
                    continue
                aid = q[head[lane]]
                a = acts[aid]
                if any(finish[d] is None or finish[d] > t for d in a.deps):
                    continue
                if a.kind is ActionKind.PREFETCH_M and a.subgroup in dyn and a.subgroup not in window_no:
                    w = len(closes)
                    if w >= num_slots and (closes[w - num_slots] is None or closes[w - num_slots] > t):
                        continue
                    window_no[a.subgroup] = w
                    closes.append(None)
                head[lane] += 1
                if work[aid] <= 0:
                    finish[aid] = t
                    done += 1
                    if a.kind is ActionKind.FLUSH_OUT_P and a.subgroup in window_no:
                        closes[window_no[a.subgroup]] = t
                else:
                    running[lane] = [aid, work[aid]]
                progressed = True
        if not running:
            if done < n:
                raise RuntimeError("fluid simulation stalled (plan order not executable)")
            break
        demand = sum(dram[aid] * cap[aid] for aid, _ in running.values())
        f = min(1.0, host_dram_bytes_per_s / demand) if demand > 0 else 1.0
        rate = {lane: cap[aid] * (f if dram[aid] > 0 else 1.0) for lane, (aid, _) in running.items()}
        dt = min(rem / rate[lane] for lane, (_, rem) in running.items())
        t += dt
        for lane in list(running):
            aid, rem = running[lane]
            rem -= rate[lane] * dt
            if rem <= 1e-9 * max(1.0, work[aid]):
                finish[aid] = t
                done += 1
                a = acts[aid]
                if a.kind is ActionKind.FLUSH_OUT_P and a.subgroup in window_no:
                    closes[window_no[a.subgroup]] = t
                del running[lane]
            else:
                running[lane][1] = rem
    return int(round(max(finish) * 1e9)) if n else 0
