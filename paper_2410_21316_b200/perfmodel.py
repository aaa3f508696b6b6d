"""Closed-form model of the interleaved update phase (Eq. 1).

Restates pkg/src/optistate/perfmodel.py with identical floating-point
evaluation (the planner's choice must be bit-identical for the same profile):

    k_real = (3/B + 1/U_g) / (1/U_c + 1/D_c - 1/(2B))      (perfmodel.py:80-91)

B = host link per direction, U_g/U_c = fast/CPU update rates, D_c = CPU
downscale rate, all in fp32 params/s.  A non-positive denominator means the
host never binds: ``ALL_CPU``.  The integer choice is the cheaper of the two
neighbours of k_real under ``estimate_update_time`` (perfmodel.py:155-179),
and — the reference's documented quirk (perfmodel.py:19-28) — that k is used
directly as the plan *stride*.

On a B200 node the inputs come from measurement (``profile_b200``) and are
re-fitted per iteration, so the CPU/GPU split follows the machine.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .state import SystemProfile


class _AllCpuType:
    """Singleton marker: every subgroup updates on the host, serialized."""

    _only: "_AllCpuType | None" = None

    def __new__(cls) -> "_AllCpuType":
        if cls._only is None:
            cls._only = object.__new__(cls)
        return cls._only

    def __repr__(self) -> str:
        return "ALL_CPU"

    def __reduce__(self):
        return (_AllCpuType, ())

    def __copy__(self):
        return self

    def __deepcopy__(self, memo):
        return self


ALL_CPU = _AllCpuType()


@dataclass(frozen=True)
class StrideResult:
    """``k_real`` (inf when the host never binds), the chosen ``k`` (or
    ALL_CPU) and ``gpu_fraction`` = 1/k of subgroup slots on the fast tier."""

    k_real: float
    k: "int | _AllCpuType"
    gpu_fraction: float


def _check_ratio(k) -> None:
    if not isinstance(k, int) or k < 1:
        raise ValueError(f"ratio k must be an int >= 1 or ALL_CPU, got {k!r}")


def k_real_value(profile: SystemProfile) -> float:
    b = profile.channel_params_per_s
    num = 3.0 / b + 1.0 / profile.fast_update_params_per_s
    den = 1.0 / profile.cpu_update_params_per_s + 1.0 / profile.cpu_downscale_params_per_s - 1.0 / (2.0 * b)
    return math.inf if den <= 0.0 else num / den


def plan_stride_for(k: "int | _AllCpuType") -> "int | _AllCpuType":
    """Stride realising an analysis ratio of k CPU subgroups per fast one."""
    if k is ALL_CPU:
        return ALL_CPU
    _check_ratio(k)
    return k + 1


def estimate_update_time(
    profile: SystemProfile,
    num_subgroups: int,
    subgroup_size: int,
    k: "int | _AllCpuType",
    static_residents: int = 0,
) -> float:
    """Seconds for the phase under ratio ``k`` (perfmodel.py:107-152).

    ALL_CPU: each dynamic subgroup pays update + downscale + half-width H2D
    in series.  Otherwise cycles of k+1 subgroups cost the max of the host
    arm (k updates + downscales, times the contention factor) and the link
    arm (3 state prefetches, k half-width shipments, one fast update).
    Static residents add one fast update each.
    """
    if num_subgroups < 0:
        raise ValueError("num_subgroups must be >= 0")
    if subgroup_size <= 0:
        raise ValueError("subgroup_size must be positive")
    if not 0 <= static_residents <= num_subgroups:
        raise ValueError("static_residents must be in [0, num_subgroups]")
    s = float(subgroup_size)
    p = profile
    b = p.channel_params_per_s
    dynamic = num_subgroups - static_residents
    fixed = static_residents * s / p.fast_update_params_per_s
    if dynamic == 0:
        return fixed
    if k is ALL_CPU:
        one = s / p.cpu_update_params_per_s + s / p.cpu_downscale_params_per_s + s / (2.0 * b)
        return dynamic * one + fixed
    _check_ratio(k)
    host_arm = k * (s / p.cpu_update_params_per_s + s / p.cpu_downscale_params_per_s) * p.host_contention
    link_arm = 3.0 * s / b + k * s / (2.0 * b) + s / p.fast_update_params_per_s
    return dynamic / (k + 1.0) * max(host_arm, link_arm) + fixed


def optimal_stride(profile: SystemProfile, num_subgroups: int = 100,
                   subgroup_size: int = 100_000_000) -> StrideResult:
    """Integer ratio minimising the estimate; ties go to the smaller k."""
    kr = k_real_value(profile)
    if math.isinf(kr):
        return StrideResult(k_real=kr, k=ALL_CPU, gpu_fraction=0.0)
    options = sorted({max(1, math.floor(kr)), max(1, math.ceil(kr))})
    best = options[0]
    best_t = estimate_update_time(profile, num_subgroups, subgroup_size, best)
    for c in options[1:]:
        t = estimate_update_time(profile, num_subgroups, subgroup_size, c)
        if t < best_t:
            best, best_t = c, t
    return StrideResult(k_real=kr, k=best, gpu_fraction=1.0 / best)
