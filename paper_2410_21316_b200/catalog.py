"""Named machine profiles (reference: pkg/src/optistate/catalog.py:23-63).

The two reference nodes are kept verbatim so the planner reproduces the
reference's frozen decisions.  ``b200-node`` is measured: its constants come
from ``profile_b200.measure_profile`` on the GPU box (pinned link per
direction under duplex, K1 params/s, H1 params/s on the host team); the
stored numbers are the latest measurement committed under
``profiles/b200_node_profile.json`` and are replaced at run time when the
caller re-measures (``profile_b200.current_profile``).
"""

from __future__ import annotations

import json
from pathlib import Path

from .state import SystemProfile

_H100_CAVEAT = (
    "host-side conversion and allocation rates in this profile are calibrated from mixed-unit sources; "
    "absolute times are indicative, ratios and placement decisions are robust"
)

_MEASURED = Path(__file__).resolve().parent.parent / "profiles" / "b200_node_profile.json"


def _b200_default() -> SystemProfile:
    """The committed measurement, or conservative placeholders if absent."""
    if _MEASURED.exists():
        d = json.loads(_MEASURED.read_text())
        fields = {k: d[k] for k in SystemProfile.__dataclass_fields__ if k in d}
        fields["name"] = "b200-node"
        return SystemProfile(**fields)
    return SystemProfile(
        name="b200-node",
        channel_params_per_s=46e9 / 4,  # pinned PCIe Gen5 x16, duplex, per direction
        fast_update_params_per_s=200e9,
        cpu_update_params_per_s=4e9,
        cpu_downscale_params_per_s=float("inf"),  # fused into H1
        fast_convert_bytes_per_s=3e12,
        host_convert_bytes_per_s=60e9,
        host_alloc_bytes_per_s=4e9,
        pageable_d2h_bytes_per_s=18e9,
        pageable_h2d_bytes_per_s=11e9,
        fast_capacity_bytes=None,
        caveat="placeholder constants: run profile_b200.measure_profile on the box",
    )


PROFILES: dict[str, SystemProfile] = {
    "v100-node": SystemProfile(
        name="v100-node",
        channel_params_per_s=3.0e9,
        fast_update_params_per_s=35.0e9,
        cpu_update_params_per_s=2.0e9,
        cpu_downscale_params_per_s=8.7e9,
        fast_convert_bytes_per_s=0.9e12,
        host_convert_bytes_per_s=30.0e9,
        host_alloc_bytes_per_s=4.0e9,
        pageable_d2h_bytes_per_s=6.0e9,
        pageable_h2d_bytes_per_s=5.5e9,
        fast_capacity_bytes=8_000_000_000,
    ),
    "h100-node": SystemProfile(
        name="h100-node",
        channel_params_per_s=13.75e9,
        fast_update_params_per_s=100.0e9,
        cpu_update_params_per_s=8.0e9,
        cpu_downscale_params_per_s=15.5e9,
        fast_convert_bytes_per_s=1.2e12,
        host_convert_bytes_per_s=62.0e9,
        host_alloc_bytes_per_s=4.0e9,
        pageable_d2h_bytes_per_s=10.0e9,
        pageable_h2d_bytes_per_s=9.0e9,
        fast_capacity_bytes=16_000_000_000,
        caveat=_H100_CAVEAT,
    ),
    "b200-node": _b200_default(),
}


def get_profile(name: str) -> SystemProfile:
    if name not in PROFILES:
        raise KeyError(f"unknown profile {name!r}; known profiles: {', '.join(sorted(PROFILES))}")
    return PROFILES[name]


def list_profiles() -> list[str]:
    return sorted(PROFILES)
