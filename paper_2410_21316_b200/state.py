"""Rank-local optimizer state: subgroups, the ZeRO-3 partition, byte
accounting, machine profiles, precision conversions and the sharded state
container.

API-compatible with the reference's ``optistate.core``
(pkg/src/optistate/core.py).  What changes is where the bytes live:

* fp32 master params / momentum / variance and the half-precision grads and
  working copy are views of the *pinned host pool* (``dos_host_alloc``:
  page-locked, THP-backed, registered with CUDA), so subgroup prefetch and
  flush are DMA copies with no staging;
* once the optimizer is attached to a B200 (``to_device``), the device holds
  the grads and the authoritative half-precision working copy, plus the
  fp32 state of any static residents; the host images of those are
  refreshed lazily when read, never inside the update phase;
* conversions run in libdos (numpy-exact fp16, torch-exact bf16), not numpy.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass
from typing import TYPE_CHECKING

import numpy as np

from . import _native as N

if TYPE_CHECKING:  # pragma: no cover
    from .device import DeviceResidency

# Byte costs per parameter (core.py:19-29): fp32 p, m, v + an fp32 grad
# slot for optimizer state; 2 B working copy; 2 B grads; a 12 B (p, m, v)
# window for each in-flight subgroup.
OPTIMIZER_BYTES_PER_PARAM = 16
MODEL16_BYTES_PER_PARAM = 2
GRADS16_BYTES_PER_PARAM = 2
SUBGROUP_STATE_BYTES_PER_PARAM = 12

# numpy dtype used to hold each half-precision kind on the host (bf16 has no
# numpy dtype: its raw bits are kept as uint16).
_LOWP_NP = {"fp16": np.dtype(np.float16), "bf16": np.dtype(np.uint16)}


class Precision(enum.Enum):
    FP16 = "fp16"
    FP32 = "fp32"
    BF16 = "bf16"

    @property
    def itemsize(self) -> int:
        return 4 if self is Precision.FP32 else 2


@dataclass(frozen=True)
class Subgroup:
    """Contiguous ``[start, start + size)`` slice of one rank's flat shard."""

    index: int
    start: int
    size: int

    def __post_init__(self) -> None:
        if self.size <= 0:
            raise ValueError(f"subgroup size must be positive, got {self.size}")
        if self.start < 0:
            raise ValueError(f"subgroup start must be >= 0, got {self.start}")

    @property
    def stop(self) -> int:
        return self.start + self.size

    @property
    def slice(self) -> slice:
        return slice(self.start, self.stop)

    def state_bytes(self) -> int:
        return SUBGROUP_STATE_BYTES_PER_PARAM * self.size


_RATE_FIELDS = (
    "channel_params_per_s",
    "fast_update_params_per_s",
    "cpu_update_params_per_s",
    "cpu_downscale_params_per_s",
    "fast_convert_bytes_per_s",
    "host_convert_bytes_per_s",
    "host_alloc_bytes_per_s",
    "pageable_d2h_bytes_per_s",
    "pageable_h2d_bytes_per_s",
)


@dataclass(frozen=True)
class SystemProfile:
    """Machine rates feeding the performance model and the simulator.

    ``*_params_per_s`` count fp32 parameters per second, ``*_bytes_per_s``
    count bytes on the half-precision / wire side (core.py:68-113).
    ``channel_params_per_s`` is the pinned host link per direction.
    """

    name: str
    channel_params_per_s: float
    fast_update_params_per_s: float
    cpu_update_params_per_s: float
    cpu_downscale_params_per_s: float
    fast_convert_bytes_per_s: float
    host_convert_bytes_per_s: float
    host_alloc_bytes_per_s: float
    pageable_d2h_bytes_per_s: float
    pageable_h2d_bytes_per_s: float
    fast_capacity_bytes: int | None = None
    host_contention: float = 1.0
    caveat: str | None = None

    def __post_init__(self) -> None:
        bad = [f for f in _RATE_FIELDS if not (getattr(self, f) > 0)]
        if bad:
            raise ValueError(f"{bad[0]} must be positive, got {getattr(self, bad[0])}")
        if self.host_contention < 1.0:
            raise ValueError(f"host_contention must be >= 1.0, got {self.host_contention}")
        if self.fast_capacity_bytes is not None and self.fast_capacity_bytes < 0:
            raise ValueError("fast_capacity_bytes must be >= 0 when set")


@dataclass(frozen=True)
class FootprintReport:
    """Exact integer byte accounting of one rank's shard."""

    total_params: int
    subgroup_size: int
    num_subgroups: int
    optimizer32_bytes: int
    model16_bytes: int
    grads16_bytes: int
    per_subgroup_state_bytes: int

    @property
    def host_resident_bytes(self) -> int:
        return self.optimizer32_bytes

    @property
    def fast_resident_bytes(self) -> int:
        return self.model16_bytes + self.grads16_bytes


def _positive(**kw) -> None:
    for k, v in kw.items():
        if v <= 0:
            raise ValueError(f"{k} must be positive")


def shard(total_params: int, num_ranks: int, subgroup_size: int) -> list[list[Subgroup]]:
    """ZeRO-3 partition then subgroup cut (core.py:139-170).

    Ranks take ``ceil(P / N)`` params each until the remainder runs out; each
    rank's share is cut into ``subgroup_size`` pieces with a ragged tail.
    Offsets are rank-local.
    """
    _positive(total_params=total_params, num_ranks=num_ranks, subgroup_size=subgroup_size)
    quota = -(-total_params // num_ranks)
    ranks: list[list[Subgroup]] = []
    left = total_params
    for _ in range(num_ranks):
        mine = min(quota, left)
        left -= mine
        cuts = range(0, mine, subgroup_size)
        ranks.append([Subgroup(index=k, start=s, size=min(subgroup_size, mine - s)) for k, s in enumerate(cuts)])
    return ranks


def footprint(total_params: int, subgroup_size: int) -> FootprintReport:
    _positive(total_params=total_params, subgroup_size=subgroup_size)
    return FootprintReport(
        total_params=total_params,
        subgroup_size=subgroup_size,
        num_subgroups=-(-total_params // subgroup_size),
        optimizer32_bytes=OPTIMIZER_BYTES_PER_PARAM * total_params,
        model16_bytes=MODEL16_BYTES_PER_PARAM * total_params,
        grads16_bytes=GRADS16_BYTES_PER_PARAM * total_params,
        per_subgroup_state_bytes=SUBGROUP_STATE_BYTES_PER_PARAM * subgroup_size,
    )


# ---------------------------------------------------------------- conversions


def _flat_contig(x: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(x).reshape(-1)


def downscale_rne(x: np.ndarray) -> np.ndarray:
    """float32 -> float16, IEEE round-to-nearest-even (core.py:190-198).

    Overflow becomes +/-inf, subnormals are exact, NaN payloads follow numpy.
    Runs in libdos (dos_downscale_host) on the host team.
    """
    if x.dtype != np.float32:
        raise TypeError(f"downscale_rne expects float32, got {x.dtype}")
    src = _flat_contig(x)
    out = np.empty(src.shape, dtype=np.float16)
    N.check(N.lib().dos_downscale_host(N.ptr(src), N.ptr(out), N.DOS_F16, src.size, 0))
    return out.reshape(x.shape)


def upscale(x: np.ndarray) -> np.ndarray:
    """float16 -> float32, always exact (core.py:201-205)."""
    if x.dtype != np.float16:
        raise TypeError(f"upscale expects float16, got {x.dtype}")
    src = _flat_contig(x)
    out = np.empty(src.shape, dtype=np.float32)
    N.check(N.lib().dos_upscale_host(N.ptr(src), N.DOS_F16, N.ptr(out), src.size, 0))
    return out.reshape(x.shape)


def downscale_bf16(x: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 bits (uint16), round-to-nearest-even (torch rule)."""
    if x.dtype != np.float32:
        raise TypeError(f"downscale_bf16 expects float32, got {x.dtype}")
    src = _flat_contig(x)
    out = np.empty(src.shape, dtype=np.uint16)
    N.check(N.lib().dos_downscale_host(N.ptr(src), N.ptr(out), N.DOS_BF16, src.size, 0))
    return out.reshape(x.shape)


def upscale_bf16(x: np.ndarray) -> np.ndarray:
    """bfloat16 bits (uint16) -> float32, exact."""
    if x.dtype != np.uint16:
        raise TypeError(f"upscale_bf16 expects uint16 bf16 bits, got {x.dtype}")
    src = _flat_contig(x)
    out = np.empty(src.shape, dtype=np.float32)
    N.check(N.lib().dos_upscale_host(N.ptr(src), N.DOS_BF16, N.ptr(out), src.size, 0))
    return out.reshape(x.shape)


def lowp_downscale(x: np.ndarray, lowp: str) -> np.ndarray:
    return downscale_rne(x) if lowp == "fp16" else downscale_bf16(x)


def lowp_upscale(x: np.ndarray, lowp: str) -> np.ndarray:
    return upscale(x) if lowp == "fp16" else upscale_bf16(x)


# ---------------------------------------------------------------- state


def pinned_empty(count: int, dtype, numa_node: int = -1) -> np.ndarray:
    """A flat array in the pinned host pool."""
    dt = np.dtype(dtype)
    if count == 0:
        return np.empty(0, dtype=dt)
    return N.HostBuffer(dt.itemsize * count, numa_node=numa_node).array(dt, count)


class ShardedOptimizer:
    """One rank's optimizer shard (core.py:208-293).

    ``params32``/``momentum32``/``variance32`` are the fp32 master state,
    ``model16`` the half-precision working copy, ``grads16`` the step's
    half-precision gradients (float16, or bf16 bits as uint16 when
    ``lowp == "bf16"``).  ``step`` counts completed optimizer steps.

    After ``to_device`` the B200 holds the authoritative working copy and
    static residents; the host attributes re-synchronise on first read.
    """

    def __init__(
        self,
        subgroups: list[Subgroup],
        params32: np.ndarray,
        momentum32: np.ndarray,
        variance32: np.ndarray,
        model16: np.ndarray,
        grads16: np.ndarray,
        step: int = 0,
        lowp: str = "fp16",
    ) -> None:
        if lowp not in _LOWP_NP:
            raise ValueError(f"lowp must be 'fp16' or 'bf16', got {lowp!r}")
        self.subgroups = list(subgroups)
        self.lowp = lowp
        self.step = step
        total = sum(g.size for g in self.subgroups)
        want16 = _LOWP_NP[lowp]
        for name, arr, want in (
            ("params32", params32, np.dtype(np.float32)),
            ("momentum32", momentum32, np.dtype(np.float32)),
            ("variance32", variance32, np.dtype(np.float32)),
            ("model16", model16, want16),
            ("grads16", grads16, want16),
        ):
            if arr.dtype != want:
                raise TypeError(f"{name} must be {want}, got {arr.dtype}")
            if arr.shape != (total,):
                raise ValueError(f"{name} must be flat with {total} elements, got {arr.shape}")
        self._p, self._m, self._v = params32, momentum32, variance32
        self._w, self._g = model16, grads16
        self._total = total
        self.residency: DeviceResidency | None = None
        # sparse host pool (allocate(host_homed=...)): per array group, which
        # subgroups' host ranges are committed; None = dense (all committed)
        self._sparse: dict | None = None

    # -- sparse host pool
    _GROUPS = {"state": ("_p", "_m", "_v"), "lowp": ("_g", "_w")}

    def host_committed(self, sg: int, group: str = "state") -> bool:
        return self._sparse is None or bool(self._sparse[group][sg])

    def ensure_host(self, subgroups, group: str = "state") -> None:
        """Commit (touch, page-lock, register) the host ranges of ``subgroups``
        in the arrays of ``group`` ("state": p/m/v, "lowp": grads/working copy).
        No-op for a dense pool or ranges already committed."""
        if self._sparse is None:
            return
        have = self._sparse[group]
        todo = sorted(i for i in subgroups if not have[i])
        if not todo:
            return
        for a, b in _runs([self.subgroups[i] for i in todo]):
            for name in self._GROUPS[group]:
                arr = getattr(self, name)
                self._sparse["bufs"][name].commit(a * arr.itemsize, (b - a) * arr.itemsize)
        have[todo] = True
        if self.residency is not None:  # fill the new host ranges from the device where it is authoritative
            self.residency.on_host_commit(todo, group)

    def host_runs(self, group: str = "state") -> list[tuple[int, int]]:
        """Element ranges ``[a, b)`` whose host images are committed (merged)."""
        if self._sparse is None:
            return [(0, self._total)] if self._total else []
        have = self._sparse[group]
        return _runs([g for g in self.subgroups if have[g.index]])

    @property
    def host_bytes(self) -> int:
        """Host memory committed for this shard's arrays."""
        arrays = (self._p, self._m, self._v, self._g, self._w)
        if self._sparse is None:
            return sum(a.nbytes for a in arrays)
        return sum(self._sparse["bufs"][n].committed_bytes for n in ("_p", "_m", "_v", "_g", "_w"))

    # -- host views (lazily refreshed from the device when it is authoritative)
    def _host(self, name: str) -> np.ndarray:
        if self._sparse is not None:  # a full-array read materialises every range
            self.ensure_host(range(len(self.subgroups)), "state" if name in ("_p", "_m", "_v") else "lowp")
        if self.residency is not None:
            self.residency.sync_host(name)
        return getattr(self, name)

    @property
    def params32(self) -> np.ndarray:
        return self._host("_p")

    @property
    def momentum32(self) -> np.ndarray:
        return self._host("_m")

    @property
    def variance32(self) -> np.ndarray:
        return self._host("_v")

    @property
    def model16(self) -> np.ndarray:
        return self._host("_w")

    @property
    def grads16(self) -> np.ndarray:
        return self._host("_g")  # after an in-phase grad flush the device holds the step's grads

    @property
    def total_params(self) -> int:
        return self._total

    @property
    def lowp_code(self) -> int:
        return N.LOWP_CODES[self.lowp]

    # -- construction
    @classmethod
    def allocate(cls, total_params: int, subgroup_size: int, lowp: str = "fp16",
                 numa_node: int = -1, host_homed=None) -> "ShardedOptimizer":
        """Zero-filled state in the pinned pool (no RNG).

        ``host_homed``: None commits every array for the whole shard (the
        reference's layout, core.py:208-272).  A collection of subgroup
        indices reserves the address space but commits host memory only for
        those subgroups — the rest are to be homed in HBM as static residents
        (``DeviceResidency.set_static``), so a shard whose state exceeds the
        host RAM still runs.  Uncommitted ranges read as zeros and are
        committed on demand (``ensure_host``, or any full-array read).
        """
        groups = shard(total_params, 1, subgroup_size)[0]
        dt16 = _LOWP_NP[lowp]
        if host_homed is None:
            return cls(
                subgroups=groups,
                params32=pinned_empty(total_params, np.float32, numa_node),
                momentum32=pinned_empty(total_params, np.float32, numa_node),
                variance32=pinned_empty(total_params, np.float32, numa_node),
                model16=pinned_empty(total_params, dt16, numa_node),
                grads16=pinned_empty(total_params, dt16, numa_node),
                lowp=lowp,
            )
        homed = sorted({int(i) for i in host_homed})
        if homed and (homed[0] < 0 or homed[-1] >= len(groups)):
            raise ValueError(f"host_homed indices must be in [0, {len(groups)})")
        bufs, arrays = {}, {}
        for name, dt in (("_p", np.float32), ("_m", np.float32), ("_v", np.float32), ("_w", dt16), ("_g", dt16)):
            dt = np.dtype(dt)
            hb = N.HostBuffer(max(1, dt.itemsize * total_params), numa_node=numa_node, sparse=True)
            bufs[name] = hb
            arrays[name] = hb.array(dt, total_params)
        opt = cls(subgroups=groups, params32=arrays["_p"], momentum32=arrays["_m"], variance32=arrays["_v"],
                  model16=arrays["_w"], grads16=arrays["_g"], lowp=lowp)
        opt._sparse = {"bufs": bufs, "state": np.zeros(len(groups), dtype=bool),
                       "lowp": np.zeros(len(groups), dtype=bool)}
        opt.ensure_host(homed, "state")
        opt.ensure_host(homed, "lowp")
        return opt

    @classmethod
    def initialize(cls, total_params: int, subgroup_size: int, seed: int = 0,
                   lowp: str = "fp16") -> "ShardedOptimizer":
        """Seeded synthetic state, draw-for-draw identical to core.py:249-272.

        p ~ N(0, 0.02), m ~ N(0, 1e-3), v ~ U[0,1) * 1e-4 (fp32 product),
        g ~ N(0, 1) rounded to ``lowp``; model16 = lowp(p).  For the bf16
        kind the same fp32 draws are rounded RNE to bf16.
        """
        opt = cls.allocate(total_params, subgroup_size, lowp)
        rng = np.random.default_rng(seed)
        opt._p[:] = rng.normal(0.0, 0.02, total_params).astype(np.float32)
        opt._m[:] = rng.normal(0.0, 1e-3, total_params).astype(np.float32)
        opt._v[:] = rng.random(total_params).astype(np.float32) * np.float32(1e-4)
        g32 = rng.normal(0.0, 1.0, total_params).astype(np.float32)
        opt._g[:] = lowp_downscale(g32, lowp)
        opt._w[:] = lowp_downscale(opt._p, lowp)
        return opt

    def copy(self) -> "ShardedOptimizer":
        """Host-only deep copy (plain memory; no device residency)."""
        return ShardedOptimizer(
            subgroups=list(self.subgroups),
            params32=self.params32.copy(),
            momentum32=self.momentum32.copy(),
            variance32=self.variance32.copy(),
            model16=self.model16.copy(),
            grads16=self.grads16.copy(),
            step=self.step,
            lowp=self.lowp,
        )

    def state_equal(self, other: "ShardedOptimizer") -> bool:
        """Bitwise equality of all five arrays (NaN-safe)."""
        pairs = (
            (self.params32, other.params32),
            (self.momentum32, other.momentum32),
            (self.variance32, other.variance32),
            (self.model16, other.model16),
            (self.grads16, other.grads16),
        )
        return all(a.view(np.uint8).tobytes() == b.view(np.uint8).tobytes() for a, b in pairs)

    # -- device attachment
    def to_device(self, device=None, grads=None, model16=None) -> "DeviceResidency":
        """Attach (or return) the B200 residency: grads + working copy in HBM
        (optionally in caller-owned CUDA views, see DeviceResidency)."""
        from .device import DeviceResidency

        if self.residency is None:
            self.residency = DeviceResidency(self, device, grads=grads, model16=model16)
        return self.residency

    def load_grads(self, grads) -> None:
        """Replace this step's gradients (host array of the lowp kind, or a
        CUDA tensor); keeps the host and device images consistent."""
        if self.residency is not None:
            self.residency.load_grads(grads)
            return
        arr = np.asarray(grads)
        if arr.dtype != self._g.dtype or arr.shape != self._g.shape:
            raise TypeError(f"grads must be {self._g.dtype}{self._g.shape}")
        self._g[:] = arr


def _runs(subgroups) -> list[tuple[int, int]]:
    """Merged element ranges covered by ``subgroups``."""
    out: list[list[int]] = []
    for g in sorted(subgroups, key=lambda g: g.start):
        if out and g.start <= out[-1][1]:
            out[-1][1] = max(out[-1][1], g.stop)
        else:
            out.append([g.start, g.stop])
    return [(a, b) for a, b in out]


def bias_corrections(beta1: float, beta2: float, step: int) -> tuple[np.float32, np.float32]:
    """bc1, bc2 exactly as kernels.py:122-123: f32(1 - pow(beta, step)) in fp64."""
    return np.float32(1.0 - math.pow(beta1, step)), np.float32(1.0 - math.pow(beta2, step))
