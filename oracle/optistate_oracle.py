"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

numpy restatement of the reference's update-phase numerics.  Each function
cites the reference lines it follows (paths under /root/reference/pkg/src/
optistate/).  Pinned against tests/golden/* (generated from the reference).
"""
from __future__ import annotations

import hashlib
import math

import numpy as np


def bias_corrections(beta1: float, beta2: float, step: int):
    """kernels.py:122-123 — fp64 pow, then one rounding to fp32."""
    return np.float32(1.0 - math.pow(beta1, step)), np.float32(1.0 - math.pow(beta2, step))


def adam_step(p, m, v, g, lr, beta1, beta2, eps, step, weight_decay=0.0):
    """In-place fp32 Adam, op order of kernels.py:77-85 (== the numba loop :93-101).

    weight_decay > 0 (AdamW) is NOT pinned by the reference (it has no weight
    decay, executor.py:45-56); declared order: p *= f32(1 - f32(lr*wd)) first.
    """
    if step < 1:
        raise ValueError("step must be >= 1")
    bc1, bc2 = bias_corrections(beta1, beta2, step)
    f = np.float32
    lr32, b1, b2, e32 = f(lr), f(beta1), f(beta2), f(eps)
    one = f(1.0)
    if weight_decay:
        decay = one - f(lr32 * f(weight_decay))
        p *= decay
    m[:] = b1 * m + (one - b1) * g
    v[:] = b2 * v + (one - b2) * (g * g)
    mh = m / bc1
    vh = v / bc2
    p -= (lr32 * mh) / (np.sqrt(vh) + e32)


def f16_from_f32(x: np.ndarray) -> np.ndarray:
    """core.py:190-198 downscale_rne: numpy's astype(float16)."""
    with np.errstate(over="ignore"):
        return np.asarray(x, dtype=np.float32).astype(np.float16)


def f32_from_f16(x: np.ndarray) -> np.ndarray:
    """core.py:201-205 upscale."""
    return np.asarray(x, dtype=np.float16).astype(np.float32)


def bf16_from_f32(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bits (uint16), round-to-nearest-even on the bit pattern,
    NaN -> 0x7FC0 (torch/c10's rule; the reference has no bf16)."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r[nan] = 0x7FC0
    return r


def f32_from_bf16(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def lowp_from_f32(x, lowp):
    return f16_from_f32(x) if lowp == "fp16" else bf16_from_f32(x)


def f32_from_lowp(x, lowp):
    return f32_from_f16(x) if lowp == "fp16" else f32_from_bf16(x)


def reduce_scatter(sources, lowp, scale=1.0):
    """The ZeRO-3 grad reduce-scatter for one rank's shard, as the fused
    B200 path defines it (include/dos.h, dos_state_desc.src_g).  NOT pinned by
    the reference, which has no collectives:
    declared order — widen every rank's grads exactly (core.py:201-205), sum
    in fp32 in rank order with one RN rounding per add, round once to the
    grad dtype (RNE), then, if scale != 1, round(f32(x) * f32(scale)) again.
    ``sources`` are the ranks' half-precision arrays in rank order."""
    acc = f32_from_lowp(sources[0], lowp).astype(np.float32, copy=True)
    for src in sources[1:]:
        acc = np.add(acc, f32_from_lowp(src, lowp), dtype=np.float32)
    out = lowp_from_f32(acc, lowp)
    if scale != 1.0:
        out = lowp_from_f32(np.multiply(f32_from_lowp(out, lowp), np.float32(scale), dtype=np.float32), lowp)
    return out


def shard_subgroups(total: int, subgroup_size: int):
    """core.py:139-170 for one rank: (start, size) per subgroup."""
    return [(s, min(subgroup_size, total - s)) for s in range(0, total, subgroup_size)]


def initialize(total: int, subgroup_size: int, seed: int = 0, lowp: str = "fp16"):
    """core.py:249-272: the reference's seeded synthetic shard (same draws)."""
    rng = np.random.default_rng(seed)
    p = rng.normal(0.0, 0.02, total).astype(np.float32)
    m = rng.normal(0.0, 1e-3, total).astype(np.float32)
    v = rng.random(total).astype(np.float32) * np.float32(1e-4)
    g = rng.normal(0.0, 1.0, total).astype(np.float32)
    return {"p": p, "m": m, "v": v, "w": lowp_from_f32(p, lowp), "g": lowp_from_f32(g, lowp),
            "subgroups": shard_subgroups(total, subgroup_size), "step": 0, "lowp": lowp}


def sequential_oracle(state: dict, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0) -> dict:
    """executor.py:103-117: every subgroup in order — widen grads, Adam,
    refresh the working copy; one step number for the whole phase."""
    step = state["step"] + 1
    lowp = state["lowp"]
    for a, n in state["subgroups"]:
        sl = slice(a, a + n)
        g32 = f32_from_lowp(state["g"][sl], lowp)
        adam_step(state["p"][sl], state["m"][sl], state["v"][sl], g32, lr, beta1, beta2, eps, step, weight_decay)
        state["w"][sl] = lowp_from_f32(state["p"][sl], lowp)
    state["step"] = step
    return state


def state_digest(state: dict) -> str:
    """sha256 over p, m, v, working copy, grads (core.py:285-293 order)."""
    h = hashlib.sha256()
    for k in ("p", "m", "v", "w", "g"):
        h.update(np.ascontiguousarray(state[k]).tobytes())
    return h.hexdigest()
