"""ctypes stub binding libdos's host entry points as an optistate backend.

This is the file INTEGRATION.md §1 describes: a maintainer drops it into
`optistate/` as `_dos_native.py` and routes

* `kernels.adam_step_arrays` (reference `kernels.py:136-139`) to
  `dos_adam_step_host` when `OPTISTATE_BACKEND=native`, and
* `core.downscale_rne` / `core.upscale` (reference `core.py:190-205`) to
  `dos_downscale_host` / `dos_upscale_host` under the same backend.

It depends on numpy and ctypes only (no torch): the library is located by
`$DOS_LIBRARY`, else next to the B200 package of this repository.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_DOS_F32, _DOS_F16, _DOS_NONE = 0, 1, -1


class _Scalars(C.Structure):  # include/dos.h: dos_adam_scalars
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("bc1", C.c_float), ("bc2", C.c_float), ("weight_decay", C.c_float), ("adamw", C.c_int32)]


def _find_library() -> str:
    env = os.environ.get("DOS_LIBRARY")
    if env:
        return env
    here = Path(__file__).resolve()
    for root in (here.parent, *here.parents):
        cand = root / "paper_2410_21316_b200" / "libdos.so"
        if cand.exists():
            return str(cand)
    raise OSError("libdos.so not found: set DOS_LIBRARY to its path")


_dos = C.CDLL(_find_library())
_dos.dos_adam_step_host.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                    C.c_int64, C.POINTER(_Scalars), C.c_int]
_dos.dos_downscale_host.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_int]
_dos.dos_upscale_host.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_int]
_dos.dos_last_error.restype = C.c_char_p


# calls routed here, per entry point (the harness checks the backend was used)
CALLS = {"adam_step": 0, "downscale_f16": 0, "upscale_f16": 0}


def _check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(f"libdos error {rc}: {_dos.dos_last_error().decode()}")


def adam_step(p, m, v, g, lr, beta1, beta2, eps, bc1, bc2) -> None:
    """The fused loop of `_adam_step_jit` (kernels.py:88-101) on the host
    team: same arguments (flat fp32 arrays updated in place, np.float32
    scalars already prepared by `adam_step_arrays`)."""
    CALLS["adam_step"] += 1
    # strided views are updated through contiguous copies (the numpy backend
    # accepts them too); flat slices of the shard go straight through
    work = [a if a.flags.c_contiguous else np.ascontiguousarray(a) for a in (p, m, v)]
    g = np.ascontiguousarray(g)
    s = _Scalars(float(lr), float(beta1), float(beta2), float(eps), float(bc1), float(bc2), 0.0, 0)
    _check(_dos.dos_adam_step_host(work[0].ctypes.data, work[1].ctypes.data, work[2].ctypes.data, g.ctypes.data,
                                   _DOS_F32, None, _DOS_NONE, p.size, C.byref(s), 0))
    for dst, src in zip((p, m, v), work):
        if dst is not src:
            dst[...] = src


def downscale_f16(x: np.ndarray) -> np.ndarray:
    """fp32 -> fp16 RNE, numpy `astype` semantics incl. NaN payloads
    (core.py:190-198); any shape."""
    CALLS["downscale_f16"] += 1
    src = np.ascontiguousarray(x)
    out = np.empty(src.shape, dtype=np.float16)
    if src.size:
        _check(_dos.dos_downscale_host(src.ctypes.data, out.ctypes.data, _DOS_F16, src.size, 0))
    return out


def upscale_f16(x: np.ndarray) -> np.ndarray:
    """fp16 -> fp32, exact (core.py:201-205); any shape."""
    CALLS["upscale_f16"] += 1
    src = np.ascontiguousarray(x)
    out = np.empty(src.shape, dtype=np.float32)
    if src.size:
        _check(_dos.dos_upscale_host(src.ctypes.data, _DOS_F16, out.ctypes.data, src.size, 0))
    return out
