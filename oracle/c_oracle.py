"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): ctypes loader of the C oracle."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_DIR = Path(__file__).resolve().parent
_LIB = _DIR / "_build" / "liboracle.so"
_lib = None


def build() -> Path:
    if not _LIB.exists() or _LIB.stat().st_mtime < (_DIR / "adam_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_DIR)], check=True)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        if not _LIB.exists():
            build()
        _lib = C.CDLL(str(_LIB))
        f = C.c_float
        _lib.oracle_adam_mt.restype = C.c_int
        _lib.oracle_adam_mt.argtypes = [C.c_void_p] * 4 + [C.c_int, C.c_void_p, C.c_int, C.c_int64] + [f] * 6 + [C.c_int]
    return _lib


GKIND = {"fp32": 0, "fp16": 1, "bf16": 2}
LOWP = {None: 0, "fp16": 1, "bf16": 2}


def adam_mt(p, m, v, g, gkind: str, w, lowp, lr, b1, b2, eps, step, nthreads=None):
    """In-place threaded C Adam (+ optional working-copy write)."""
    import math
    bc1 = np.float32(1.0 - math.pow(b1, step))
    bc2 = np.float32(1.0 - math.pow(b2, step))
    n = p.size
    nthreads = nthreads or len(os.sched_getaffinity(0))
    rc = lib().oracle_adam_mt(p.ctypes.data, m.ctypes.data, v.ctypes.data, g.ctypes.data, GKIND[gkind],
                              w.ctypes.data if w is not None else None, LOWP[lowp], n,
                              float(np.float32(lr)), float(np.float32(b1)), float(np.float32(b2)),
                              float(np.float32(eps)), float(bc1), float(bc2), int(nthreads))
    if rc != 0:
        raise RuntimeError("oracle thread launch failed")
