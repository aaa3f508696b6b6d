"""ctypes binding of libdos.so (declared in include/dos.h).

ctypes releases the GIL for the duration of every foreign call, so the host
team, the engine's host-lane worker and the CUDA copy engines all run while
Python is free.  There is no fallback: if the library is missing this module
raises on first use (set DOS_AUTOBUILD=1 to compile it in-tree on demand).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libdos.so"

# error codes (include/dos.h)
DOS_OK = 0
DOS_EINVAL = -1
DOS_ETYPE = -2
DOS_ECUDA = -3
DOS_ESYS = -4
DOS_EINFEASIBLE = -5
DOS_ESTATE = -6

# dtypes
DOS_NONE = -1
DOS_F32 = 0
DOS_F16 = 1
DOS_BF16 = 2

LOWP_CODES = {"fp16": DOS_F16, "bf16": DOS_BF16}


class dos_adam_scalars(C.Structure):
    _fields_ = [
        ("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
        ("bc1", C.c_float), ("bc2", C.c_float), ("weight_decay", C.c_float), ("adamw", C.c_int32),
    ]


class dos_state_desc(C.Structure):
    _fields_ = [
        ("num_subgroups", C.c_int32),
        ("sg_start", C.POINTER(C.c_int64)),
        ("sg_size", C.POINTER(C.c_int64)),
        ("static_offset", C.POINTER(C.c_int64)),
        ("lowp_dtype", C.c_int32),
        ("host_p", C.c_void_p), ("host_m", C.c_void_p), ("host_v", C.c_void_p),
        ("host_g", C.c_void_p), ("host_lowp", C.c_void_p),
        ("dev_g", C.c_void_p), ("dev_lowp", C.c_void_p),
        ("dev_static_p", C.c_void_p), ("dev_static_m", C.c_void_p), ("dev_static_v", C.c_void_p),
        ("host_io", C.c_int32),
        ("npeers", C.c_int32),
        ("peer_lowp", C.POINTER(C.c_void_p)),
        ("flush_grads", C.c_int32),
        ("nsrc_g", C.c_int32),
        ("self_rank", C.c_int32),
        ("src_g", C.POINTER(C.c_void_p)),
        ("grad_scale", C.c_float),
        ("dev_static_sg", C.POINTER(C.c_void_p)),
        ("host_io_ahead", C.c_int32),
        ("host_updates", C.c_int32),
    ]


DOS_MAX_PEERS = 7


class dos_exec_config(C.Structure):
    _fields_ = [
        ("device", C.c_int32), ("num_slots", C.c_int32), ("slot_elems", C.c_int64),
        ("host_threads", C.c_int32), ("fuse_downscale", C.c_int32),
    ]


class dos_action_desc(C.Structure):
    _fields_ = [
        ("id", C.c_int32), ("kind", C.c_int32), ("subgroup", C.c_int32), ("lane", C.c_int32),
        ("is_static", C.c_int32), ("num_deps", C.c_int32), ("deps", C.POINTER(C.c_int32)),
        ("batch_len", C.c_int32), ("batch", C.POINTER(C.c_int32)),
    ]


class dos_coh_range(C.Structure):
    _fields_ = [("p32", C.c_void_p), ("lowp", C.c_void_p), ("n", C.c_int64), ("window", C.c_int64),
                ("nwin", C.c_int64)]


# every symbol include/dos.h declares, with its ctypes signature
_VP, _I, _I64, _SZ = C.c_void_p, C.c_int, C.c_int64, C.c_size_t
SIGNATURES: dict[str, tuple] = {
    "dos_last_error": (C.c_char_p, []),
    "dos_version": (_I, []),
    "dos_launch_count": (_I64, []),
    "dos_adam_step_cuda": (_I, [_VP, _VP, _VP, _VP, _I, _VP, _I, _I64, C.POINTER(dos_adam_scalars), _VP]),
    "dos_adam_step_host": (_I, [_VP, _VP, _VP, _VP, _I, _VP, _I, _I64, C.POINTER(dos_adam_scalars), _I]),
    "dos_adam_step_cuda_bcast": (_I, [_VP, _VP, _VP, _VP, _I, _VP, _I, C.POINTER(_VP), _I, _I64,
                                      C.POINTER(dos_adam_scalars), _VP]),
    "dos_adam_step_cuda_rs": (_I, [_VP, _VP, _VP, C.POINTER(_VP), _I, _I, _I, C.c_float, _VP, _I, C.POINTER(_VP),
                                   _I, _I64, C.POINTER(dos_adam_scalars), _VP]),
    "dos_reduce_scatter_cuda": (_I, [_VP, C.POINTER(_VP), _I, _I, C.c_float, _I64, _VP]),
    "dos_coherence_cuda": (_I, [C.POINTER(dos_coh_range), _I, _I, C.POINTER(C.c_ulonglong), _VP]),
    "dos_ipc_export": (_I, [_VP, C.c_char_p, C.POINTER(C.c_uint64)]),
    "dos_ipc_import": (_I, [C.c_char_p, C.c_uint64, C.POINTER(_VP)]),
    "dos_ipc_close_all": (_I, []),
    "dos_downscale_host": (_I, [_VP, _VP, _I, _I64, _I]),
    "dos_upscale_host": (_I, [_VP, _I, _VP, _I64, _I]),
    "dos_downscale_cuda": (_I, [_VP, _VP, _I, _I64, _VP]),
    "dos_upscale_cuda": (_I, [_VP, _I, _VP, _I64, _VP]),
    "dos_host_alloc": (_I, [_SZ, _I, _I, C.POINTER(_VP)]),
    "dos_host_free": (_I, [_VP]),
    "dos_host_reserve": (_I, [_SZ, _I, _I, C.POINTER(_VP)]),
    "dos_host_commit": (_I, [_VP, _SZ, _SZ]),
    "dos_host_committed": (C.c_int64, [_VP]),
    "dos_host_threads": (_I, []),
    "dos_host_membw": (_I, [_VP, _VP, _SZ, _I, _I, C.POINTER(C.c_double)]),
    "dos_set_host_threads": (_I, [_I]),
    "dos_exec_create": (_I, [C.POINTER(dos_exec_config), C.POINTER(_VP)]),
    "dos_exec_destroy": (_I, [_VP]),
    "dos_exec_begin": (_I, [_VP, C.POINTER(dos_state_desc), C.POINTER(dos_adam_scalars), C.c_int32]),
    "dos_exec_submit": (_I, [_VP, C.POINTER(dos_action_desc)]),
    "dos_exec_finish": (_I, [_VP, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.c_int32]),
    "dos_exec_slot_ptr": (_I, [_VP, C.c_int32, C.c_int32, C.POINTER(C.POINTER(C.c_float))]),
    "dos_exec_stream_wait": (_I, [_VP, C.c_int32, _VP]),
}

_lock = threading.Lock()
_lib: C.CDLL | None = None


class InfeasibleConfigError(Exception):
    """The fast tier cannot hold even one in-flight subgroup window.

    Same meaning as the reference's scheduler.InfeasibleConfigError
    (pkg/src/optistate/scheduler.py:92-93); defined here so the native
    error mapping and the planner share one class.
    """


def lib() -> C.CDLL:
    """Load libdos.so (building it first only if DOS_AUTOBUILD=1)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            if os.environ.get("DOS_AUTOBUILD") == "1":
                from . import _build

                _build.build()
            else:
                raise RuntimeError(
                    f"libdos.so not found at {LIB_PATH}; run `python -m paper_2410_21316_b200._build` "
                    "(or __graft_entry__.build()) — there is no non-native fallback"
                )
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
        return handle


def check(rc: int) -> None:
    """Map a libdos return code to the reference's exception types."""
    if rc == DOS_OK:
        return
    msg = lib().dos_last_error().decode(errors="replace")
    if rc == DOS_EINVAL:
        raise ValueError(msg)
    if rc == DOS_ETYPE:
        raise TypeError(msg)
    if rc == DOS_EINFEASIBLE:
        raise InfeasibleConfigError(msg)
    if rc == DOS_ESTATE:
        raise AssertionError(msg)
    raise RuntimeError(f"libdos error {rc}: {msg}")


def ptr(a) -> int:
    """Raw address of a numpy array or torch tensor (no copy)."""
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def scalars(lr: float, beta1: float, beta2: float, eps: float, bc1, bc2,
            weight_decay: float = 0.0) -> dos_adam_scalars:
    """Per-step scalars; bc1/bc2 are already-rounded np.float32 values."""
    return dos_adam_scalars(
        float(np.float32(lr)), float(np.float32(beta1)), float(np.float32(beta2)), float(np.float32(eps)),
        float(bc1), float(bc2), float(np.float32(weight_decay)), 1 if weight_decay else 0,
    )


class HostBuffer:
    """A region of the pinned host pool, freed on GC.

    Dense (default, dos_host_alloc): committed and registered whole.
    ``sparse=True`` (dos_host_reserve): address space only; ``commit`` makes
    byte ranges resident, page-locked and registered (dos_host_commit)."""

    def __init__(self, nbytes: int, numa_node: int = -1, register_cuda: bool = True, sparse: bool = False):
        out = C.c_void_p()
        fn = lib().dos_host_reserve if sparse else lib().dos_host_alloc
        check(fn(int(nbytes), int(numa_node), 1 if register_cuda else 0, C.byref(out)))
        self.address = out.value
        self.nbytes = int(nbytes)
        self.sparse = sparse

    def commit(self, offset_bytes: int, nbytes: int) -> None:
        if offset_bytes < 0 or nbytes < 0 or offset_bytes + nbytes > self.nbytes:
            raise ValueError("commit range exceeds the host buffer")
        check(lib().dos_host_commit(self.address, int(offset_bytes), int(nbytes)))

    @property
    def committed_bytes(self) -> int:
        n = lib().dos_host_committed(self.address)
        check(int(n) if n < 0 else 0)
        return int(n)

    def array(self, dtype, count: int, offset_bytes: int = 0) -> np.ndarray:
        dt = np.dtype(dtype)
        if offset_bytes + dt.itemsize * count > self.nbytes:
            raise ValueError("view exceeds the host buffer")
        buf = (C.c_char * (dt.itemsize * count)).from_address(self.address + offset_bytes)
        buf._dos_owner = self  # the view's base keeps this region alive
        return np.frombuffer(buf, dtype=dt, count=count)

    def __del__(self):
        addr = getattr(self, "address", None)
        if addr and _lib is not None:
            _lib.dos_host_free(addr)
            self.address = None

