"""The fused Adam step entry point (reference: pkg/src/optistate/kernels.py).

``adam_step_arrays(p, m, v, g, lr, beta1, beta2, eps, step)`` keeps the
reference's signature, validation and exception types (kernels.py:107-139)
and dispatches on where the arrays live:

* numpy arrays      -> H1, ``dos_adam_step_host`` (host team, AVX-512)
* CUDA torch tensors -> K1, ``dos_adam_step_cuda`` (sm_100a) on the current stream

Both are bit-identical to the reference's numba loop.  Backend selection
(kernels.py:36-69) keeps the ``OPTISTATE_BACKEND`` variable: ``auto``,
``native`` and, for compatibility, ``numba``/``numpy`` all select the native
host kernel; any other value (notably ``cuda``) fails at import, as in the
reference (pkg/tests/test_kernels.py:52-59).  The device is chosen by the
arrays, never by the variable.
"""

from __future__ import annotations

import os

import numpy as np

from . import _native as N
from .state import bias_corrections

_ENV_VAR = "OPTISTATE_BACKEND"
_ACCEPTED = ("", "auto", "native", "numba", "numpy")


def _resolve_backend() -> str:
    choice = os.environ.get(_ENV_VAR, "auto").strip().lower()
    if choice not in _ACCEPTED:
        raise ValueError(f"unrecognised {_ENV_VAR}={choice!r} (use auto|native)")
    return "native"


_BACKEND = _resolve_backend()


def active_backend() -> str:
    """Name of the host backend selected at import time."""
    return _BACKEND


def _is_cuda_tensor(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


_TORCH_CODES = None


def _torch_code(t) -> int | None:
    global _TORCH_CODES
    if _TORCH_CODES is None:
        import torch

        _TORCH_CODES = {torch.float32: N.DOS_F32, torch.float16: N.DOS_F16, torch.bfloat16: N.DOS_BF16}
    return _TORCH_CODES.get(t.dtype)


def adam_step_arrays(p, m, v, g, lr, beta1, beta2, eps, step, *, weight_decay: float = 0.0,
                     p_lowp=None) -> None:
    """Fused in-place Adam on flat fp32 arrays (kernels.py:107-139).

    ``p``/``m``/``v`` update in place from fp32 grads ``g``; ``step`` is the
    1-based bias-correction step.  Optional extensions (no reference pin):
    ``weight_decay`` (decoupled, AdamW) and ``p_lowp`` (a float16/bfloat16
    output receiving the updated params in the same pass).
    """
    if step < 1:
        raise ValueError("step must be >= 1 for bias correction")
    bc1, bc2 = bias_corrections(beta1, beta2, step)
    sc = N.scalars(lr, beta1, beta2, eps, bc1, bc2, weight_decay)
    if _is_cuda_tensor(p):
        import torch

        for name, arr in (("p", p), ("m", m), ("v", v), ("g", g)):
            if not _is_cuda_tensor(arr):
                raise TypeError(f"{name} must be a CUDA tensor like p")
            if arr.dtype != torch.float32:
                raise TypeError(f"expected float32 for {name}, got {arr.dtype}")
            if not arr.is_contiguous():
                raise ValueError(f"{name} must be contiguous")
        if not (p.shape == m.shape == v.shape == g.shape) or p.dim() != 1:
            raise ValueError("p, m, v, g must share one flat shape")
        lp_code, lp_ptr = N.DOS_NONE, None
        if p_lowp is not None:
            lp_code = _torch_code(p_lowp)
            if lp_code not in (N.DOS_F16, N.DOS_BF16) or p_lowp.shape != p.shape:
                raise TypeError("p_lowp must be a float16/bfloat16 tensor shaped like p")
            lp_ptr = p_lowp.data_ptr()
        stream = torch.cuda.current_stream(p.device).cuda_stream
        N.check(N.lib().dos_adam_step_cuda(p.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(), N.DOS_F32,
                                           lp_ptr, lp_code, p.numel(), sc, stream))
        return
    for name, arr in (("p", p), ("m", m), ("v", v), ("g", g)):
        if not isinstance(arr, np.ndarray):
            raise TypeError(f"{name} must be a numpy array (or every array a CUDA tensor)")
        if arr.dtype != np.float32:
            raise TypeError(f"expected float32 for {name}, got {arr.dtype}")
    if not (p.shape == m.shape == v.shape == g.shape):
        raise ValueError("p, m, v, g must share one flat shape")
    for name, arr in (("p", p), ("m", m), ("v", v), ("g", g)):
        if not arr.flags.c_contiguous:
            raise ValueError(f"{name} must be contiguous")
    lp_code, lp_ptr = N.DOS_NONE, None
    if p_lowp is not None:
        if p_lowp.dtype == np.float16:
            lp_code = N.DOS_F16
        elif p_lowp.dtype == np.uint16:
            lp_code = N.DOS_BF16
        else:
            raise TypeError("p_lowp must be float16 or uint16 (bf16 bits)")
        if p_lowp.shape != p.shape:
            raise ValueError("p_lowp must be shaped like p")
        lp_ptr = N.ptr(p_lowp)
    N.check(N.lib().dos_adam_step_host(N.ptr(p), N.ptr(m), N.ptr(v), N.ptr(g), N.DOS_F32, lp_ptr, lp_code,
                                       p.size, sc, 0))
