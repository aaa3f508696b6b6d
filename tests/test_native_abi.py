"""libdos.so: loads without a GPU, exports every include/dos.h symbol, maps
errors to the reference's exception types, and H1 (host) is bit-exact."""
from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

from oracle import optistate_oracle as O
import paper_2410_21316_b200 as D
from paper_2410_21316_b200 import _native as N

HEADER = Path(__file__).resolve().parent.parent / "include" / "dos.h"


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    declared = set(re.findall(r"\b(dos_[a-z0-9_]+)\s*\(", HEADER.read_text()))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(N.SIGNATURES), declared ^ set(N.SIGNATURES)
    assert lib.dos_version() >= 1


def test_error_codes_map_to_reference_exceptions():
    lib = N.lib()
    sc = N.scalars(1e-3, 0.9, 0.999, 1e-8, 0.1, 0.001)
    x = np.zeros(4, np.float32)
    with pytest.raises(TypeError):
        N.check(lib.dos_adam_step_host(x.ctypes.data, x.ctypes.data, x.ctypes.data, x.ctypes.data, 7, None, -1, 4, sc, 0))
    with pytest.raises(ValueError):
        N.check(lib.dos_adam_step_host(x.ctypes.data, x.ctypes.data, x.ctypes.data, x.ctypes.data, 0, None, -1, -1, sc, 0))
    with pytest.raises(ValueError):
        N.check(lib.dos_host_free(12345))


def _state(n, seed):
    rng = np.random.default_rng(seed)
    p = rng.normal(0, 0.02, n).astype(np.float32)
    m = rng.normal(0, 1e-3, n).astype(np.float32)
    v = (rng.random(n) * 1e-4).astype(np.float32)
    g = rng.normal(0, 1.0, n).astype(np.float32)
    return p, m, v, g


@pytest.mark.parametrize("n", [0, 1, 7, 64, 1000, 65_537, 300_001])
@pytest.mark.parametrize("step", [1, 7])
def test_adam_step_arrays_host_bit_exact(n, step):
    p, m, v, g = _state(n, n + step)
    rp, rm, rv = p.copy(), m.copy(), v.copy()
    D.adam_step_arrays(p, m, v, g, 1e-3, 0.9, 0.999, 1e-8, step)
    if n:
        O.adam_step(rp, rm, rv, g, 1e-3, 0.9, 0.999, 1e-8, step)
    assert p.tobytes() == rp.tobytes() and m.tobytes() == rm.tobytes() and v.tobytes() == rv.tobytes()


def test_host_adam_non_finite_inputs():
    """H1 with overflowed / NaN grads and infinite moments: finite results
    bit-exact, NaN at the oracle's positions (NaN bits are not compared)."""
    import warnings

    n = 100_003
    p, m, v, g = _state(n, 5)
    rng = np.random.default_rng(6)
    idx = rng.choice(n, 400, replace=False)
    g[idx[:100]] = np.inf
    g[idx[100:200]] = np.nan
    g[idx[200:300]] = 3e38
    m[idx[300:]] = -np.inf
    rp, rm, rv = p.copy(), m.copy(), v.copy()
    D.adam_step_arrays(p, m, v, g, 1e-3, 0.9, 0.999, 1e-8, 2)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        O.adam_step(rp, rm, rv, g, 1e-3, 0.9, 0.999, 1e-8, 2)
    for a, b in ((p, rp), (m, rm), (v, rv)):
        assert np.array_equal(np.isnan(a), np.isnan(b))
        ok = ~np.isnan(a)
        assert a[ok].tobytes() == b[ok].tobytes()
    assert np.isnan(rp).any()


@pytest.mark.parametrize("lowp", ["fp16", "bf16"])
@pytest.mark.parametrize("wd", [0.0, 0.01])
def test_host_fused_lowp_grads_and_working_copy(lowp, wd):
    n = 200_003
    p, m, v, g32 = _state(n, 9)
    g = O.lowp_from_f32(g32, lowp)
    w = np.empty(n, dtype=np.uint16)
    rp, rm, rv = p.copy(), m.copy(), v.copy()
    sc = N.scalars(3e-4, 0.85, 0.99, 1e-7, *O.bias_corrections(0.85, 0.99, 4), weight_decay=wd)
    N.check(N.lib().dos_adam_step_host(p.ctypes.data, m.ctypes.data, v.ctypes.data, g.ctypes.data,
                                       N.LOWP_CODES[lowp], w.ctypes.data, N.LOWP_CODES[lowp], n, sc, 0))
    O.adam_step(rp, rm, rv, O.f32_from_lowp(g, lowp), 3e-4, 0.85, 0.99, 1e-7, 4, weight_decay=wd)
    assert p.tobytes() == rp.tobytes() and m.tobytes() == rm.tobytes() and v.tobytes() == rv.tobytes()
    assert w.tobytes() == O.lowp_from_f32(rp, lowp).view(np.uint16).tobytes()


def test_adam_step_arrays_validation():
    p, m, v, g = _state(4, 0)
    with pytest.raises(ValueError):
        D.adam_step_arrays(p, m, v, g, 1e-3, 0.9, 0.999, 1e-8, 0)
    with pytest.raises(TypeError):
        D.adam_step_arrays(p.astype(np.float64), m, v, g, 1e-3, 0.9, 0.999, 1e-8, 1)
    with pytest.raises(TypeError):
        D.adam_step_arrays(p, m, v, g.astype(np.float16), 1e-3, 0.9, 0.999, 1e-8, 1)
    with pytest.raises(ValueError):
        D.adam_step_arrays(p, m, v, g[:2], 1e-3, 0.9, 0.999, 1e-8, 1)


def test_backend_env_flag(tmp_path):
    import os
    import subprocess
    import sys

    root = str(Path(__file__).resolve().parent.parent)
    ok = subprocess.run([sys.executable, "-c", "import paper_2410_21316_b200.kernels as k; assert k.active_backend()=='native'"],
                        env=dict(os.environ, OPTISTATE_BACKEND="numpy", PYTHONPATH=root), capture_output=True, text=True)
    assert ok.returncode == 0, ok.stderr
    bad = subprocess.run([sys.executable, "-c", "import paper_2410_21316_b200.kernels"],
                         env=dict(os.environ, OPTISTATE_BACKEND="cuda", PYTHONPATH=root), capture_output=True, text=True)
    assert bad.returncode != 0 and "OPTISTATE_BACKEND" in bad.stderr


def test_downscale_matches_golden_bits_including_nan_payloads():
    d = np.load(Path(__file__).resolve().parent / "golden" / "fp16_vectors.npz")
    got = D.downscale_rne(d["f32_bits"].view(np.float32)).view(np.uint16)
    assert np.array_equal(got, d["f16_bits"])


def test_fp16_roundtrip_exhaustive():
    all16 = np.arange(2**16, dtype=np.uint16)
    back = D.downscale_rne(D.upscale(all16.view(np.float16))).view(np.uint16)
    assert np.array_equal(all16, back)
    # widening equals numpy's, payloads included
    assert D.upscale(all16.view(np.float16)).view(np.uint32).tobytes() == all16.view(np.float16).astype(np.float32).view(np.uint32).tobytes()


def test_bf16_conversions_match_oracle():
    rng = np.random.default_rng(5)
    x = rng.integers(0, 2**32, 500_000, dtype=np.uint32).view(np.float32)
    assert np.array_equal(D.downscale_bf16(x), O.bf16_from_f32(x))
    b = np.arange(2**16, dtype=np.uint16)
    assert D.upscale_bf16(b).view(np.uint32).tobytes() == O.f32_from_bf16(b).view(np.uint32).tobytes()


def test_conversion_type_errors():
    with pytest.raises(TypeError):
        D.downscale_rne(np.zeros(3, dtype=np.float64))
    with pytest.raises(TypeError):
        D.upscale(np.zeros(3, dtype=np.float32))


def test_pinned_pool_alloc_roundtrip():
    buf = N.HostBuffer(3 << 20, register_cuda=False)
    a = buf.array(np.float32, 1000)
    a[:] = np.arange(1000, dtype=np.float32)
    assert a.sum() == np.arange(1000, dtype=np.float32).sum()
    assert a.ctypes.data % 4096 == 0


def test_team_resize_while_h1_runs():
    """dos_set_host_threads while another thread is inside an H1 section:
    the running section keeps its team (no use-after-free) and every result
    stays bit-exact (dos_host.cpp team lifetime)."""
    import threading

    n = 1 << 20
    rng = np.random.default_rng(5)
    p0, m0, g = (rng.normal(0, s, n).astype(np.float32) for s in (0.02, 1e-3, 1.0))
    v0 = (rng.random(n) * 1e-4).astype(np.float32)
    want = [x.copy() for x in (p0, m0, v0)]
    O.adam_step(*want, g, 1e-3, 0.9, 0.999, 1e-8, 1)
    errors, stop = [], threading.Event()

    def work():
        try:
            while not stop.is_set():
                p, m, v = p0.copy(), m0.copy(), v0.copy()
                D.adam_step_arrays(p, m, v, g, 1e-3, 0.9, 0.999, 1e-8, 1)
                if p.tobytes() != want[0].tobytes() or v.tobytes() != want[2].tobytes():
                    errors.append("mismatch")
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    th = threading.Thread(target=work)
    th.start()
    try:
        for i in range(40):
            N.check(N.lib().dos_set_host_threads(1 + i % 4))
    finally:
        stop.set()
        th.join(timeout=120)
    N.check(N.lib().dos_set_host_threads(0))
    assert not th.is_alive() and not errors, errors


@pytest.mark.parametrize("knob", ["DOS_H1_NT=all", "DOS_H1_WSTORE=cached", "DOS_H1_PF=0 DOS_H1_CHUNK=0",
                                  "DOS_H1_PF=64 DOS_H1_CHUNK=64", "DOS_H1_PF=8192 DOS_H1_CHUNK=1000", ""])
def test_host_store_variants_bit_exact(knob):
    """The A/B variants of H1 (streaming p/m/v stores; cached working-copy
    stores; prefetch distance and dynamic chunk, incl. chunks that split the
    64-byte store phase) give the same bits, at aligned and misaligned starts."""
    import os
    import subprocess
    import sys

    code = r"""
import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2410_21316_b200 as D
from paper_2410_21316_b200 import _native as N
from oracle import optistate_oracle as O
rng = np.random.default_rng(3)
for n, off in ((1 << 20, 0), (300_001, 5), (4097, 17)):
    p0, m0 = (rng.normal(0, s, n + off).astype(np.float32) for s in (0.02, 1e-3))
    v0 = (rng.random(n + off) * 1e-4).astype(np.float32)
    g = O.lowp_from_f32(rng.normal(0, 1, n + off).astype(np.float32), "bf16").view(np.uint16)
    # page-aligned (pool) buffers, so the 64-byte streaming-store paths run
    hb = N.HostBuffer((n + off) * 16, register_cuda=False)
    p, m, v = (hb.array(np.float32, n + off, k * 4 * (n + off)) for k in range(3))
    w = hb.array(np.uint16, n + off, 12 * (n + off))
    p[:], m[:], v[:], w[:] = p0, m0, v0, 0
    sc = N.scalars(1e-3, 0.9, 0.999, 1e-8, np.float32(1 - 0.9 ** 2), np.float32(1 - 0.999 ** 2))
    N.check(N.lib().dos_adam_step_host(p[off:].ctypes.data, m[off:].ctypes.data, v[off:].ctypes.data,
                                       g[off:].ctypes.data, N.DOS_BF16, w[off:].ctypes.data, N.DOS_BF16, n, sc, 0))
    rp, rm, rv = p0[off:].copy(), m0[off:].copy(), v0[off:].copy()
    O.adam_step(rp, rm, rv, O.f32_from_lowp(g[off:], "bf16"), 1e-3, 0.9, 0.999, 1e-8, 2)
    assert p[off:].tobytes() == rp.tobytes() and m[off:].tobytes() == rm.tobytes() and v[off:].tobytes() == rv.tobytes()
    assert w[off:].tobytes() == O.lowp_from_f32(rp, "bf16").view(np.uint16).tobytes()
print("ok")
"""
    env = dict(os.environ, **dict(kv.split("=") for kv in knob.split()))
    root = Path(__file__).resolve().parent.parent
    proc = subprocess.run([sys.executable, "-c", code], cwd=root, env=env,
                          capture_output=True, text=True, timeout=300)
    assert proc.returncode == 0 and "ok" in proc.stdout, proc.stderr[-3000:]
