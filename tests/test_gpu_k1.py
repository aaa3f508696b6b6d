"""K1 (sm_100a fused Adam) and the device conversions, bit-exact against the
oracle.  Runs on the B200 (marker: gpu)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import optistate_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2410_21316_b200 as D  # noqa: E402
from paper_2410_21316_b200 import _native as N  # noqa: E402

DT = {"fp32": N.DOS_F32, "fp16": N.DOS_F16, "bf16": N.DOS_BF16, None: N.DOS_NONE}


def _inputs(n, seed):
    rng = np.random.default_rng(seed)
    return (rng.normal(0, 0.02, n).astype(np.float32), rng.normal(0, 1e-3, n).astype(np.float32),
            (rng.random(n) * 1e-4).astype(np.float32), rng.normal(0, 1.0, n).astype(np.float32))


def _grads_of(g32, kind):
    if kind == "fp32":
        return g32, g32
    g = O.lowp_from_f32(g32, kind)
    return g.view(np.uint16), O.f32_from_lowp(g, kind)


def _run_k1(p, m, v, g, gkind, lowp, n, off, hyper, step, wd=0.0):
    dev = torch.device("cuda")
    pad = 8
    tp = torch.zeros(n + pad, dtype=torch.float32, device=dev)
    tm, tv = torch.zeros_like(tp), torch.zeros_like(tp)
    gd = torch.float32 if gkind == "fp32" else torch.int16
    tg = torch.zeros(n + pad, dtype=gd, device=dev)
    tw = torch.zeros(n + pad, dtype=torch.int16, device=dev)
    tp[off:off + n] = torch.from_numpy(p)
    tm[off:off + n] = torch.from_numpy(m)
    tv[off:off + n] = torch.from_numpy(v)
    tg[off:off + n] = torch.from_numpy(g if gkind == "fp32" else g.view(np.int16))
    bc1, bc2 = O.bias_corrections(hyper[1], hyper[2], step)
    sc = N.scalars(*hyper, bc1, bc2, wd)
    es = {"fp32": 4, "fp16": 2, "bf16": 2}[gkind]
    N.check(N.lib().dos_adam_step_cuda(tp.data_ptr() + 4 * off, tm.data_ptr() + 4 * off, tv.data_ptr() + 4 * off,
                                       tg.data_ptr() + es * off, DT[gkind],
                                       tw.data_ptr() + 2 * off if lowp else None, DT[lowp], n, sc,
                                       torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    out = [t[off:off + n].cpu().numpy() for t in (tp, tm, tv)]
    w = tw[off:off + n].cpu().numpy().view(np.uint16) if lowp else None
    # guard bands untouched
    assert torch.count_nonzero(tp[:off]) == 0 and torch.count_nonzero(tp[off + n:]) == 0
    return (*out, w)


@pytest.mark.parametrize("gkind", ["fp32", "fp16", "bf16"])
@pytest.mark.parametrize("lowp", [None, "fp16", "bf16"])
@pytest.mark.parametrize("n,off", [(1, 0), (7, 3), (8, 0), (9, 1), (1000, 5), (65_537, 2), (1 << 20, 0), (1_000_003, 7)])
def test_k1_bit_exact(gkind, lowp, n, off):
    p, m, v, g32 = _inputs(n, n + off)
    g, gw = _grads_of(g32, gkind)
    hyper = (1e-3, 0.9, 0.999, 1e-8)
    rp, rm, rv = p.copy(), m.copy(), v.copy()
    O.adam_step(rp, rm, rv, gw, *hyper, 3)
    gp, gm, gv, gwc = _run_k1(p, m, v, g, gkind, lowp, n, off, hyper, 3)
    assert gp.tobytes() == rp.tobytes()
    assert gm.tobytes() == rm.tobytes()
    assert gv.tobytes() == rv.tobytes()
    if lowp:
        assert gwc.tobytes() == O.lowp_from_f32(rp, lowp).view(np.uint16).tobytes()


@pytest.mark.parametrize("step,hyper,wd", [(1, (3e-4, 0.8, 0.95, 1e-6), 0.0), (1000, (1e-2, 0.95, 0.9995, 1e-9), 0.0),
                                           (5, (1e-3, 0.9, 0.999, 1e-8), 0.1)])
def test_k1_hyper_and_adamw(step, hyper, wd):
    n = 300_001
    p, m, v, g32 = _inputs(n, step)
    g, gw = _grads_of(g32, "bf16")
    rp, rm, rv = p.copy(), m.copy(), v.copy()
    O.adam_step(rp, rm, rv, gw, *hyper, step, weight_decay=wd)
    gp, gm, gv, gwc = _run_k1(p, m, v, g, "bf16", "bf16", n, 0, hyper, step, wd)
    assert gp.tobytes() == rp.tobytes() and gm.tobytes() == rm.tobytes() and gv.tobytes() == rv.tobytes()
    assert gwc.tobytes() == O.bf16_from_f32(rp).tobytes()


def test_k1_full_subgroup_size():
    n = 100_000_000  # one 1e8-param subgroup (the paper's subgroup size)
    p, m, v, g32 = _inputs(n, 1)
    g, gw = _grads_of(g32, "bf16")
    rp, rm, rv = p.copy(), m.copy(), v.copy()
    O.adam_step(rp, rm, rv, gw, 1e-3, 0.9, 0.999, 1e-8, 2)
    gp, gm, gv, gwc = _run_k1(p, m, v, g, "bf16", "bf16", n, 0, (1e-3, 0.9, 0.999, 1e-8), 2)
    assert np.array_equal(gp.view(np.uint32), rp.view(np.uint32))
    assert np.array_equal(gm.view(np.uint32), rm.view(np.uint32))
    assert np.array_equal(gv.view(np.uint32), rv.view(np.uint32))
    assert np.array_equal(gwc, O.bf16_from_f32(rp))


def test_adam_step_arrays_on_cuda_tensors():
    n = 123_457
    p, m, v, g = _inputs(n, 4)
    rp, rm, rv = p.copy(), m.copy(), v.copy()
    O.adam_step(rp, rm, rv, g, 1e-3, 0.9, 0.999, 1e-8, 2)
    tp, tm, tv, tg = (torch.from_numpy(x).cuda() for x in (p, m, v, g))
    w = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    D.adam_step_arrays(tp, tm, tv, tg, 1e-3, 0.9, 0.999, 1e-8, 2, p_lowp=w)
    assert tp.cpu().numpy().tobytes() == rp.tobytes() and tv.cpu().numpy().tobytes() == rv.tobytes()
    assert w.view(torch.int16).cpu().numpy().view(np.uint16).tobytes() == O.bf16_from_f32(rp).tobytes()
    with pytest.raises(TypeError):
        D.adam_step_arrays(tp, tm, tv, tg.half(), 1e-3, 0.9, 0.999, 1e-8, 2)


def test_device_conversions_exact():
    rng = np.random.default_rng(3)
    x = rng.integers(0, 2**32, 1 << 22, dtype=np.uint32).view(np.float32)
    tx = torch.from_numpy(x).cuda()
    for kind, code in (("fp16", N.DOS_F16), ("bf16", N.DOS_BF16)):
        out = torch.empty(x.size, dtype=torch.int16, device="cuda")
        N.check(N.lib().dos_downscale_cuda(tx.data_ptr(), out.data_ptr(), code, x.size, None))
        torch.cuda.synchronize()
        want = O.lowp_from_f32(x, kind).view(np.uint16)
        assert np.array_equal(out.cpu().numpy().view(np.uint16), want)
        allb = torch.arange(-32768, 32768, dtype=torch.int32).to(torch.int16).cuda()
        up = torch.empty(65536, dtype=torch.float32, device="cuda")
        N.check(N.lib().dos_upscale_cuda(allb.data_ptr(), code, up.data_ptr(), 65536, None))
        torch.cuda.synchronize()
        ref = O.f32_from_lowp(allb.cpu().numpy().view(np.uint16).view(np.float16) if kind == "fp16"
                              else allb.cpu().numpy().view(np.uint16), kind)
        assert up.cpu().numpy().view(np.uint32).tobytes() == ref.view(np.uint32).tobytes()


@pytest.mark.parametrize("npeers", [1, 3, 7])
@pytest.mark.parametrize("n,off", [(5, 0), (4096 * 3 + 77, 0), (1_000_003, 3)])
def test_k1_fused_broadcast_to_peers(npeers, n, off):
    """dos_adam_step_cuda_bcast: every peer destination receives exactly the
    local working copy (local buffers stand in for IPC-mapped peers)."""
    p, m, v, g32 = _inputs(n, 11 + n)
    g = O.bf16_from_f32(g32)
    rp, rm, rv = p.copy(), m.copy(), v.copy()
    O.adam_step(rp, rm, rv, O.f32_from_bf16(g), 1e-3, 0.9, 0.999, 1e-8, 2)
    dev = torch.device("cuda")
    pad = 8
    tp, tm, tv = (torch.zeros(n + pad, dtype=torch.float32, device=dev) for _ in range(3))
    tg = torch.zeros(n + pad, dtype=torch.int16, device=dev)
    tw = torch.zeros(n + pad, dtype=torch.int16, device=dev)
    peers = [torch.zeros(n + pad, dtype=torch.int16, device=dev) for _ in range(npeers)]
    for t, x in ((tp, p), (tm, m), (tv, v)):
        t[off:off + n] = torch.from_numpy(x)
    tg[off:off + n] = torch.from_numpy(g.view(np.int16))
    import ctypes as C

    arr = (C.c_void_p * npeers)(*[q.data_ptr() + 2 * off for q in peers])
    sc = N.scalars(1e-3, 0.9, 0.999, 1e-8, *O.bias_corrections(0.9, 0.999, 2))
    N.check(N.lib().dos_adam_step_cuda_bcast(tp.data_ptr() + 4 * off, tm.data_ptr() + 4 * off, tv.data_ptr() + 4 * off,
                                             tg.data_ptr() + 2 * off, N.DOS_BF16, tw.data_ptr() + 2 * off, N.DOS_BF16,
                                             arr, npeers, n, sc, None))
    torch.cuda.synchronize()
    want = O.bf16_from_f32(rp).tobytes()
    assert tp[off:off + n].cpu().numpy().tobytes() == rp.tobytes()
    assert tw[off:off + n].cpu().numpy().view(np.uint16).tobytes() == want
    for q in peers:
        assert q[off:off + n].cpu().numpy().view(np.uint16).tobytes() == want
        assert torch.count_nonzero(q[:off]) == 0 and torch.count_nonzero(q[off + n:]) == 0


@pytest.mark.parametrize("gkind", ["fp32", "bf16"])
def test_k1_non_finite_grads(gkind):
    """Non-finite inputs (overflowed or NaN grads, an infinite moment): every
    finite result is bit-identical to the oracle, and NaN appears exactly
    where the oracle has NaN.  (The NaN *bit patterns* are not compared: the
    GPU returns the canonical NaN while x86 propagates payloads — the
    reference pins payloads only for its conversions.)"""
    n = 4096 * 3 + 77
    p, m, v, g32 = _inputs(n, 11)
    rng = np.random.default_rng(12)
    idx = rng.choice(n, 200, replace=False)
    g32[idx[:50]] = np.inf
    g32[idx[50:100]] = -np.inf
    g32[idx[100:150]] = np.nan
    g32[idx[150:175]] = 3e38  # finite, but g*g overflows in fp32
    m[idx[175:]] = np.inf
    g, gw = _grads_of(g32, gkind)
    hyper = (1e-3, 0.9, 0.999, 1e-8)
    got = _run_k1(p.copy(), m.copy(), v.copy(), g, gkind, "bf16", n, 0, hyper, 3)
    wp, wm, wv = p.copy(), m.copy(), v.copy()
    O.adam_step(wp, wm, wv, gw, *hyper, 3)
    for a, b in zip(got[:3], (wp, wm, wv)):
        nan_a, nan_b = np.isnan(a), np.isnan(b)
        assert np.array_equal(nan_a, nan_b)
        assert np.array_equal(a[~nan_a].view(np.uint32), b[~nan_b].view(np.uint32))
    assert np.isnan(wp).any() and np.isinf(wm).any()  # the cases really happened
