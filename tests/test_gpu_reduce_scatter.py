"""The reduce-scatter fused into the update phase, bit-exact
against the oracle's declared semantics (oracle.reduce_scatter: rank-order
fp32 sum, one rounding, optional averaging scale).  Separate device buffers
on the one B200 stand in for the ranks' IPC-mapped grad buffers; the
two-process IPC version runs in test_gpu_optim_dist.py."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from oracle import optistate_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2410_21316_b200 as D  # noqa: E402
from paper_2410_21316_b200 import _native as N  # noqa: E402
from paper_2410_21316_b200.distributed import GradSources  # noqa: E402

LOWP = {"fp16": N.DOS_F16, "bf16": N.DOS_BF16}
HYPER = D.AdamHyper()


def _rank_grads(n, world, lowp, seed):
    rng = np.random.default_rng(seed)
    return [O.lowp_from_f32(rng.normal(0, 1.0, n).astype(np.float32), lowp).view(np.uint16) for _ in range(world)]


def _dev16(x, n, off, pad=8):
    t = torch.zeros(n + pad, dtype=torch.int16, device="cuda")
    t[off:off + n] = torch.from_numpy(x.view(np.int16))
    return t


@pytest.mark.parametrize("lowp", ["bf16", "fp16"])
@pytest.mark.parametrize("world,self_rank", [(1, 0), (2, 0), (2, 1), (3, 1), (8, 0), (8, 5)])
@pytest.mark.parametrize("n,off", [(5, 0), (4096 * 3 + 77, 0), (1_000_003, 3)])
@pytest.mark.parametrize("avg", [False, True])
def test_k1_fused_reduce_scatter(lowp, world, self_rank, n, off, avg):
    """dos_adam_step_cuda_rs == oracle Adam on oracle.reduce_scatter(grads);
    the local grads are replaced by the reduced ones, the peers' untouched,
    and the working copy is also broadcast to one peer."""
    rng = np.random.default_rng(n + world)
    p = rng.normal(0, 0.02, n).astype(np.float32)
    m = rng.normal(0, 1e-3, n).astype(np.float32)
    v = (rng.random(n) * 1e-4).astype(np.float32)
    grads = _rank_grads(n, world, lowp, 7 * n + world)
    scale = 1.0 / world if avg else 1.0
    red = O.reduce_scatter([g.view(np.float16) if lowp == "fp16" else g for g in grads], lowp, scale)
    rp, rm, rv = p.copy(), m.copy(), v.copy()
    O.adam_step(rp, rm, rv, O.f32_from_lowp(red, lowp), 1e-3, 0.9, 0.999, 1e-8, 3)

    pad = 8
    tp, tm, tv = (torch.zeros(n + pad, dtype=torch.float32, device="cuda") for _ in range(3))
    for t, x in ((tp, p), (tm, m), (tv, v)):
        t[off:off + n] = torch.from_numpy(x)
    tg = [_dev16(g, n, off) for g in grads]
    tw = torch.zeros(n + pad, dtype=torch.int16, device="cuda")
    peer = torch.zeros(n + pad, dtype=torch.int16, device="cuda")
    srcs = (C.c_void_p * world)(*[t.data_ptr() + 2 * off for t in tg])
    peers = (C.c_void_p * 1)(peer.data_ptr() + 2 * off)
    sc = N.scalars(1e-3, 0.9, 0.999, 1e-8, *O.bias_corrections(0.9, 0.999, 3))
    N.check(N.lib().dos_adam_step_cuda_rs(tp.data_ptr() + 4 * off, tm.data_ptr() + 4 * off, tv.data_ptr() + 4 * off,
                                          srcs, world, self_rank, LOWP[lowp], scale, tw.data_ptr() + 2 * off,
                                          LOWP[lowp], peers, 1, n, sc, None))
    torch.cuda.synchronize()
    assert tp[off:off + n].cpu().numpy().tobytes() == rp.tobytes()
    assert tm[off:off + n].cpu().numpy().tobytes() == rm.tobytes()
    assert tv[off:off + n].cpu().numpy().tobytes() == rv.tobytes()
    want_w = O.lowp_from_f32(rp, lowp).view(np.uint16).tobytes()
    assert tw[off:off + n].cpu().numpy().view(np.uint16).tobytes() == want_w
    assert peer[off:off + n].cpu().numpy().view(np.uint16).tobytes() == want_w
    for r, (t, g) in enumerate(zip(tg, grads)):
        got = t[off:off + n].cpu().numpy().view(np.uint16)
        want = red.view(np.uint16) if r == self_rank else g
        assert got.tobytes() == want.tobytes(), f"rank {r} grads"
        assert torch.count_nonzero(t[:off]) == 0 and torch.count_nonzero(t[off + n:]) == 0


@pytest.mark.parametrize("lowp", ["bf16", "fp16"])
@pytest.mark.parametrize("world", [1, 2, 5, 8])
@pytest.mark.parametrize("n,off", [(3, 1), (8 * 1000 + 5, 0), (300_001, 2)])
def test_reduce_scatter_kernel_in_place(lowp, world, n, off):
    grads = _rank_grads(n, world, lowp, 99 + n)
    red = O.reduce_scatter([g.view(np.float16) if lowp == "fp16" else g for g in grads], lowp, 0.5)
    tg = [_dev16(g, n, off) for g in grads]
    srcs = (C.c_void_p * world)(*[t.data_ptr() + 2 * off for t in tg])
    N.check(N.lib().dos_reduce_scatter_cuda(tg[0].data_ptr() + 2 * off, srcs, world, LOWP[lowp], 0.5, n, None))
    torch.cuda.synchronize()
    assert tg[0][off:off + n].cpu().numpy().view(np.uint16).tobytes() == red.view(np.uint16).tobytes()


def test_reduce_scatter_argument_errors():
    t = torch.zeros(16, dtype=torch.int16, device="cuda")
    one = (C.c_void_p * 1)(t.data_ptr())
    sc = N.scalars(1e-3, 0.9, 0.999, 1e-8, *O.bias_corrections(0.9, 0.999, 1))
    f = torch.zeros(16, dtype=torch.float32, device="cuda")
    lib = N.lib()
    assert lib.dos_reduce_scatter_cuda(t.data_ptr(), one, 0, N.DOS_BF16, 1.0, 16, None) == N.DOS_EINVAL
    assert lib.dos_reduce_scatter_cuda(t.data_ptr(), one, 1, N.DOS_F32, 1.0, 16, None) == N.DOS_ETYPE
    assert lib.dos_reduce_scatter_cuda(t.data_ptr(), one, 1, N.DOS_BF16, 0.0, 16, None) == N.DOS_EINVAL
    args = (f.data_ptr(), f.data_ptr(), f.data_ptr(), one, 1)
    assert lib.dos_adam_step_cuda_rs(*args, 1, N.DOS_BF16, 1.0, None, N.DOS_NONE, None, 0, 16, sc, None) == N.DOS_EINVAL
    assert lib.dos_adam_step_cuda_rs(*args, 0, N.DOS_F32, 1.0, None, N.DOS_NONE, None, 0, 16, sc, None) == N.DOS_ETYPE
    assert lib.dos_adam_step_cuda_rs(*args, 0, N.DOS_BF16, 1.0, t.data_ptr(), N.DOS_F16, None, 0, 16, sc,
                                     None) == N.DOS_ETYPE


@pytest.mark.parametrize("stride,ratio", [(2, 0.0), (3, 0.25), (D.ALL_CPU, 0.0), (1, 0.3)])
@pytest.mark.parametrize("world,self_rank,avg", [(2, 1, False), (4, 0, True), (8, 6, False)])
def test_phase_with_fused_reduce_scatter(h100, stride, ratio, world, self_rank, avg):
    """execute_plan(grad_sources=...): fast subgroups reduce inside K1, host
    subgroups on the grad stream before their flush; the whole shard equals
    the oracle phase on the reduced grads, and the device grads hold them."""
    total, sg = 70_003, 7_000
    opt = D.ShardedOptimizer.initialize(total, sg, seed=5, lowp="bf16")
    res = opt.to_device()
    own = opt.grads16.copy()
    others = _rank_grads(total, world, "bf16", 1234)
    grads = [own if r == self_rank else others[r] for r in range(world)]
    scale = 1.0 / world if avg else 1.0
    red = O.reduce_scatter(grads, "bf16", scale)
    peers = [None if r == self_rank else torch.from_numpy(g.view(np.int16)).cuda() for r, g in enumerate(grads)]
    ptrs = tuple(res.grads.data_ptr() if r == self_rank else peers[r].data_ptr() for r in range(world))
    plan = D.build_plan(len(opt.subgroups), stride, ratio)
    D.execute_plan(opt, plan, h100, HYPER, flush_grads=True, grad_sources=GradSources(ptrs, self_rank, scale))
    ref = O.initialize(total, sg, 5, "bf16")
    ref["g"] = red
    O.sequential_oracle(ref)
    assert opt.params32.tobytes() == ref["p"].tobytes()
    assert opt.momentum32.tobytes() == ref["m"].tobytes()
    assert opt.variance32.tobytes() == ref["v"].tobytes()
    assert opt.model16.tobytes() == ref["w"].tobytes()
    assert res.grads.view(torch.int16).cpu().numpy().view(np.uint16).tobytes() == red.tobytes()
    for r, t in enumerate(peers):
        if t is not None:
            assert t.cpu().numpy().view(np.uint16).tobytes() == grads[r].tobytes()


def test_fused_reduce_scatter_requires_in_phase_flush(h100):
    opt = D.ShardedOptimizer.initialize(20_000, 5_000, seed=1, lowp="bf16")
    res = opt.to_device()
    gs = GradSources((res.grads.data_ptr(),), 0, 1.0)
    plan = D.build_plan(4, 2, 0.0)
    with pytest.raises(ValueError):
        D.execute_plan(opt, plan, h100, HYPER, grad_sources=gs)
    bad = GradSources((res.grads.data_ptr() + 2,), 0, 1.0)  # src_g[self] must be dev_g
    with pytest.raises(ValueError):
        D.execute_plan(opt, plan, h100, HYPER, flush_grads=True, grad_sources=bad)


@pytest.mark.parametrize("cfg", ["0,2", "1,1", "1,2"])
def test_rs_pipeline_shapes_and_depths_bit_exact(cfg):
    """Every selectable fused-RS pipeline (DOS_K1_RS=<shape>,<depth>: 512x6
    ring, peer loads 2 tiles ahead) gives the same bits as the default."""
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, DOS_K1_RS=cfg)
    proc = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                           str(Path(__file__)), "-k", "test_k1_fused_reduce_scatter and not fp16-1-0"],
                          cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert proc.returncode == 0 and " passed" in proc.stdout, proc.stdout[-3000:]
