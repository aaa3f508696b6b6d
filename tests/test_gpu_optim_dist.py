"""ZeRO-3 DeepOptimizerStates with two ranks sharing the box's one B200
(gloo process group, CUDA tensors): reduce-scatter -> sharded update phase
-> overlapped all-gather.  Every rank's shard must equal the oracle's Adam on
(its master chunk, its reduced grads), the reduced grads must equal
oracle.reduce_scatter of every rank's grads (so the fused and the bucketed
reduce-scatter leave the same bits), and all ranks must end with identical
full-model params."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, stride, fused, q, fused_reduce=False, average=False, static_ratio=0.2):
    try:
        import torch.distributed as dist

        from oracle import optistate_oracle as O
        from paper_2410_21316_b200 import get_profile
        from paper_2410_21316_b200.optim import DeepOptimizerStates

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.manual_seed(0)  # identical initial model on every rank
        model = torch.nn.Sequential(torch.nn.Linear(128, 300), torch.nn.GELU(), torch.nn.Linear(300, 50)).cuda().to(
            torch.bfloat16)
        init = torch.cat([p.detach().reshape(-1) for p in model.parameters()]).float().cpu().numpy().copy()
        opt = DeepOptimizerStates(model.parameters(), lr=1e-3, subgroup_size=9_000, profile=get_profile("h100-node"),
                                  stride=stride, static_ratio=static_ratio, process_group=dist.group.WORLD,
                                  fused_gather=fused, fused_reduce=fused_reduce, average_grads=average)
        lay, off = opt.layout, opt.offset
        mine = opt.opt.total_params
        st = {"p": init[off:off + mine].copy(), "m": np.zeros(mine, np.float32), "v": np.zeros(mine, np.float32),
              "w": None, "g": None, "subgroups": O.shard_subgroups(mine, lay.subgroup_size), "step": 0, "lowp": "bf16"}
        st["w"] = O.bf16_from_f32(st["p"])
        torch.manual_seed(100 + rank)  # different data per rank
        ok = True
        for _ in range(3):
            opt.zero_grad()
            x = torch.randn(16, 128, device="cuda", dtype=torch.bfloat16)
            model(x).float().pow(2).mean().backward()
            pre = opt.flat_grad.view(torch.int16).cpu().to(torch.int32)  # every rank's grads before the step
            everyone = [torch.zeros_like(pre) for _ in range(world)]
            dist.all_gather(everyone, pre)
            opt.step()
            st["g"] = opt.res.grads.view(torch.int16).cpu().numpy().view(np.uint16).copy()  # post reduce-scatter
            # the reduce-scatter itself, in either mode: oracle.reduce_scatter of the ranks' grads
            srcs = [e[off:off + mine].to(torch.int16).numpy().view(np.uint16) for e in everyone]
            want_g = O.reduce_scatter(srcs, "bf16", 1.0 / world if average else 1.0)
            ok &= st["g"].tobytes() == want_g.tobytes()
            O.sequential_oracle(st)
            ok &= opt.master_params().tobytes() == st["p"].tobytes()
            ok &= opt.res.model16.view(torch.int16).cpu().numpy().view(np.uint16).tobytes() == st["w"].tobytes()
            full = opt.flat.view(torch.int16).cpu().to(torch.int32)
            gathered = [torch.zeros_like(full) for _ in range(world)]
            dist.all_gather(gathered, full)
            ok &= all(torch.equal(gathered[0], g) for g in gathered[1:])
        q.put((rank, bool(ok), opt.plan.stride))
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        import traceback

        q.put((rank, False, traceback.format_exc()))


@pytest.mark.parametrize("stride,fused,fused_reduce,average,static_ratio", [
    (2, False, False, False, 0.2), ("auto", False, False, False, 0.2), (2, True, False, False, 0.2),
    ("auto", True, False, True, 0.2), (2, True, True, False, 0.2), ("auto", True, True, True, 0.2),
    (3, False, True, False, 0.2), (2, True, True, False, "auto")])
def test_two_rank_zero3_step_matches_oracle(stride, fused, fused_reduce, average, static_ratio):
    """fused: all-gather in K1's epilogue; fused_reduce: reduce-scatter in
    K1's grad load (both over CUDA IPC); otherwise the bucketed collectives."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, stride, fused, q, fused_reduce, average, static_ratio))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res


@pytest.mark.parametrize("stride,fused,fused_reduce,average", [
    (2, True, True, False), (3, True, True, True), (2, False, False, False)])
def test_four_rank_zero3_step_matches_oracle(stride, fused, fused_reduce, average):
    """Four ranks on the one B200: three IPC peers per rank, the local tile at
    every position of the rank-order sum (ranks 1 and 2 sit in the middle)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 4, port, stride, fused, q, fused_reduce, average, 0.2))
             for r in range(4)]
    for p in procs:
        p.start()
    res = [q.get(timeout=400) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res


def _resume_worker(rank, world, port, q):
    try:
        import torch.distributed as dist

        from paper_2410_21316_b200 import get_profile
        from paper_2410_21316_b200.optim import DeepOptimizerStates

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.manual_seed(0)
        model = torch.nn.Sequential(torch.nn.Linear(96, 200), torch.nn.GELU(), torch.nn.Linear(200, 40)).cuda().to(
            torch.bfloat16)
        opt = DeepOptimizerStates(model.parameters(), subgroup_size=7_000, profile=get_profile("h100-node"), stride=2,
                                  static_ratio=0.25, process_group=dist.group.WORLD)
        torch.manual_seed(50 + rank)

        def step():
            opt.zero_grad()
            model(torch.randn(8, 96, device="cuda", dtype=torch.bfloat16)).float().pow(2).mean().backward()
            opt.step()

        step()
        step()
        sd = opt.state_dict()
        saved = opt.flat.clone()  # the full model every rank holds at the save
        step()  # perturb every rank's chunk
        moved = not torch.equal(opt.flat.view(torch.int16), saved.view(torch.int16))
        opt.load_state_dict(sd)
        # every rank's copy of EVERY rank's chunk is back at the save, not only its own
        ok = moved and torch.equal(opt.flat.view(torch.int16), saved.view(torch.int16))
        step()  # and training continues from there on every rank alike
        full = opt.flat.view(torch.int16).cpu().to(torch.int32)
        gathered = [torch.zeros_like(full) for _ in range(world)]
        dist.all_gather(gathered, full)
        ok &= all(torch.equal(gathered[0], g) for g in gathered[1:])
        q.put((rank, bool(ok), ""))
        dist.destroy_process_group()
    except Exception:
        import traceback

        q.put((rank, False, traceback.format_exc()))


def test_two_rank_resume_republishes_every_chunk():
    """load_state_dict at world 2: the rewritten chunk reaches every rank's
    full-model buffer right away (peers kept stale params until
    the next step's all-gather)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_resume_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
