"""ZeRO-3 on distinct B200s: one process per GPU over NCCL (the product
configuration), in every reduce-scatter / all-gather mode — the fused ones
over CUDA IPC peer memory (NVLink), the bucketed ones over NCCL.

Each rank's shard must equal the oracle's Adam on (its master chunk, the
oracle's reduce-scatter of every rank's grads), the reduced grads must be
bit-identical across modes (oracle.reduce_scatter's rule), and every rank
must end with the same full model.  Skipped where fewer GPUs are visible
(the gloo runs on one shared GPU, tests/test_gpu_optim_dist.py, cover the
same code paths there)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _ngpu() -> int:
    try:
        return torch.cuda.device_count()
    except Exception:
        return 0


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fused_gather, fused_reduce, average, static_ratio, q):
    try:
        import torch.distributed as dist

        from oracle import optistate_oracle as O
        from paper_2410_21316_b200 import get_profile
        from paper_2410_21316_b200.optim import DeepOptimizerStates

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        torch.manual_seed(0)  # identical initial model on every rank
        model = torch.nn.Sequential(torch.nn.Linear(128, 300), torch.nn.GELU(), torch.nn.Linear(300, 50)).to(
            dev).to(torch.bfloat16)
        init = torch.cat([p.detach().reshape(-1) for p in model.parameters()]).float().cpu().numpy().copy()
        opt = DeepOptimizerStates(model.parameters(), lr=1e-3, subgroup_size=9_000, profile=get_profile("h100-node"),
                                  stride=2, static_ratio=static_ratio, process_group=dist.group.WORLD,
                                  fused_gather=fused_gather, fused_reduce=fused_reduce, average_grads=average)
        off, mine = opt.offset, opt.opt.total_params
        st = {"p": init[off:off + mine].copy(), "m": np.zeros(mine, np.float32), "v": np.zeros(mine, np.float32),
              "w": None, "g": None, "subgroups": O.shard_subgroups(mine, opt.layout.subgroup_size), "step": 0,
              "lowp": "bf16"}
        st["w"] = O.bf16_from_f32(st["p"])
        torch.manual_seed(100 + rank)  # different data per rank
        ok, why = True, []
        for it in range(3):
            opt.zero_grad()
            x = torch.randn(16, 128, device=dev, dtype=torch.bfloat16)
            model(x).float().pow(2).mean().backward()
            pre = opt.flat_grad.view(torch.int16).to(torch.int32)
            everyone = [torch.zeros_like(pre) for _ in range(world)]
            dist.all_gather(everyone, pre)
            opt.step()
            st["g"] = opt.res.grads.view(torch.int16).cpu().numpy().view(np.uint16).copy()
            srcs = [e[off:off + mine].cpu().to(torch.int16).numpy().view(np.uint16) for e in everyone]
            if st["g"].tobytes() != O.reduce_scatter(srcs, "bf16", 1.0 / world if average else 1.0).tobytes():
                ok, _ = False, why.append(f"step {it}: reduced grads differ from oracle.reduce_scatter")
            O.sequential_oracle(st)
            if opt.master_params().tobytes() != st["p"].tobytes():
                ok, _ = False, why.append(f"step {it}: fp32 params differ")
            if opt.res.model16.view(torch.int16).cpu().numpy().view(np.uint16).tobytes() != st["w"].tobytes():
                ok, _ = False, why.append(f"step {it}: working copy differs")
            full = opt.flat.view(torch.int16).to(torch.int32)
            gathered = [torch.zeros_like(full) for _ in range(world)]
            dist.all_gather(gathered, full)
            if not all(torch.equal(gathered[0], g) for g in gathered[1:]):
                ok, _ = False, why.append(f"step {it}: ranks hold different models")
        q.put((rank, ok, "; ".join(why)))
        dist.destroy_process_group()
    except Exception:
        import traceback

        q.put((rank, False, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("fused_gather,fused_reduce,average,static_ratio", [
    (True, True, False, 0.2), (False, False, False, 0.2), (True, False, True, 0.0), (False, True, True, 0.2)])
def test_zero3_on_distinct_gpus_nccl(world, fused_gather, fused_reduce, average, static_ratio):
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs, {_ngpu()} visible")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fused_gather, fused_reduce, average, static_ratio, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
