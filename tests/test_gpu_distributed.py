"""The overlapped all-gather hook on a real NCCL group (world size 1 on the
one GPU of this box): every bucket gathers the final working copy."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402

import paper_2410_21316_b200 as D  # noqa: E402
from paper_2410_21316_b200.distributed import BucketedCollectives, ShardLayout, gather_params_overlapped  # noqa: E402


@pytest.fixture(scope="module")
def nccl_group():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("stride,ratio", [(2, 0.0), (3, 0.25), (1, 0.0), (D.ALL_CPU, 0.0)])
def test_overlapped_gather_matches_working_copy(nccl_group, h100, stride, ratio):
    total, sg = 90_000, 10_000
    opt = D.ShardedOptimizer.initialize(total, sg, seed=3, lowp="bf16")
    res = opt.to_device()
    lay = ShardLayout.build(total, 1, sg)
    coll = BucketedCollectives(lay)
    full = torch.full((lay.padded_total,), -1.0, dtype=torch.bfloat16, device="cuda")
    plan = D.build_plan(len(opt.subgroups), stride, ratio)
    hook = gather_params_overlapped(coll, plan, res.model16, full)
    D.execute_plan(opt, plan, h100, D.AdamHyper(), on_submitted=hook)
    for w in hook.works:
        if w is not None:
            w.wait()
    torch.cuda.synchronize()
    assert torch.equal(full.view(torch.int16), res.model16.view(torch.int16))
    assert np.array_equal(full.view(torch.int16).cpu().numpy().view(np.uint16), opt.model16)


def test_stream_wait_rejects_host_actions(h100):
    opt = D.ShardedOptimizer.initialize(40_000, 10_000, seed=1, lowp="bf16")
    plan = D.build_plan(4, 2)
    cpu_update = next(a.id for a in plan.actions if a.kind is D.ActionKind.CPU_UPDATE)
    seen = {}

    def hook(target):
        with pytest.raises(ValueError):
            target.stream_wait(cpu_update, torch.cuda.current_stream())
        gpu = next(a.id for a in plan.actions if a.kind is D.ActionKind.GPU_UPDATE)
        target.stream_wait(gpu, torch.cuda.current_stream())
        seen["ok"] = True

    D.execute_plan(opt, plan, h100, D.AdamHyper(), on_submitted=hook)
    assert seen.get("ok")
