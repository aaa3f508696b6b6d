"""DeepOptimizerStates: a real (small) bf16 model trained through the B200
update phase; every step's params equal the oracle's Adam on fp32 masters."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import optistate_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
from paper_2410_21316_b200 import get_profile  # noqa: E402
from paper_2410_21316_b200.optim import DeepOptimizerStates  # noqa: E402


def _model():
    torch.manual_seed(0)
    return torch.nn.Sequential(torch.nn.Linear(256, 512), torch.nn.GELU(), torch.nn.Linear(512, 64)).cuda().to(
        torch.bfloat16)


@pytest.mark.parametrize("stride", [1, 2, 3])
def test_training_steps_match_oracle(stride):
    model = _model()
    masters = torch.cat([p.detach().float().reshape(-1).cpu() for p in model.parameters()]).numpy().copy()
    opt = DeepOptimizerStates(model.parameters(), lr=1e-3, subgroup_size=20_000, profile=get_profile("h100-node"),
                              stride=stride, static_ratio=0.2)
    total = masters.size
    st = {"p": masters.copy(), "m": np.zeros(total, np.float32), "v": np.zeros(total, np.float32),
          "w": O.bf16_from_f32(masters), "g": None, "subgroups": O.shard_subgroups(total, 20_000), "step": 0,
          "lowp": "bf16"}
    x = torch.randn(32, 256, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        opt.zero_grad()
        loss = model(x).float().pow(2).mean()
        loss.backward()
        g = torch.cat([p.grad.reshape(-1) for p in model.parameters()]).view(torch.int16).cpu().numpy().view(np.uint16)
        st["g"] = g.copy()
        opt.step()
        O.sequential_oracle(st)
        got = torch.cat([p.detach().reshape(-1) for p in model.parameters()]).view(torch.int16).cpu().numpy()
        assert got.view(np.uint16).tobytes() == st["w"].tobytes()
        assert opt.master_params().tobytes() == st["p"].tobytes()
    assert opt.step_count == 3
