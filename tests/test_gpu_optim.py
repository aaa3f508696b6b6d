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
@pytest.mark.parametrize("static_ratio", [0.2, "auto"])
def test_training_steps_match_oracle(stride, static_ratio):
    model = _model()
    masters = torch.cat([p.detach().float().reshape(-1).cpu() for p in model.parameters()]).numpy().copy()
    opt = DeepOptimizerStates(model.parameters(), lr=1e-3, subgroup_size=20_000, profile=get_profile("h100-node"),
                              stride=stride, static_ratio=static_ratio)
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


def test_capacity_aware_state_dict_roundtrip():
    """static_ratio="auto" homes the whole (small) shard in HBM with no host
    state; state_dict/load_state_dict still round-trip it exactly."""
    model = _model()
    opt = DeepOptimizerStates(model.parameters(), subgroup_size=20_000, profile=get_profile("h100-node"),
                              stride=2, static_ratio="auto")
    assert opt.static_ratio == 1.0 and opt.opt.host_bytes == 0
    x = torch.randn(32, 256, device="cuda", dtype=torch.bfloat16)
    for _ in range(2):
        opt.zero_grad()
        model(x).float().pow(2).mean().backward()
        opt.step()
    sd = opt.state_dict()
    assert opt.opt.host_bytes == 0  # exported from HBM without materialising the sparse pool
    before = torch.cat([p.detach().reshape(-1) for p in model.parameters()]).clone()
    opt.load_state_dict(sd)
    assert opt.opt.host_bytes == 0
    after = torch.cat([p.detach().reshape(-1) for p in model.parameters()])
    assert torch.equal(before.view(torch.int16), after.view(torch.int16))
    sd2 = opt.state_dict()
    for k in ("params32", "momentum32", "variance32"):
        assert sd2[k].tobytes() == sd[k].tobytes()


def test_capacity_aware_respects_hbm_budget():
    model = _model()
    n = sum(p.numel() for p in model.parameters())
    # room for two windows of 20k params and two residents: the rest stays on the host
    budget = 2 * 12 * 20_000 + 2 * 12 * 20_000
    opt = DeepOptimizerStates(model.parameters(), subgroup_size=20_000, profile=get_profile("h100-node"),
                              stride=2, static_ratio="auto", hbm_budget_bytes=budget)
    nsg = -(-n // 20_000)
    assert opt.static_ratio == 2 / nsg and len(opt.plan.static_set) == 2
    assert 0 < opt.opt.host_bytes


@pytest.mark.parametrize("static_ratio", [0.0, 0.5])
def test_state_dict_roundtrip_continues_training_exactly(static_ratio):
    """Save after two steps, perturb, load, take a step: identical to taking
    that step straight after the save."""
    def run(load_from=None):
        model = _model()
        opt = DeepOptimizerStates(model.parameters(), subgroup_size=20_000, profile=get_profile("h100-node"),
                                  stride=2, static_ratio=static_ratio)
        x = torch.randn(32, 256, device="cuda", dtype=torch.bfloat16, generator=torch.Generator("cuda").manual_seed(3))
        for _ in range(2):
            opt.zero_grad()
            model(x).float().pow(2).mean().backward()
            opt.step()
        sd = opt.state_dict()
        if load_from is not None:
            # perturb every tier first: an extra step moves p/m/v and the working
            # copy, so only a load that restores all of them can match run A
            opt.zero_grad()
            model(x).float().pow(2).mean().backward()
            opt.step()
            assert opt.state_dict()["momentum32"].tobytes() != load_from["momentum32"].tobytes()
            opt.load_state_dict(load_from)
            assert opt.step_count == load_from["step"]
        opt.zero_grad()
        model(x).float().pow(2).mean().backward()
        opt.step()
        return sd, torch.cat([p.detach().reshape(-1) for p in model.parameters()]).clone(), opt.state_dict()

    sd, params_a, end_a = run()
    _, params_b, end_b = run(load_from=sd)
    assert torch.equal(params_a.view(torch.int16), params_b.view(torch.int16))
    for k in ("params32", "momentum32", "variance32"):
        assert end_a[k].tobytes() == end_b[k].tobytes()


def test_replaced_grads_are_refused():
    """model.zero_grad() (set_to_none=True) detaches .grad from the flat
    buffer: step() refuses instead of updating with stale grads."""
    model = _model()
    opt = DeepOptimizerStates(model.parameters(), subgroup_size=20_000, profile=get_profile("h100-node"), stride=2)
    x = torch.randn(8, 256, device="cuda", dtype=torch.bfloat16)
    model(x).float().pow(2).mean().backward()
    opt.step()
    model.zero_grad()  # torch 2.x default: set_to_none=True
    model(x).float().pow(2).mean().backward()
    with pytest.raises(RuntimeError, match="no longer aliases"):
        opt.step()
