"""Parity at BASELINE's full sizes on the B200: a 7B shard (configs[1], 20%
HBM-resident, stride 5), a 13B shard (configs[2], capacity-aware
residency, sparse host pool) and one rank of 70B/8 (configs[4]: 8.75e9
params, 88 subgroups with a ragged 5e7 tail, 50% resident) run real update
phases; sampled subgroups —
first, last, and one of each kind (static resident, host-updated, streamed
through the GPU) — are snapshotted before the second step and checked bit for
bit against the C oracle (oracle/adam_oracle.c, pinned to the reference) on
the same inputs."""
from __future__ import annotations

import gc

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2410_21316_b200 as D  # noqa: E402
from paper_2410_21316_b200 import get_profile, policy  # noqa: E402

SG = 100_000_000


def _bits(t) -> np.ndarray:
    return t.detach().view(torch.int32 if t.element_size() == 4 else torch.int16).cpu().numpy().copy()


@pytest.mark.parametrize("params, ratio, stride, flush", [(7e9, 0.2, 5, True), (13e9, "auto", 6, False),
                                                          (8.75e9, 0.5, 3, True)])
def test_full_size_sampled_parity(params, ratio, stride, flush):
    """flush: the bench's mode — the host-updated subgroups' grads flushed D2H
    inside the phase, and the checked step asserts coherence over every
    element of every subgroup ("full")."""
    from bench import fill_shard, host_available_bytes
    from oracle import c_oracle

    P = int(params)
    dev = torch.device("cuda", 0)
    gc.collect()
    torch.cuda.empty_cache()
    sizes = [g.size for g in D.shard(P, 1, SG)[0]]
    n = len(sizes)
    r = policy.capacity_static_ratio(sizes, torch.cuda.mem_get_info(dev)[0]) if ratio == "auto" else ratio
    plan = D.build_plan(n, stride, static_ratio=r)
    host_need = 16 * sum(s for i, s in enumerate(sizes) if i not in plan.static_set)
    if host_need > host_available_bytes() - (16 << 30):
        pytest.skip(f"needs {host_need / 1e9:.0f} GB of pinned host memory")
    opt = D.ShardedOptimizer.allocate(P, SG, lowp="bf16",
                                      host_homed=[i for i in range(n) if i not in plan.static_set])
    res = opt.to_device(dev)
    res.set_static(plan.static_set)
    fill_shard(opt, seed=99, device=dev)
    hyper = D.AdamHyper()
    prof = get_profile("b200-node")
    D.execute_plan(opt, plan, prof, hyper)  # step 1

    kinds = {"static": sorted(plan.static_set),
             "host": [i for i, d in enumerate(plan.devices) if d is D.Device.CPU],
             "streamed": [i for i in plan.dynamic_fast]}
    sample = {0, n - 1} | {v[len(v) // 2] for v in kinds.values() if v}
    assert all(kinds.values()), kinds

    def home(i):
        g = opt.subgroups[i]
        if i in res.static_set:
            return tuple(_bits(t) for t in res.static_views(i))
        return tuple(a[g.slice].view(np.int32).copy() for a in (opt._p, opt._m, opt._v))

    snap = {i: (home(i), _bits(res.grads[opt.subgroups[i].slice])) for i in sample}
    step = opt.step + 1
    D.execute_plan(opt, plan, prof, hyper, flush_grads=flush,
                   check_coherence="full" if flush else "sampled")  # step 2 (the checked one)
    torch.cuda.synchronize()
    for i in sorted(sample):
        (p, m, v), g = snap[i]
        p, m, v = (x.view(np.float32) for x in (p, m, v))
        w = np.empty(p.size, dtype=np.uint16)
        c_oracle.adam_mt(p, m, v, g.view(np.uint16), "bf16", w, "bf16", hyper.lr, hyper.beta1, hyper.beta2,
                         hyper.eps, step)
        got_p, got_m, got_v = home(i)
        assert np.array_equal(got_p, p.view(np.int32)), f"subgroup {i} params"
        assert np.array_equal(got_m, m.view(np.int32)), f"subgroup {i} momentum"
        assert np.array_equal(got_v, v.view(np.int32)), f"subgroup {i} variance"
        got_w = _bits(res.model16[opt.subgroups[i].slice]).view(np.uint16)
        assert np.array_equal(got_w, w), f"subgroup {i} working copy"
    del opt, res, snap
    gc.collect()
    torch.cuda.empty_cache()
