"""Soak test: many consecutive 7B update phases (20% resident, residents
first, measured-best stride, alternating device / host-buffer / in-phase
flush modes); before every step two sampled subgroups of different kinds are
snapshotted and after it compared bit for bit with the C oracle.  Catches
rare races in the engine (slot reuse, event chaining) that short tests miss.
  python tools/soak.py [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2410_21316_b200 as D  # noqa: E402
from bench import fill_shard  # noqa: E402
from oracle import c_oracle  # noqa: E402
from paper_2410_21316_b200 import profile_b200  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
P, SG = 7_000_000_000, 100_000_000
dev = torch.device("cuda", 0)
rng = np.random.default_rng(5)
plan = D.build_plan(70, 4, static_ratio=0.2, placement=D.Placement.STATIC_FIRST)
opt = D.ShardedOptimizer.allocate(P, SG, lowp="bf16", host_homed=[i for i in range(70) if i not in plan.static_set])
res = opt.to_device(dev)
res.set_static(plan.static_set)
fill_shard(opt, 11, dev)
prof = profile_b200.measure_profile(quick=True)
hyper = D.AdamHyper()
kinds = {"static": sorted(plan.static_set), "host": [i for i, d in enumerate(plan.devices) if d is D.Device.CPU],
         "streamed": list(plan.dynamic_fast)}


def bits(t):
    return t.detach().view(torch.int32 if t.element_size() == 4 else torch.int16).cpu().numpy().copy()


def home(i):
    g = opt.subgroups[i]
    if i in res.static_set:
        return tuple(bits(t) for t in res.static_views(i))
    return tuple(a[g.slice].view(np.int32).copy() for a in (opt._p, opt._m, opt._v))


bad, times = [], []
for step in range(steps):
    mode = ("device", "host_io", "flush")[step % 3]
    names = list(kinds)
    pick = [int(rng.choice(kinds[names[(step + j) % 3]])) for j in range(2)]
    g_src = (opt._g if mode == "host_io" else None)
    snap = {}
    for i in pick:
        sl = opt.subgroups[i].slice
        g = g_src[sl].copy() if g_src is not None else bits(res.grads[sl]).view(np.uint16)
        snap[i] = (home(i), g)
    t0 = time.perf_counter()
    D.execute_plan(opt, plan, prof, hyper, host_io=mode == "host_io", flush_grads=mode == "flush")
    times.append((mode, round((time.perf_counter() - t0) * 1e3, 1)))
    for i in pick:
        (p, m, v), g = snap[i]
        p, m, v = (x.view(np.float32) for x in (p, m, v))
        w = np.empty(p.size, dtype=np.uint16)
        c_oracle.adam_mt(p, m, v, g.view(np.uint16), "bf16", w, "bf16", hyper.lr, hyper.beta1, hyper.beta2, hyper.eps,
                         opt.step)
        got = home(i)
        gw = (opt._w[opt.subgroups[i].slice].copy() if mode == "host_io"
              else bits(res.model16[opt.subgroups[i].slice]).view(np.uint16))
        ok = all(np.array_equal(a, b.view(np.int32)) for a, b in zip(got, (p, m, v))) and np.array_equal(gw, w)
        if not ok:
            bad.append({"step": step, "mode": mode, "subgroup": i})
print(json.dumps({"steps": steps, "mismatches": bad, "checked_subgroups": 2 * steps, "phase_ms": times}))
