"""A few measured phases on one 7B shard (regression check for host-side changes)."""
import json, sys, time
sys.path.insert(0, ".")
import torch
import paper_2410_21316_b200 as D
from paper_2410_21316_b200 import profile_b200
from bench import fill_shard
P, SG = 7_000_000_000, 100_000_000
dev = torch.device("cuda", 0)
opt = D.ShardedOptimizer.allocate(P, SG, lowp="bf16")
opt.to_device(dev)
fill_shard(opt, 7, dev)
print(json.dumps({"h1_alone": profile_b200.measure_h1(100_000_000), "h1_dma": profile_b200.measure_h1(100_000_000, with_dma=True)}))
prof = profile_b200.measure_profile(quick=True)
hyper = D.AdamHyper()
for static, stride in ((0.0, 3), (0.0, 4), (0.2, 4), (0.2, 5), (0.2, 6)):
    plan = D.build_plan(70, stride, static_ratio=static)
    D.execute_plan(opt, plan, prof, hyper)
    t0 = time.perf_counter()
    r = [D.execute_plan(opt, plan, prof, hyper) for _ in range(3)]
    ms = (time.perf_counter() - t0) / 3 * 1e3
    print(json.dumps({"static": static, "stride": stride, "ms": round(ms, 1),
                      "busy_ms": {k.value: round(v / 1e6, 1) for k, v in r[-1].measured.lane_busy_ns.items()}}), flush=True)
