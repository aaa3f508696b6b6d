"""Measured update-phase time over (stride, host threads, static ratio) on
one allocated 7B shard.  python tools/phase_sweep.py [params]"""
import json, sys, time
sys.path.insert(0, ".")
import torch
import paper_2410_21316_b200 as D
from paper_2410_21316_b200 import profile_b200
from bench import fill_shard

P = int(float(sys.argv[1])) if len(sys.argv) > 1 else 7_000_000_000
SG = 100_000_000
dev = torch.device("cuda", 0)
opt = D.ShardedOptimizer.allocate(P, SG, lowp="bf16")
opt.to_device(dev)
fill_shard(opt, 7, dev)
prof = profile_b200.measure_profile(quick=True)
hyper = D.AdamHyper()
n = len(opt.subgroups)
out = []
for static in (0.0, 0.2):
    for stride in (1, 2, 3, 4):
        for th in (8, 12, 16):
            D._native.lib().dos_set_host_threads(th)
            plan = D.build_plan(n, stride, static_ratio=static)
            D.execute_plan(opt, plan, prof, hyper)
            t0 = time.perf_counter()
            r = [D.execute_plan(opt, plan, prof, hyper) for _ in range(2)]
            ms = (time.perf_counter() - t0) / 2 * 1e3
            busy = {k.value: v / 1e6 for k, v in r[-1].measured.lane_busy_ns.items()}
            row = {"static": static, "stride": stride, "threads": th, "ms": round(ms, 1),
                   "span_ms": r[-1].measured.span_ns / 1e6, "busy_ms": busy}
            out.append(row)
            print(json.dumps(row), flush=True)
json.dump(out, open("gpurun_out/phase_sweep.json", "w"), indent=1)
