"""7B phase (20% resident, residents first) over stride x H1 team size."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2410_21316_b200 as D
from bench import fill_shard
from paper_2410_21316_b200 import profile_b200
P, SG = 7_000_000_000, 100_000_000
dev = torch.device("cuda", 0)
st = D.build_plan(70, 1, static_ratio=0.2, placement=D.Placement.STATIC_FIRST).static_set
opt = D.ShardedOptimizer.allocate(P, SG, lowp="bf16", host_homed=[i for i in range(70) if i not in st])
res = opt.to_device(dev); res.set_static(st); fill_shard(opt, 7, dev)
prof = profile_b200.measure_profile(quick=True)
hy = D.AdamHyper()
out = []
for rep in range(2):
    for stride in (4, 5):
        for th in (16, 15, 14, 12):
            D._native.lib().dos_set_host_threads(th)
            plan = D.build_plan(70, stride, static_ratio=0.2, placement=D.Placement.STATIC_FIRST)
            D.execute_plan(opt, plan, prof, hy)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(2):
                D.execute_plan(opt, plan, prof, hy)
            e1.record(); torch.cuda.synchronize()
            row = {"rep": rep, "stride": stride, "threads": th, "ms": round(e0.elapsed_time(e1) / 2, 1)}
            out.append(row); print(json.dumps(row), flush=True)
