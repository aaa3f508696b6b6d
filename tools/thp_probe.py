"""THP behaviour of the pinned pool on this box: vmstat THP/compaction
counters around a 90 GB sparse-pool allocation and a few 7B phases."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_21316_b200 as D  # noqa: E402
from bench import fill_shard  # noqa: E402
from paper_2410_21316_b200 import profile_b200  # noqa: E402

KEYS = ("thp_fault_alloc", "thp_fault_fallback", "thp_collapse_alloc", "thp_collapse_alloc_failed", "compact_stall",
        "compact_success", "thp_split_page", "pgmajfault")


def vm():
    d = {}
    for line in open("/proc/vmstat"):
        k, v = line.split()
        if k in KEYS:
            d[k] = int(v)
    return d


def rd(p):
    try:
        return open(p).read().strip()
    except OSError as e:
        return str(e)


out = {"enabled": rd("/sys/kernel/mm/transparent_hugepage/enabled"),
       "defrag": rd("/sys/kernel/mm/transparent_hugepage/defrag"),
       "khugepaged_defrag": rd("/sys/kernel/mm/transparent_hugepage/khugepaged/defrag"),
       "meminfo": [l.strip() for l in open("/proc/meminfo") if l.split(":")[0] in
                   ("MemTotal", "MemFree", "AnonHugePages", "HugePages_Total", "Hugepagesize")]}
v0 = vm()
P, SG = 7_000_000_000, 100_000_000
plan = D.build_plan(70, 5, static_ratio=0.2, placement=D.Placement.STATIC_FIRST)
t0 = time.perf_counter()
opt = D.ShardedOptimizer.allocate(P, SG, lowp="bf16", host_homed=[i for i in range(70) if i not in plan.static_set])
out["alloc_s"] = time.perf_counter() - t0
v1 = vm()
res = opt.to_device(torch.device("cuda", 0))
res.set_static(plan.static_set)
fill_shard(opt, 7, torch.device("cuda", 0))
prof = profile_b200.measure_profile(quick=True)
hyper = D.AdamHyper()
times = []
for _ in range(8):
    t = time.perf_counter()
    D.execute_plan(opt, plan, prof, hyper)
    times.append(round((time.perf_counter() - t) * 1e3, 1))
v2 = vm()
out["phase_ms"] = times
out["vmstat_alloc_delta"] = {k: v1[k] - v0[k] for k in v0}
out["vmstat_run_delta"] = {k: v2[k] - v1[k] for k in v0}
out["anon_huge_after"] = [l.strip() for l in open("/proc/meminfo") if l.startswith("AnonHugePages")]
print(json.dumps(out, indent=1))
