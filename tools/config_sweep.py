"""Measured update phase of one rank's shard over (static ratio, stride):
the BASELINE configs as one rank sees them on one B200, e.g. rank 0 of
70B/8 (8.75e9 params, 88 subgroups, ragged 5e7 tail) or of 20B/8 (2.5e9).

  python tools/config_sweep.py --params 8.75e9 --ratios 0,auto --strides 1,2,3,4,5,6,all_cpu

Each cell: one untimed step, then --steps steps timed with CUDA events.
Ratios whose host-homed state would not fit in host memory are skipped.
Writes gpurun_out/config_sweep_<params>.json."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_21316_b200 as D  # noqa: E402
from bench import fill_shard, host_available_bytes  # noqa: E402
from paper_2410_21316_b200 import policy, profile_b200  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--params", type=float, default=8.75e9)
ap.add_argument("--subgroup", type=float, default=1e8)
ap.add_argument("--ratios", default="0,auto")
ap.add_argument("--strides", default="1,2,3,4,5,6,all_cpu")
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
P, SG = int(a.params), int(a.subgroup)
dev = torch.device("cuda", 0)
sizes = [g.size for g in D.shard(P, 1, SG)[0]]
n = len(sizes)
ratios = []
for tok in a.ratios.split(","):
    ratios.append(policy.capacity_static_ratio(sizes, torch.cuda.mem_get_info(dev)[0]) if tok == "auto" else float(tok))
strides = [D.ALL_CPU if t == "all_cpu" else int(t) for t in a.strides.split(",")]
first_static = D.build_plan(n, 1, static_ratio=max(ratios)).static_set
t0 = time.perf_counter()
opt = D.ShardedOptimizer.allocate(P, SG, lowp="bf16", host_homed=[i for i in range(n) if i not in first_static])
res = opt.to_device(dev)
res.set_static(first_static)
fill_shard(opt, 7, dev)
setup_s = time.perf_counter() - t0
prof = profile_b200.measure_profile(quick=True)
hyper = D.AdamHyper()
rows = []
for ratio in sorted(ratios, reverse=True):
    static = D.build_plan(n, 1, static_ratio=ratio).static_set
    need = 16 * sum(s for i, s in enumerate(sizes) if i not in static)
    if need > opt.host_bytes + host_available_bytes() - (8 << 30):
        rows.append({"static_ratio": ratio, "skipped": "host-homed state would not fit in host memory"})
        print(json.dumps(rows[-1]), flush=True)
        continue
    for stride in strides:
        if stride is D.ALL_CPU and static:
            continue  # the reference's offload schedule has no residents
        plan = D.build_plan(n, stride, static_ratio=ratio)
        D.execute_plan(opt, plan, prof, hyper)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rr = [D.execute_plan(opt, plan, prof, hyper) for _ in range(a.steps)]
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        fast = sum(sizes[i] for i, d in enumerate(plan.devices) if d is D.Device.FAST)
        rows.append({"static_ratio": round(ratio, 4), "static_subgroups": len(static),
                     "stride": "all_cpu" if stride is D.ALL_CPU else stride,
                     "gpu_fraction": fast / P, "ms": ms, "params_per_s": P / (ms * 1e-3),
                     "span_ms": rr[-1].measured.span_ns / 1e6,
                     "busy_ms": {k.value: v / 1e6 for k, v in rr[-1].measured.lane_busy_ns.items()}})
        print(json.dumps(rows[-1]), flush=True)
out = {"params": P, "subgroup": SG, "subgroups": n, "setup_s": setup_s, "host_threads": D._native.lib().dos_host_threads(),
       "cells": rows}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/config_sweep_{P / 1e9:g}B.json", "w"), indent=1)
