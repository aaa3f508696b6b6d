"""Measured timelines of the 7B phase with and without the in-phase grad
flush (same plan): where does the flush's extra time go?
  python tools/flush_trace.py [stride]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_21316_b200 as D  # noqa: E402
from bench import fill_shard  # noqa: E402
from paper_2410_21316_b200 import profile_b200  # noqa: E402
from paper_2410_21316_b200.timing import write_trace_csv  # noqa: E402

P, SG = 7_000_000_000, 100_000_000
stride = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dev = torch.device("cuda", 0)
plan = D.build_plan(70, stride, static_ratio=0.2, placement=D.Placement.STATIC_FIRST)
opt = D.ShardedOptimizer.allocate(P, SG, lowp="bf16", host_homed=[i for i in range(70) if i not in plan.static_set])
res = opt.to_device(dev)
res.set_static(plan.static_set)
fill_shard(opt, 7, dev)
prof = profile_b200.measure_profile(quick=True)
hyper = D.AdamHyper()
os.makedirs("gpurun_out/flush", exist_ok=True)
out = {}
for flush in (False, True, False, True):
    D.execute_plan(opt, plan, prof, hyper, flush_grads=flush)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = D.execute_plan(opt, plan, prof, hyper, flush_grads=flush)
    e1.record()
    torch.cuda.synchronize()
    tag = "flush" if flush else "noflush"
    with open(f"gpurun_out/flush/{tag}.csv", "w") as fh:
        write_trace_csv(r.measured, fh)
    cpu = sorted((e.start_ns, e.end_ns) for e in r.measured.events if e.action.lane.value == "cpu_compute"
                 and e.action.kind.value == "cpu_update")
    gaps = [b[0] - a[1] for a, b in zip(cpu, cpu[1:])]
    out.setdefault(tag, []).append({
        "ms": e0.elapsed_time(e1), "span_ms": r.measured.span_ns / 1e6,
        "cpu_first_start_ms": cpu[0][0] / 1e6, "cpu_last_end_ms": cpu[-1][1] / 1e6,
        "cpu_busy_ms": sum(b - a for a, b in cpu) / 1e6, "cpu_gaps_ms": sum(gaps) / 1e6,
        "busy_ms": {k.value: v / 1e6 for k, v in r.measured.lane_busy_ns.items()}})
print(json.dumps(out, indent=1))
