#!/bin/bash
# H1 store variants on the GPU box: the host probe under each, then the 7B phase A/B
mkdir -p gpurun_out
for cfg in "DOS_H1_NT=default" "DOS_H1_NT=all"; do
  env $cfg timeout 300 python tools/h1_bytes_probe.py > gpurun_out/h1_probe_${cfg#DOS_H1_NT=}.json 2>/dev/null
  echo "$cfg $(tr -d '\n ' < gpurun_out/h1_probe_${cfg#DOS_H1_NT=}.json)"
done
: > gpurun_out/h1_nt_ab.jsonl
ARGS="--steps 8 --warmup 3 --static-variants '' --no-copy-streams --no-ref-schedule --no-e2e --cpu-sample 2"
for cfg in "DOS_H1_NT=default" "DOS_H1_NT=all" "DOS_H1_NT=default" "DOS_H1_NT=all"; do
  env $cfg timeout 420 bash -c "python bench.py $ARGS" > gpurun_out/h1_nt_ab.json 2> gpurun_out/h1_nt_ab.err
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/h1_nt_ab.json").read().strip().splitlines()[-1])
r = {"cfg": sys.argv[1], "ms_per_step": d["ms_per_step"], "stride": d["config"]["stride"],
     "measured_span_ms_by_stride": d["config"]["measured_span_ms_by_stride"],
     "lane_busy_ms_per_step": d["iteration"]["lane_busy_ms_per_step"],
     "joint_bound_frac": d["phase_roofline"]["joint_bound"]["frac"]}
open("gpurun_out/h1_nt_ab.jsonl", "a").write(json.dumps(r) + "\n")
print(r["cfg"], round(r["ms_per_step"], 1), r["stride"], {k: round(v, 1) for k, v in r["lane_busy_ms_per_step"].items()})
PY
done
