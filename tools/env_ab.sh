#!/bin/bash
# A/B of environment knobs on the 7B headline phase, back to back on one box.
#   bash tools/env_ab.sh <tag> "<cfg A>" "<cfg B>" ...   (each cfg: space-separated VAR=value, or "-" for none)
# -> gpurun_out/<tag>.jsonl (one line per run: ms/step, stride, lane busy, joint-bound fraction)
mkdir -p gpurun_out
TAG=$1; shift
: > gpurun_out/$TAG.jsonl
ARGS="--steps 8 --warmup 3 --static-variants '' --no-copy-streams --no-ref-schedule --no-e2e --cpu-sample 2 ${AB_ARGS:-}"
for cfg in "$@"; do
  envs=""; [ "$cfg" != "-" ] && envs="$cfg"
  env $envs timeout 480 bash -c "python bench.py $ARGS" > gpurun_out/$TAG.json 2> gpurun_out/$TAG.err
  python - "$cfg" "$TAG" <<'PY'
import json, sys
cfg, tag = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/{tag}.json").read().strip().splitlines()[-1])
except Exception as e:  # keep going: one failed arm must not lose the others
    print(cfg, "FAILED", e); sys.exit(0)
r = {"cfg": cfg, "ms_per_step": d["ms_per_step"], "stride": d["config"]["stride"],
     "measured_span_ms_by_stride": d["config"]["measured_span_ms_by_stride"],
     "lane_busy_ms_per_step": d["iteration"]["lane_busy_ms_per_step"],
     "joint_bound_frac": d["phase_roofline"]["joint_bound"]["frac"], "k1_frac": d["roofline"]["frac"]}
open(f"gpurun_out/{tag}.jsonl", "a").write(json.dumps(r) + "\n")
print(r["cfg"], round(r["ms_per_step"], 1), r["stride"], {k: round(v, 1) for k, v in r["lane_busy_ms_per_step"].items()})
PY
done
