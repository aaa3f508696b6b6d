#!/bin/bash
# A/B of how the host lane's working copy leaves the host, on the 7B headline
# phase, back to back on one box: the default (H1 NT-stores it into the host
# image, H2D_PARAMS16 ships it), cached stores into the image, and the
# per-thread staging rings served by the shuttle.  -> gpurun_out/ring_ab.jsonl
mkdir -p gpurun_out
: > gpurun_out/ring_ab.jsonl
ARGS="--steps 8 --warmup 3 --static-variants '' --no-copy-streams --no-ref-schedule --no-e2e --cpu-sample 2"
for cfg in "DOS_W_RING=0" "DOS_H1_WSTORE=cached" "DOS_W_RING=1" "DOS_W_RING=0" "DOS_H1_WSTORE=cached" "DOS_SHUTTLE_CTAS=16"; do
  env $cfg timeout 420 bash -c "python bench.py $ARGS" > gpurun_out/ring_ab.json 2> gpurun_out/ring_ab.err
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ring_ab.json").read().strip().splitlines()[-1])
r = {"cfg": sys.argv[1], "ms_per_step": d["ms_per_step"], "stride": d["config"]["stride"],
     "measured_span_ms_by_stride": d["config"]["measured_span_ms_by_stride"],
     "lane_busy_ms_per_step": d["iteration"]["lane_busy_ms_per_step"],
     "joint_bound_frac": d["phase_roofline"]["joint_bound"]["frac"], "k1_frac": d["roofline"]["frac"]}
open("gpurun_out/ring_ab.jsonl", "a").write(json.dumps(r) + "\n")
print(r["cfg"], round(r["ms_per_step"], 1), r["stride"], {k: round(v, 1) for k, v in r["lane_busy_ms_per_step"].items()})
PY
done
