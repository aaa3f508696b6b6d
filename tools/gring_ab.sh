#!/bin/bash
# A/B of the in-phase grad flush path on the 7B headline phase (back to back):
# whole-subgroup D2H into the host image (DOS_G_RING=0) vs the grad ring.
mkdir -p gpurun_out
: > gpurun_out/gring_ab.jsonl
ARGS="--steps 8 --warmup 3 --static-variants '' --no-copy-streams --no-ref-schedule --no-e2e --cpu-sample 2"
for cfg in "DOS_G_RING=0" "DOS_G_RING=1" "DOS_G_RING=0" "DOS_G_RING=1" "DOS_G_RING_SLOTS=2" "DOS_G_RING_CHUNK=16384"; do
  env $cfg timeout 420 bash -c "python bench.py $ARGS" > gpurun_out/gring_ab.json 2> gpurun_out/gring_ab.err
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/gring_ab.json").read().strip().splitlines()[-1])
r = {"cfg": sys.argv[1], "ms_per_step": d["ms_per_step"], "stride": d["config"]["stride"],
     "measured_span_ms_by_stride": d["config"]["measured_span_ms_by_stride"],
     "lane_busy_ms_per_step": d["iteration"]["lane_busy_ms_per_step"],
     "phase_on_prestaged_grads_ms": d["iteration"]["phase_on_prestaged_grads_ms"],
     "joint_bound_frac": d["phase_roofline"]["joint_bound"]["frac"], "k1_frac": d["roofline"]["frac"]}
open("gpurun_out/gring_ab.jsonl", "a").write(json.dumps(r) + "\n")
print(r["cfg"], round(r["ms_per_step"], 1), "prestaged", round(r["phase_on_prestaged_grads_ms"], 1), r["stride"],
      {k: round(v, 1) for k, v in r["lane_busy_ms_per_step"].items()})
PY
done
