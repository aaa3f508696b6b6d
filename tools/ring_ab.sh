#!/bin/bash
# A/B of the working-copy staging ring on the 7B headline phase (same box,
# back to back): DOS_W_RING=0 (H1 -> host image -> H2D_PARAMS16) vs the ring
# at two chunk sizes.  -> gpurun_out/ring_ab_*.json
mkdir -p gpurun_out
ARGS="--steps 10 --warmup 3 --static-variants '' --no-copy-streams --no-ref-schedule --no-e2e --cpu-sample 2"
for cfg in "DOS_W_RING=0" "DOS_W_RING=1" "DOS_W_RING_CHUNK=131072" "DOS_W_RING_CHUNK=2097152" "DOS_W_RING=0"; do
  tag=$(echo $cfg | tr '=' '_')
  env $cfg bash -c "python bench.py $ARGS" > gpurun_out/ring_ab_$tag.json 2> gpurun_out/ring_ab_$tag.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/ring_ab_$tag.json').read().strip().splitlines()[-1]); print('$cfg', round(d['ms_per_step'],1), d['config']['stride'], {k: round(v,1) for k,v in d['iteration']['lane_busy_ms_per_step'].items()}, round(d['phase_roofline']['joint_bound']['frac'],3))"
done
