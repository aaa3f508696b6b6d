#!/bin/bash
# the staging ring served by the shuttle: tests (incl. one hardware queue), smoke, A/B on the 7B phase
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ring.py -m gpu -x -q > gpurun_out/r2_ring_tests.txt 2>&1
echo "ring tests rc=$? $(tail -1 gpurun_out/r2_ring_tests.txt)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
ARGS="--steps 8 --warmup 3 --static-variants '' --no-copy-streams --no-ref-schedule --no-e2e --cpu-sample 2"
for cfg in "DOS_W_RING=0" "DOS_W_RING=1" "DOS_W_RING=0" "DOS_W_RING=1" "DOS_W_RING_CHUNK=262144" "DOS_W_RING_CHUNK=16384" "DOS_SHUTTLE_CTAS=4"; do
  env $cfg timeout 420 bash -c "python bench.py $ARGS" > gpurun_out/ring_ab.json 2> gpurun_out/ring_ab.err
  echo "$cfg rc=$?"
  python -c "import json,sys; d=json.loads(open('gpurun_out/ring_ab.json').read().strip().splitlines()[-1]); print('$cfg', round(d['ms_per_step'],1), d['config']['stride'], d['config']['measured_span_ms_by_stride'], {k: round(v,1) for k,v in d['iteration']['lane_busy_ms_per_step'].items()}, round(d['phase_roofline']['joint_bound']['frac'],3), round(d['roofline']['frac'],3))" 2>&1 | tail -1
done
