#!/bin/bash
# deadlock hypothesis (stream/channel sharing) + the ring's A/B with 32 hardware connections
mkdir -p gpurun_out
for e in "CUDA_DEVICE_MAX_CONNECTIONS=1" "CUDA_DEVICE_MAX_CONNECTIONS=32 DOS_W_RING_CHUNK=12288 DOS_W_RING_SLOTS=3"; do
  env $e timeout 120 python -m pytest tests/test_gpu_ring.py -m gpu -x -q -k "env0 or env2" > gpurun_out/r2_ring_hyp.txt 2>&1
  echo "$e rc=$? $(tail -1 gpurun_out/r2_ring_hyp.txt)"
done
ARGS="--steps 8 --warmup 3 --static-variants '' --no-copy-streams --no-ref-schedule --no-e2e --cpu-sample 2"
for cfg in "DOS_W_RING=0" "DOS_W_RING=1" "DOS_W_RING=0" "DOS_W_RING=1"; do
  CUDA_DEVICE_MAX_CONNECTIONS=32 env $cfg timeout 400 bash -c "python bench.py $ARGS" > gpurun_out/ring_ab.json 2> gpurun_out/ring_ab.err
  echo "$cfg rc=$?"
  python -c "import json,sys; d=json.loads(open('gpurun_out/ring_ab.json').read().strip().splitlines()[-1]); print('$cfg', round(d['ms_per_step'],1), d['config']['stride'], d['config']['measured_span_ms_by_stride'], {k: round(v,1) for k,v in d['iteration']['lane_busy_ms_per_step'].items()}, round(d['phase_roofline']['joint_bound']['frac'],3))" 2>&1 | tail -1
done
