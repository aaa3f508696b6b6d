#!/bin/bash
# BASELINE configs[2-4] on the final code: one-rank slices (13B/2, 20B/4,
# 20B/8, 70B/8 with its stride sweep) and 13B on one B200 (capacity-aware)
mkdir -p gpurun_out
timeout 2400 python bench.py --steps 3 --warmup 3 --static-variants '' --no-copy-streams --no-ref-schedule --no-e2e \
  --cpu-sample 2 --configs 20B/8,20B/4,13B/2,70B/8 > gpurun_out/r02d_configs.out 2> gpurun_out/r02d_configs.err
echo "configs rc=$?"; tail -2 gpurun_out/r02d_configs.err
timeout 1800 python bench.py --params 13e9 --static-ratio auto --static-variants 0.5 --steps 5 --warmup 3 \
  --no-copy-streams --cpu-sample 2 > gpurun_out/r02d_13b.out 2> gpurun_out/r02d_13b.err
echo "13b rc=$?"; tail -2 gpurun_out/r02d_13b.err
