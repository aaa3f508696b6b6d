#!/bin/bash
# 13B on one B200, capacity-aware residency (BASELINE configs[2] at N=1)
mkdir -p gpurun_out
timeout 1800 python bench.py --params 13e9 --static-ratio auto --static-variants 0.5 --steps 5 --warmup 3 \
  --no-copy-streams --cpu-sample 2 > gpurun_out/r02d_13b.out 2> gpurun_out/r02d_13b.err
echo "13b rc=$?"; tail -2 gpurun_out/r02d_13b.err
