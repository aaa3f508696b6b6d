#!/bin/bash
# GPU suite + one-rank slices of BASELINE configs[2-4] at N=1 (bench --configs)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_gpu_suite2.txt 2>&1
echo "gpu suite rc=$? $(tail -1 gpurun_out/r2_gpu_suite2.txt)"
timeout 2400 python bench.py --steps 3 --warmup 3 --static-variants '' --no-copy-streams --no-ref-schedule --no-e2e \
  --cpu-sample 2 --configs 20B/8,20B/4,13B/2,70B/8 > gpurun_out/r2_configs.out 2> gpurun_out/r2_configs.err
echo "configs rc=$?"; tail -2 gpurun_out/r2_configs.err
