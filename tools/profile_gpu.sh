#!/bin/bash
# ncu evidence for the bench: launch list of the default bench command's timed
# region (NVTX range "timed") + one full capture of K1.  Run under gpurun; outputs land in
# gpurun_out/.  Never used for timing: numbers printed under ncu are not bench values.
set -x
mkdir -p gpurun_out
ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --static-variants '' --no-copy-streams --no-ref-schedule --no-e2e \
    > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_adam_tma -s 3 -c 1 -f -o gpurun_out/k1_full \
    python tools/k1_once.py > gpurun_out/k1_full.log 2>&1
ncu -i gpurun_out/k1_full.ncu-rep --page raw --csv > gpurun_out/k1_full_raw.csv 2>/dev/null
ncu -i gpurun_out/k1_full.ncu-rep --page source --csv > gpurun_out/k1_full_source.csv 2>/dev/null
