#!/bin/bash
mkdir -p gpurun_out
timeout 1500 bash tools/sanitize.sh > gpurun_out/r2_sanitize.txt 2>&1; echo "sanitize rc=$?"
grep -E "==|ERROR SUMMARY|ok" gpurun_out/r2_sanitize.txt | head -20
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29555 \
  bench.py --gpus 8 --dist-backend gloo --params 8e8 --subgroup 2.5e7 --steps 2 --warmup 3 --static-variants '' \
  --no-copy-streams --no-e2e --config-scale 0.01 > gpurun_out/r2_gloo8.out 2> gpurun_out/r2_gloo8.err
echo "gloo8 rc=$?"; tail -2 gpurun_out/r2_gloo8.err
