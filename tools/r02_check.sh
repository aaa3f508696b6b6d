#!/bin/bash
# round-2 checks: changed GPU tests, the fused-RS shape/depth sweep, and a
# two-rank gloo dry run of bench.py's per-config path on the one B200
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_execute.py tests/test_gpu_reduce_scatter.py tests/test_multigpu.py tests/test_gpu_optim_dist.py -m gpu -x -q > gpurun_out/r2_t3.txt 2>&1
tail -5 gpurun_out/r2_t3.txt
timeout 600 bash tools/k1_rs_sweep.sh > gpurun_out/r2_rs_sweep.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --dist-backend gloo --params 8e8 --subgroup 5e7 --steps 2 --warmup 3 --static-variants "" \
  --no-copy-streams --no-e2e --config-scale 0.02 --configs 13B/2,20B/8,70B/8 > gpurun_out/r2_dry2.out 2> gpurun_out/r2_dry2.err
echo "dry rc=$?"; tail -3 gpurun_out/r2_dry2.err
