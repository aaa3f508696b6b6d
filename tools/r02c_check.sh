#!/bin/bash
# round-2 (session 3) checks: driver-style bench pair on the current code and
# a two-rank gloo dry run of the N>1 path (ranks share the one B200)
mkdir -p gpurun_out
STEPS=20 WARM=5 TAG=r02c timeout 1500 bash tools/bench_pair.sh > /dev/null 2>&1; echo "bench rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --dist-backend gloo --params 8e8 --subgroup 5e7 --steps 2 --warmup 3 --static-variants "" \
  --no-copy-streams --no-e2e --config-scale 0.02 --configs 13B/2,20B/8,70B/8 > gpurun_out/r02c_dry2.out 2> gpurun_out/r02c_dry2.err
echo "dry rc=$?"; tail -3 gpurun_out/r02c_dry2.err
