#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_ring.py tests/test_gpu_execute.py tests/test_gpu_optim.py tests/test_gpu_optim_dist.py tests/test_bench_contract.py -m gpu -x -q > gpurun_out/r2_gring_tests.txt 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/r2_gring_tests.txt)"
timeout 2700 bash tools/gring_ab.sh
