#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_ring.py tests/test_gpu_execute.py -m gpu -x -q > gpurun_out/r2_ring_tests.txt 2>&1
tail -3 gpurun_out/r2_ring_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 bash tools/ring_ab.sh 2>&1 | tail -8
