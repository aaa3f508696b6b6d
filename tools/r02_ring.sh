#!/bin/bash
# the staging ring served by the shuttle: tests (incl. one hardware queue), smoke, A/B on the 7B phase
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_ring.py -m gpu -x -q > gpurun_out/r2_ring_tests.txt 2>&1
echo "ring tests rc=$? $(tail -1 gpurun_out/r2_ring_tests.txt)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1


timeout 2700 bash tools/ring_ab.sh
