#!/bin/bash
# confirmation on the final code: full GPU suite, smoke, both bench arms (driver style)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02e_gpu_suite.txt 2>&1
echo "gpu suite rc=$? $(tail -1 gpurun_out/r02e_gpu_suite.txt)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02e_smoke.txt 2>&1; echo "smoke rc=$?"
STEPS=20 WARM=5 TAG=r02e timeout 1500 bash tools/bench_pair.sh > /dev/null 2>&1; echo "bench rc=$?"
