#!/bin/bash
# round-2 evidence: full GPU suite, smoke, both bench arms (driver style), ncu
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gpu_suite.txt 2>&1
echo "gpu suite rc=$? $(tail -1 gpurun_out/r2_gpu_suite.txt)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; echo "smoke rc=$?"
STEPS=20 WARM=5 TAG=r02final timeout 1500 bash tools/bench_pair.sh > /dev/null 2>&1; echo "bench rc=$?"
timeout 1500 bash tools/profile_gpu.sh > gpurun_out/r2_profile.log 2>&1; echo "ncu rc=$?"
