mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2b_gpu_suite.txt 2>&1
echo "gpu suite rc=$? $(tail -1 gpurun_out/r2b_gpu_suite.txt)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --gpus 1 --steps 10 --warmup 3 > gpurun_out/r2b_b200.out 2> gpurun_out/r2b_b200.err; echo "bench rc=$?"
