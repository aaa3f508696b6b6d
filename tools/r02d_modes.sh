#!/bin/bash
# Other bench modes on the final code: fp16, the 125M config (both arms),
# capacity-aware 7B, the ALL_CPU stride, and the eight-rank gloo dry run
mkdir -p gpurun_out
Q="--steps 3 --warmup 3 --cpu-sample 2"
timeout 900 python bench.py $Q --lowp fp16 --static-variants '' > gpurun_out/m_fp16.out 2> gpurun_out/m_fp16.err; echo "fp16 rc=$?"
timeout 600 python bench.py $Q --params 1.25e8 --subgroup 7812500 --cpu-sample 16 > gpurun_out/m_125m.out 2> gpurun_out/m_125m.err; echo "125m rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 --params 1.25e8 --subgroup 7812500 > gpurun_out/m_125m_ref.out 2> gpurun_out/m_125m_ref.err; echo "125m ref rc=$?"
timeout 900 python bench.py $Q --static-ratio auto --static-variants '' --no-copy-streams > gpurun_out/m_auto.out 2> gpurun_out/m_auto.err; echo "auto rc=$?"
timeout 900 python bench.py $Q --stride all_cpu --static-variants '' --no-copy-streams --no-ref-schedule > gpurun_out/m_allcpu.out 2> gpurun_out/m_allcpu.err; echo "allcpu rc=$?"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 8 --dist-backend gloo --params 8e8 --subgroup 2.5e7 --steps 2 --warmup 3 --static-variants "" \
  --no-copy-streams --no-e2e --config-scale 0.01 > gpurun_out/m_dry8.out 2> gpurun_out/m_dry8.err
echo "dry8 rc=$?"
for f in m_fp16 m_125m m_125m_ref m_auto m_allcpu m_dry8; do echo "== $f"; grep -v "^\s*$" gpurun_out/$f.err | grep -iv "warn\|nccl\|OMP_NUM\|\*\*\*" | tail -3; done
