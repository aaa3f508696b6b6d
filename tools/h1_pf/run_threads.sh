#!/bin/bash
# H1 (shipped variant: prefetchw 1 KB + 256K dynamic chunks) next to duplex DMA
# at 2..16 threads: how the DRAM splits between the host team and the copy engines
cd "$(dirname "$0")" && make -s
OUT=../../gpurun_out/h1_threads_dma.jsonl
: > $OUT
for rep in 1 2; do
  for t in 2 4 6 8 10 12 14 16; do
    ./h1_pf $t 1e8 4 1 pwdyn1024 | tee -a $OUT
  done
done
./h1_pf 16 1e8 4 0 pwdyn1024 | tee -a $OUT
