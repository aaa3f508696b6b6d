#!/bin/bash
# H1 loop variants on the GPU box's host cores, alone and next to duplex DMA
cd "$(dirname "$0")" && make -s
mkdir -p ../../gpurun_out
OUT=../../gpurun_out/h1_pf_box2.jsonl
: > $OUT
for dma in 0 1; do
  for rep in 1 2; do
    ./h1_pf 16 1e8 4 $dma base pw1024 pw2048 dyn262144 dyn1048576 pf1024 | tee -a $OUT
  done
  ./h1_pf 15 1e8 4 $dma base pw1024 dyn262144 | tee -a $OUT
done
