#!/bin/bash
# Copy-engine concurrency next to H1: 1/2/4 concurrent H2D (and D2H) streams,
# with the host idle and with the full team running H1 — do more copies in
# flight win the DMA a bigger share of the host DRAM?
cd "$(dirname "$0")" && make -s
OUT=../../gpurun_out/h1_streams.jsonl
: > $OUT
for rep in 1 2; do
  for hd in "1 1" "2 2" "4 4" "2 1" "4 1"; do
    set -- $hd
    DMA_H2D=$1 DMA_D2H=$2 ./h1_pf 16 1e8 4 1 idle pwdyn1024 | tee -a $OUT
  done
done
