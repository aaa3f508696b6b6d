#!/bin/bash
# longer windows, modes alternated: flush vs push next to duplex DMA
cd "$(dirname "$0")" && make -s
OUT=../../gpurun_out/gpush2.jsonl
: > $OUT
for rep in 1 2 3; do
  ./gpush 16 1e8 60 1 flush push | tee -a $OUT
  GP_C=131072 GP_R=24 ./gpush 16 1e8 60 1 push | tee -a $OUT
  GP_C=65536 GP_R=24 GP_CTAS=4 ./gpush 16 1e8 60 1 push | tee -a $OUT
done
