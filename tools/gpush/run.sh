#!/bin/bash
# gpush modes alone and next to duplex DMA, ring shapes
cd "$(dirname "$0")" && make -s
OUT=../../gpurun_out/gpush.jsonl
: > $OUT
./gpush 16 1e8 20 0 static flush push | tee -a $OUT
./gpush 16 1e8 20 1 static flush push | tee -a $OUT
for cr in "32768 40" "65536 24" "65536 48" "131072 24" "262144 20"; do
  set -- $cr
  GP_C=$1 GP_R=$2 ./gpush 16 1e8 20 1 static push | tee -a $OUT
done
./gpush 16 1e8 20 1 static flush push | tee -a $OUT
