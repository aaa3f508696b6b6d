#!/bin/bash
# H2D by copy engine vs by SM pull (and D2H by SM push), alone and next to H1
cd "$(dirname "$0")" && make -s
OUT=../../gpurun_out/h1_pull.jsonl
: > $OUT
for rep in 1 2; do
  for cfg in "-" "DMA_PULL=16" "DMA_PULL=64" "DMA_PULL=148" "DMA_PUSH=16" "DMA_PULL=64 DMA_PUSH=16"; do
    envs=""; [ "$cfg" != "-" ] && envs="$cfg"
    env $envs ./h1_pf 16 1e8 4 1 idle pwdyn1024 | sed "s/^{/{\"cfg\": \"$cfg\", /" | tee -a $OUT
  done
done
