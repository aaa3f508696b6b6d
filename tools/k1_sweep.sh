#!/bin/bash
# K1 pipeline-shape sweep (bf16 grads + bf16 copy); one process per shape.
DOS_K1=ldg python tools/k1_ab.py
for c in 0 1 2 3 4 5 6 7 8; do echo "cfg $c"; DOS_K1_CFG=$c python tools/k1_ab.py; done
