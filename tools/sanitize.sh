#!/bin/bash
# compute-sanitizer over K1 (TMA ring), engine phases (incl. the in-phase grad
# flush and the coherence kernel) and, with the rings on, the shuttle kernel.
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  compute-sanitizer --tool $tool --print-limit 20 python tools/k1_small.py 2>&1 | tail -6
done
for ring in DOS_W_RING=1 DOS_G_RING=1; do
  echo "== memcheck $ring"
  env $ring compute-sanitizer --tool memcheck --print-limit 20 python tools/k1_small.py 2>&1 | tail -4
done
