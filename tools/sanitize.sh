#!/bin/bash
# compute-sanitizer over K1 (TMA ring) and one engine phase.
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  compute-sanitizer --tool $tool --print-limit 20 python tools/k1_small.py 2>&1 | tail -6
done
