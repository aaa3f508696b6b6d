#!/bin/bash
# K1 with the fused reduce-scatter at 1/2/4/8 grad sources, for every
# selectable pipeline shape x peer-prefetch depth (one process each: the
# choice is read once per process) -> gpurun_out/k1_rs_<shape>_<depth>.json
mkdir -p gpurun_out
for cfg in 0,1 0,2 1,1 1,2; do
  DOS_K1_RS=$cfg python tools/k1_rs.py > gpurun_out/k1_rs_${cfg/,/_}.json
done
python - <<'PY'
import json, glob
out = {}
for f in sorted(glob.glob("gpurun_out/k1_rs_[01]_[12].json")):
    d = json.load(open(f))
    out[d["DOS_K1_RS"]] = {k: round(v["GBs"], 1) for k, v in d.items() if isinstance(v, dict)}
json.dump(out, open("gpurun_out/k1_rs_sweep.json", "w"), indent=1)
print(json.dumps(out, indent=1))
PY
