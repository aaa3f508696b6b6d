"""K1 A/B: python tools/k1_ab.py  (run twice: DOS_K1=ldg and default)."""
import json, os, sys
sys.path.insert(0, ".")
from paper_2410_21316_b200 import profile_b200
res = {"variant": os.environ.get("DOS_K1", "tma")}
for n in (10_000_000, 100_000_000, 400_000_000):
    r = profile_b200.measure_k1(n, reps=10)
    res[str(n)] = {"GBs": round(r["k1_GBs"], 1), "ms": round(r["k1_ms"], 4)}
print(json.dumps(res))
