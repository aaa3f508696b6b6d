"""Run K1 a few times on one 1e8-param subgroup (ncu target)."""
import sys
sys.path.insert(0, ".")
from paper_2410_21316_b200 import profile_b200
print(profile_b200.measure_k1(100_000_000, reps=3))
