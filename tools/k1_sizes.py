"""K1 vs a device copy of the same bytes over subgroup sizes (1M..100M
params): how much of the fixed per-launch cost (launch, pipeline fill, tail)
is K1's own?  Back-to-back launches on one stream, CUDA events, median."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2410_21316_b200 import _native as N

lib = N.lib()
sc = N.scalars(1e-3, 0.9, 0.999, 1e-8, np.float32(0.1), np.float32(0.001))
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
NMAX = 100_000_000
p = torch.randn(NMAX, device="cuda") * 0.02
m = torch.randn(NMAX, device="cuda") * 1e-3
v = torch.rand(NMAX, device="cuda") * 1e-4
g = torch.randn(NMAX, device="cuda").to(torch.bfloat16)
w = torch.empty(NMAX, dtype=torch.bfloat16, device="cuda")
src = torch.empty(28 * NMAX // 2, dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)


def timed(fn, reps=30, inner=10):
    fn()
    ts = []
    for _ in range(reps):
        e0.record(st)
        for _ in range(inner):
            fn()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / inner * 1e-3)
    return float(np.median(ts))


for n in (1_000_000, 2_000_000, 4_000_000, 7_812_500, 10_000_000, 25_000_000, 50_000_000, 100_000_000):
    k1 = lambda: N.check(lib.dos_adam_step_cuda(p.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(), N.DOS_BF16,
                                                w.data_ptr(), N.DOS_BF16, n, sc, st.cuda_stream))
    nb = 14 * n  # a copy moving 28 B/param: 14 read + 14 written
    cp = lambda: dst[:nb].copy_(src[:nb])
    tk, tc = timed(k1), timed(cp)
    print(json.dumps({"n": n, "k1_us": tk * 1e6, "k1_GBs": 28 * n / tk / 1e9, "copy_us": tc * 1e6,
                      "copy_GBs": 28 * n / tc / 1e9, "k1_over_copy": tc / tk}), flush=True)
