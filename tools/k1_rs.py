"""K1 with the reduce-scatter fused in (pipeline shape / peer-prefetch depth
from DOS_K1_RS, see tools/k1_rs_sweep.sh) (dos_adam_step_cuda_rs) vs plain K1,
and the stand-alone reduce kernel, on one B200.  The "ranks" are separate
local HBM buffers, so this measures the kernel's HBM efficiency with the
extra grad streams (on a real node the peers' reads go over NVLink instead).
Algorithmic bytes per param: K1 28; K1+RS 28 + 2*(world-1) (other ranks'
grads) + 2 (reduced grads written back); reduce 2*world + 2."""
import json
import os
import sys

sys.path.insert(0, ".")
import ctypes as C

import numpy as np
import torch

from paper_2410_21316_b200 import _native as N

n = 100_000_000
p, m = (torch.randn(n, device="cuda") * s for s in (0.02, 1e-3))
v = torch.rand(n, device="cuda") * 1e-4
w = torch.empty(n, dtype=torch.bfloat16, device="cuda")
gs = [torch.randn(n, device="cuda").to(torch.bfloat16) for _ in range(8)]
sc = N.scalars(1e-3, 0.9, 0.999, 1e-8, np.float32(0.1), np.float32(0.001))
lib = N.lib()


def timed(run, reps=10):
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        run()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


out = {"DOS_K1_RS": os.environ.get("DOS_K1_RS", "0,1 (default: 1024 x 3 ring, peers 1 tile ahead)")}
st = lambda: torch.cuda.current_stream().cuda_stream
t = timed(lambda: N.check(lib.dos_adam_step_cuda(p.data_ptr(), m.data_ptr(), v.data_ptr(), gs[0].data_ptr(),
                                                 N.DOS_BF16, w.data_ptr(), N.DOS_BF16, n, sc, st())))
out["k1"] = {"ms": t * 1e3, "GBs": 28 * n / t / 1e9}
for world in (1, 2, 4, 8):
    srcs = (C.c_void_p * world)(*[g.data_ptr() for g in gs[:world]])
    t = timed(lambda: N.check(lib.dos_adam_step_cuda_rs(p.data_ptr(), m.data_ptr(), v.data_ptr(), srcs, world, 0,
                                                        N.DOS_BF16, 1.0, w.data_ptr(), N.DOS_BF16, None, 0, n, sc,
                                                        st())))
    bpp = 28 + 2 * (world - 1) + 2
    out[f"k1_rs_world{world}"] = {"ms": t * 1e3, "GBs": bpp * n / t / 1e9, "bytes_per_param": bpp}
    t = timed(lambda: N.check(lib.dos_reduce_scatter_cuda(gs[0].data_ptr(), srcs, world, N.DOS_BF16, 1.0, n, st())))
    bpp = 2 * world + 2
    out[f"reduce_world{world}"] = {"ms": t * 1e3, "GBs": bpp * n / t / 1e9, "bytes_per_param": bpp}
print(json.dumps(out, indent=1))
