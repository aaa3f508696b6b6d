"""K1 with fp32 grads (the reference's adam_step_arrays signature on CUDA
tensors): 28 B/param without a working copy (read p,m,v,g 16 B; write p,m,v
12 B), 30 B/param with a bf16 copy."""
import json, sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2410_21316_b200 import _native as N

n = 100_000_000
p, m, g = (torch.randn(n, device="cuda") * s for s in (0.02, 1e-3, 1.0))
v = torch.rand(n, device="cuda") * 1e-4
w = torch.empty(n, dtype=torch.bfloat16, device="cuda")
sc = N.scalars(1e-3, 0.9, 0.999, 1e-8, np.float32(0.1), np.float32(0.001))
out = {}
for name, lp, code, bpp in (("f32_grads", None, N.DOS_NONE, 28), ("f32_grads+bf16_copy", w.data_ptr(), N.DOS_BF16, 30)):
    run = lambda: N.check(N.lib().dos_adam_step_cuda(p.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(), N.DOS_F32,
                                                     lp, code, n, sc, torch.cuda.current_stream().cuda_stream))
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        e0.record(); run(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1) * 1e-3)
    t = float(np.median(ts))
    out[name] = {"ms": t * 1e3, "GBs": bpp * n / t / 1e9}
print(json.dumps(out))
