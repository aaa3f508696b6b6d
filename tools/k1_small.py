"""Small K1 + engine run for compute-sanitizer (memcheck/racecheck/synccheck)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2410_21316_b200 as D
from oracle import optistate_oracle as O
n = 3 * 4096 * 2 + 77  # a few TMA tiles + ragged tail
rng = np.random.default_rng(0)
p, m, g = (rng.normal(0, s, n).astype(np.float32) for s in (0.02, 1e-3, 1.0))
v = (rng.random(n) * 1e-4).astype(np.float32)
gb = O.bf16_from_f32(g)
tp, tm, tv = (torch.from_numpy(x).cuda() for x in (p, m, v))
tg = torch.from_numpy(gb.view(np.int16)).cuda().view(torch.bfloat16)
w = torch.empty(n, dtype=torch.bfloat16, device="cuda")
from paper_2410_21316_b200 import _native as N
sc = N.scalars(1e-3, 0.9, 0.999, 1e-8, *O.bias_corrections(0.9, 0.999, 1))
N.check(N.lib().dos_adam_step_cuda(tp.data_ptr(), tm.data_ptr(), tv.data_ptr(), tg.data_ptr(), N.DOS_BF16,
                                   w.data_ptr(), N.DOS_BF16, n, sc, None))
torch.cuda.synchronize()
O.adam_step(p, m, v, O.f32_from_bf16(gb), 1e-3, 0.9, 0.999, 1e-8, 1)
assert tp.cpu().numpy().tobytes() == p.tobytes()
opt = D.ShardedOptimizer.initialize(60_000, 8_200, seed=1, lowp="bf16")
D.execute_plan(opt, D.build_plan(len(opt.subgroups), 2, 0.2), D.get_profile("h100-node"), D.AdamHyper())
# the bench's mode: in-phase grad flush (and, with DOS_W_RING / DOS_G_RING, the rings), full coherence check
D.execute_plan(opt, D.build_plan(len(opt.subgroups), 3, 0.2), D.get_profile("h100-node"), D.AdamHyper(),
               flush_grads=True, check_coherence="full")
print("ok")
