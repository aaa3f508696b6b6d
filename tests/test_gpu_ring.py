"""The host lane's working-copy staging ring (dos_host_adam_ring + the
shuttle kernel; opt-in, DOS_W_RING=1 — slower than the default on the
measured host, kept as an A/B arm): host-updated subgroups' working copy goes H2D in
chunks from every team thread's own L2/LLC-resident slots during the CPU
update, instead of through the host image.
Bit-exact against the oracle with many chunks per subgroup, ragged chunks,
two-slot wrap-around across subgroups, every plan shape, and with the ring
off (the A/B baseline).  The ring configuration is read once per process, so
each configuration runs in its own interpreter."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

CHECK = r"""
import sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2410_21316_b200 as D
from oracle import optistate_oracle as O
from paper_2410_21316_b200 import ALL_CPU, Placement
prof = D.get_profile("h100-node")
for total, sg in ((10 * 7000 + 333, 7000), (3 * 50_000, 50_000)):
    nsg = -(-total // sg)
    for stride in (1, 2, 3, ALL_CPU):
        for ratio, pl in ((0.0, Placement.STATIC_LAST), (0.25, Placement.STATIC_FIRST)):
            for flush in (False, True):
                opt = D.ShardedOptimizer.initialize(total, sg, seed=nsg + stride if stride is not ALL_CPU else 99,
                                                    lowp="bf16")
                want = O.initialize(total, sg, nsg + stride if stride is not ALL_CPU else 99, "bf16")
                plan = D.build_plan(nsg, stride, static_ratio=ratio, placement=pl)
                for step in range(2):
                    D.execute_plan(opt, plan, prof, D.AdamHyper(), flush_grads=flush, check_coherence="full")
                    O.sequential_oracle(want)
                got_w = opt.residency.model16.view(torch.int16).cpu().numpy().view(np.uint16)
                assert opt.params32.tobytes() == want["p"].tobytes(), (total, stride, ratio, flush)
                assert opt.variance32.tobytes() == want["v"].tobytes(), (total, stride, ratio, flush)
                assert got_w.tobytes() == want["w"].tobytes(), (total, stride, ratio, flush)
print("ring ok")
"""


@pytest.mark.parametrize("env", [
    {"DOS_W_RING": "1"},  # ring on (off by default): 4 x 64K per thread, 16 shuttle CTAs
    {"DOS_W_RING": "1", "DOS_W_RING_CHUNK": "4096", "DOS_W_RING_SLOTS": "2"},  # many ragged chunks, tight reuse
    {"DOS_W_RING": "1", "DOS_W_RING_CHUNK": "1024", "DOS_W_RING_SLOTS": "1", "DOS_SHUTTLE_CTAS": "1"},
    {"DOS_W_RING": "1", "DOS_W_RING_CHUNK": "12288", "DOS_W_RING_SLOTS": "3", "DOS_SHUTTLE_CTAS": "3"},
    # every stream on ONE hardware queue: a wait at the head of any stream blocks
    # all the others queued behind it.  The engine must still finish: every
    # GPU-side wait is on a host action emitted earlier, and the ring's copies
    # are served by a kernel launched before anything else of the phase
    {"CUDA_DEVICE_MAX_CONNECTIONS": "1", "DOS_W_RING": "1", "DOS_W_RING_CHUNK": "12288", "DOS_W_RING_SLOTS": "3"},
    {"CUDA_DEVICE_MAX_CONNECTIONS": "1"},  # the default path (ring off) on one hardware queue
    {"DOS_H1_WSTORE": "cached"},  # H1's cached-store variant (A/B knob)
    {"DOS_H1_NT": "all"},  # H1 streaming-stores p, m, v too (A/B knob)
    # the in-phase grad flush's ring (opt-in A/B arm): default rows, tiny rows
    # with one slot, and on one hardware queue
    {"DOS_G_RING": "1"},
    {"DOS_G_RING": "1", "DOS_G_RING_CHUNK": "1024", "DOS_G_RING_SLOTS": "1"},
    {"DOS_G_RING": "1", "DOS_G_RING_CHUNK": "4096", "DOS_G_RING_SLOTS": "2", "CUDA_DEVICE_MAX_CONNECTIONS": "1"},
    {},  # default: H1 -> host image (NT stores) -> H2D_PARAMS16
])
def test_ring_bit_exact(env):
    proc = subprocess.run([sys.executable, "-c", CHECK], cwd=ROOT, env=dict(os.environ, **env), capture_output=True,
                          text=True, timeout=600)
    assert proc.returncode == 0 and "ring ok" in proc.stdout, proc.stdout[-2000:] + proc.stderr[-3000:]
