"""The start-up probes must not keep HBM: bench.py takes the capacity-aware
budget after the link probe, and a probe that held its device buffers cost
residents (13B/1: two subgroups) or, on a tighter box, the engine's windows."""
from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_link_probe_releases_its_device_buffers():
    from paper_2410_21316_b200 import profile_b200

    torch.cuda.empty_cache()
    before = torch.cuda.memory_reserved()
    r = profile_b200.measure_link(1 << 28, reps=1)
    assert r["h2d_GBs"] > 0 and r["d2h_GBs"] > 0 and r["duplex_GBs_per_dir"] > 0
    assert torch.cuda.memory_reserved() <= before
    profile_b200.measure_link(1 << 28, reps=1)  # the pinned host pair is reused, the device pair made again
    assert torch.cuda.memory_reserved() <= before


def test_k1_probe_next_to_dma_reports_the_copy_ceiling():
    from paper_2410_21316_b200 import profile_b200

    r = profile_b200.measure_k1(10_000_000, reps=3, with_dma=True)
    d = r["under_duplex_dma"]
    assert r["d2d_copy_GBs"] > 0 and d["k1_GBs"] > 0 and d["d2d_copy_GBs"] > 0 and d["dma_GBs"] > 0
