"""bench.py keeps the driver's JSON-line contract: the reference arm on the
host cores (CPU), and a small B200 arm run (GPU)."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "cpu_baseline"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout[-2000:]  # exactly one JSON line
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--params", "2e8", "--steps", "1", "--warmup", "3"], 600)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "params/s" and d["higher_is_better"] is True
    assert d["e2e"] == {"value": d["value"], "unit": "params/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]


@pytest.mark.gpu
def test_b200_arm_contract():
    d = _run(["--params", "6e8", "--steps", "3", "--warmup", "3", "--cpu-sample", "2", "--static-variants", "0.0",
              "--no-ref-schedule"], 900)
    assert BASE_KEYS | {"roofline", "clocks"} <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    # every K1 launch plus one post-phase coherence launch per timed step
    assert d["gpu_launches"] > 0 and d["gpu_launches"] == d["k1_updates"] + d["steps"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["phase_roofline"]["frac"] > 0 and d["copy_streams"]["frac"] > 0


def test_joint_bound_is_a_lower_bound_for_every_split():
    """phase_roofline.joint_bound: min over the streamed fraction of the
    slowest resource — never above the bound of any concrete split, and the
    binding resources balance at the optimum."""
    import sys

    sys.path.insert(0, str(ROOT))
    import bench

    D, S = 5.6e9, 1.4e9
    hbm, link, dram, h1 = 6.5e12, 48e9, 180e9, 5e9
    for flush in (False, True):
        jb = bench.joint_bound(D, S, hbm, link, dram, h1, flush)
        gB = 2.0 if flush else 0.0
        for x in (0.0, 0.1, 0.25, 0.5, 0.75, 1.0):
            t = max(28 * (S + x * D) / hbm, max((12 * x + 2 * (1 - x)) * D, (12 * x + gB * (1 - x)) * D) / link,
                    (24 * x + (30 + gB) * (1 - x)) * D / dram, (1 - x) * D / h1)
            assert jb["ideal_ms"] <= t * 1e3 + 1e-6
        at = jb["bounds_ms_at_optimum"]
        assert abs(at["link"] - at["host_dram"]) / jb["ideal_ms"] < 0.01  # link and DRAM balance here
