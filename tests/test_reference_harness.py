"""The drop-in boundary proven inside the reference's own harness.

* CPU: the reference's complete test suite (166 tests,
  `pkg/tests/*.py`) runs on a copy of the unmodified reference with
  INTEGRATION.md §1's `native` backend patched in — every Adam step
  (`kernels.py:136-139`) and every fp16 conversion (`core.py:190-205`) the
  suite performs goes through libdos (`dos_adam_step_host`,
  `dos_downscale_host`, `dos_upscale_host`).
* GPU: the reference's own engine `run_update` (`scheduler.py:402-466`)
  drives `B200Target` with the reference's own plans, and the result is
  bit-identical to the reference's own `sequential_oracle`
  (`executor.py:103-117`) run live on the same shard.

Both use the reference installed by `tools/install_reference.sh` into
`baseline/_ref` (git-ignored, shipped with the gpurun snapshot); they skip
where it was not installed.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
LIB = ROOT / "paper_2410_21316_b200" / "libdos.so"
pytestmark = pytest.mark.skipif(not (REF / "optistate").exists() or not (REF / "tests").exists(),
                                reason="reference not installed (run tools/install_reference.sh)")

# The one reference test that pins the closed set of backend names; a third
# backend fails it by construction (it is the point of the patch).
CLOSED_SET_TEST = "test_kernels.py::test_active_backend_is_known"


def test_reference_suite_on_native_backend(tmp_path):
    sys.path.insert(0, str(ROOT))
    from integration.patch_reference import patch

    from paper_2410_21316_b200 import _native

    _native.lib()  # builds libdos.so if needed
    patch(REF / "optistate", tmp_path)
    calls = tmp_path / "calls.json"
    env = dict(os.environ, OPTISTATE_BACKEND="native", DOS_LIBRARY=str(LIB), DOS_NATIVE_CALLS=str(calls),
               PYTHONPATH=str(tmp_path))
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "dos_native_calls_plugin",
         str(REF / "tests"), "-k", "not " + CLOSED_SET_TEST.split("::")[1]],
        cwd=tmp_path, env=env, capture_output=True, text=True, timeout=900)
    tail = proc.stdout[-3000:] + proc.stderr[-2000:]
    assert proc.returncode == 0, tail
    assert "165 passed" in proc.stdout and "failed" not in proc.stdout.splitlines()[-1], tail
    got = json.loads(calls.read_text())
    assert got["loaded"] and got["backend"] == "native", got
    # the suite's Adam steps and conversions really went through libdos
    assert got["calls"]["adam_step"] > 1000 and got["calls"]["downscale_f16"] > 1000, got
    assert got["calls"]["upscale_f16"] > 1000, got


def test_closed_set_test_fails_only_on_the_backend_name(tmp_path):
    """The deselected test fails with exactly the new name, nothing else."""
    sys.path.insert(0, str(ROOT))
    from integration.patch_reference import patch

    patch(REF / "optistate", tmp_path)
    env = dict(os.environ, OPTISTATE_BACKEND="native", DOS_LIBRARY=str(LIB), PYTHONPATH=str(tmp_path))
    proc = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                           str(REF / "tests" / CLOSED_SET_TEST)], cwd=tmp_path, env=env, capture_output=True,
                          text=True, timeout=300)
    assert proc.returncode == 1 and "assert 'native' in ('numba', 'numpy')" in proc.stdout, proc.stdout[-2000:]


def test_cuda_is_still_rejected(tmp_path):
    """`cuda` stays an invalid backend value (reference tests/test_kernels.py:37-44)."""
    sys.path.insert(0, str(ROOT))
    from integration.patch_reference import patch

    patch(REF / "optistate", tmp_path)
    env = dict(os.environ, OPTISTATE_BACKEND="cuda", PYTHONPATH=str(tmp_path))
    proc = subprocess.run([sys.executable, "-c", "import optistate.kernels"], cwd=tmp_path, env=env,
                          capture_output=True, text=True, timeout=120)
    assert proc.returncode != 0 and "OPTISTATE_BACKEND" in proc.stderr


@pytest.fixture(scope="module")
def R():
    """The unmodified reference, imported from baseline/_ref."""
    sys.path.insert(0, str(REF))
    import optistate

    assert Path(optistate.__file__).resolve().is_relative_to(REF.resolve()), optistate.__file__
    return optistate


@pytest.mark.gpu
@pytest.mark.parametrize("stride", [1, 2, 3, "all_cpu"])
@pytest.mark.parametrize("ratio,placement", [(0.0, "static_last"), (0.25, "static_last"), (0.25, "static_first")])
def test_reference_run_update_drives_b200_target(R, stride, ratio, placement):
    import paper_2410_21316_b200 as D
    from paper_2410_21316_b200.device import B200Target

    total, sg, seed = 10 * 4096 + 777, 4096, 20250816  # 11 subgroups, ragged tail
    ref = R.ShardedOptimizer.initialize(total, sg, seed=seed)
    opt = D.load_shard(ref.params32, ref.momentum32, ref.variance32, ref.grads16, ref.model16, sg, lowp="fp16",
                       static_set=R.build_plan(len(ref.subgroups), 1, ratio,
                                               R.Placement(placement)).static_set)
    k = R.ALL_CPU if stride == "all_cpu" else stride
    rplan = R.build_plan(len(ref.subgroups), k, ratio, R.Placement(placement))  # the reference's planner
    prof = R.get_profile("h100-node")
    target = B200Target(prof, rplan, opt, D.AdamHyper(), step=opt.step + 1)
    try:
        events = R.run_update(rplan, target)  # the reference's engine drives the B200
    finally:
        measured = target.finish()
    target.residency.after_phase(False)
    opt.step += 1
    R.validate_schedule(rplan, events, target)  # the reference's audit of the predicted timeline
    assert len(measured) == len(rplan.actions)
    R.sequential_oracle(ref, R.AdamHyper())  # the reference's ground truth, live
    for name in ("params32", "momentum32", "variance32", "model16", "grads16"):
        assert getattr(opt, name).tobytes() == getattr(ref, name).tobytes(), name
