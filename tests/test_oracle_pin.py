"""Pin the oracle (test infrastructure) to the reference's own outputs.

Goldens come from running /root/reference's optistate in the build container
(tests/golden/make_goldens.py).  If these pass, the oracle restates the
reference; every product test then checks against the oracle.
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import c_oracle
from oracle import optistate_oracle as O

G = Path(__file__).resolve().parent / "golden"
META = json.loads((G / "kernel_meta.json").read_text())
VEC = np.load(G / "adam_vectors.npz")
STATES = json.loads((G / "states.json").read_text())


@pytest.mark.parametrize("ci", range(len(META["cases"])))
def test_numpy_oracle_matches_reference_adam(ci):
    c = META["cases"][ci]
    p, m, v = (VEC[f"c{ci}_in_{k}"].copy() for k in "pmv")
    O.adam_step(p, m, v, VEC[f"c{ci}_g"], c["lr"], c["beta1"], c["beta2"], c["eps"], c["step"])
    for k, arr in zip("pmv", (p, m, v)):
        assert arr.tobytes() == VEC[f"c{ci}_out_{k}"].tobytes(), k


@pytest.mark.parametrize("ci", range(len(META["cases"])))
@pytest.mark.parametrize("threads", [1, 3])
def test_c_oracle_matches_reference_adam(ci, threads):
    c = META["cases"][ci]
    p, m, v = (VEC[f"c{ci}_in_{k}"].copy() for k in "pmv")
    c_oracle.adam_mt(p, m, v, VEC[f"c{ci}_g"].copy(), "fp32", None, None, c["lr"], c["beta1"], c["beta2"], c["eps"],
                     c["step"], nthreads=threads)
    for k, arr in zip("pmv", (p, m, v)):
        assert arr.tobytes() == VEC[f"c{ci}_out_{k}"].tobytes(), k


def test_fp16_oracles_match_reference_bits():
    d = np.load(G / "fp16_vectors.npz")
    got = O.f16_from_f32(d["f32_bits"].view(np.float32)).view(np.uint16)
    assert np.array_equal(got, d["f16_bits"])


def test_c_oracle_fp16_working_copy_matches_reference():
    # the C oracle's working-copy rounding through one Adam pass equals numpy's
    st = O.initialize(40_000, 4000, seed=3)
    p, m, v = st["p"].copy(), st["m"].copy(), st["v"].copy()
    w = np.empty(p.size, dtype=np.uint16)
    c_oracle.adam_mt(p, m, v, st["g"].view(np.uint16).copy(), "fp16", w, "fp16", 1e-3, 0.9, 0.999, 1e-8, 1, nthreads=2)
    ref = O.sequential_oracle(st)
    assert p.tobytes() == ref["p"].tobytes()
    assert w.tobytes() == ref["w"].view(np.uint16).tobytes()


def test_bf16_oracle_matches_torch_rne():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.normal(0, 1, 100_000).astype(np.float32),
                        rng.integers(0, 2**32, 100_000, dtype=np.uint32).view(np.float32)])
    x = x[~np.isnan(x)]  # NaN canonicalisation is a declared rule, checked below
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(O.bf16_from_f32(x), want)
    assert O.bf16_from_f32(np.array([np.nan], np.float32))[0] == 0x7FC0


@pytest.mark.parametrize("key", sorted(STATES["oracle"]))
def test_sequential_oracle_digests(key):
    total, sg, seed, which = key.split("|")
    st = O.initialize(int(total), int(sg), int(seed))
    for _ in range(0 if which == "init" else int(which)):
        O.sequential_oracle(st)
    assert O.state_digest(st) == STATES["oracle"][key]


def test_acceptance_instances_digests():
    for inst in STATES["acceptance"][:60]:
        st = O.initialize(inst["total"], inst["sg"], inst["seed"])
        O.sequential_oracle(st, **inst["hyper"])
        assert O.state_digest(st) == inst["digest"], inst


@pytest.mark.parametrize("lowp", ["bf16", "fp16"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("scale", [1.0, 0.5, 1.0 / 3])
def test_reduce_scatter_oracle_matches_torch_loop(lowp, world, scale):
    """oracle.reduce_scatter (declared semantics; the reference has no
    collectives) against an independent torch CPU statement of the same
    rule: rank-order fp32 adds, one cast, scale, cast."""
    torch = pytest.importorskip("torch")
    tdt = torch.bfloat16 if lowp == "bf16" else torch.float16
    rng = np.random.default_rng(world)
    xs = [torch.from_numpy(rng.normal(0, 1.0, 50_000).astype(np.float32)).to(tdt) for _ in range(world)]
    acc = xs[0].float()
    for x in xs[1:]:
        acc = acc + x.float()
    want = acc.to(tdt)
    if scale != 1.0:
        want = (want.float() * torch.tensor(scale, dtype=torch.float32)).to(tdt)
    srcs = [x.view(torch.int16).numpy().view(np.uint16) for x in xs]
    if lowp == "fp16":
        srcs = [s.view(np.float16) for s in srcs]
    got = O.reduce_scatter(srcs, lowp, scale)
    assert np.asarray(got).view(np.uint16).tobytes() == want.view(torch.int16).numpy().view(np.uint16).tobytes()
