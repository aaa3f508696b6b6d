"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
implementation (the `optistate` package at /root/reference/pkg/src) in this
container.  The fixtures travel; /root/reference does not.

    python tests/golden/make_goldens.py          # rewrites the fixtures

Everything stored is either small arrays or sha256 digests of canonical
encodings, so the files stay small.
"""
from __future__ import annotations

import hashlib
import json
import math
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import optistate as R  # noqa: E402
from optistate import kernels as RK  # noqa: E402


def plan_canon(plan) -> str:
    """Canonical text of a plan: independent of the enum classes used."""
    parts = [
        f"n={plan.num_subgroups}",
        "static=" + ",".join(map(str, sorted(plan.static_set))),
        "dev=" + "".join("F" if d.value == "fast" else "C" for d in plan.devices),
        "dyn=" + ",".join(map(str, plan.dynamic_fast)),
        f"blocking={int(plan.blocking)}",
    ]
    for a in plan.actions:
        parts.append(
            f"{a.id}:{a.kind.value}:{a.subgroup}:{a.lane.value}:{a.stream.value if a.stream else '-'}:"
            f"{','.join(map(str, a.batch))}:{','.join(map(str, a.deps))}"
        )
    return "\n".join(parts)


def events_canon(events) -> str:
    return "\n".join(f"{e.action.id}:{e.start_ns}:{e.end_ns}:{e.bytes}" for e in events)


def sha(s: str | bytes) -> str:
    return hashlib.sha256(s.encode() if isinstance(s, str) else s).hexdigest()


def state_digest(opt) -> str:
    h = hashlib.sha256()
    for a in (opt.params32, opt.momentum32, opt.variance32, opt.model16, opt.grads16):
        h.update(a.tobytes())
    return h.hexdigest()


def strides():
    return [1, 2, 3, 4, 5, 6, 7, R.ALL_CPU]


def stride_key(s) -> str:
    return "all_cpu" if s is R.ALL_CPU else str(s)


def gen_plans():
    out = {}
    ratios = [0.0, 0.1, 0.2, 0.25, 0.3, 0.375, 0.5, 0.75, 1.0]
    import warnings
    for n in list(range(0, 26)) + [50, 65, 70, 88, 130]:
        for s in strides():
            for r in ratios:
                for pl in R.Placement:
                    with warnings.catch_warnings():
                        warnings.simplefilter("ignore")
                        plan = R.build_plan(n, s, static_ratio=r, placement=pl)
                    out[f"{n}|{stride_key(s)}|{r}|{pl.value}"] = sha(plan_canon(plan))
    # a few plans in full, for readable diffs when a digest fails
    full = {}
    for key in ["3|1|0.0|static_last", "10|3|0.0|static_last", "8|2|0.375|static_first", "4|all_cpu|0.0|static_last",
                "8|3|0.25|static_last", "6|all_cpu|0.5|static_first"]:
        n, s, r, pl = key.split("|")
        plan = R.build_plan(int(n), R.ALL_CPU if s == "all_cpu" else int(s), float(r), R.Placement(pl))
        full[key] = plan_canon(plan)
    return {"digests": out, "full": full}


def gen_sim():
    out = {}
    for prof_name in ("v100-node", "h100-node"):
        prof = R.get_profile(prof_name)
        for n in (1, 2, 5, 8, 12, 25, 50, 70):
            for s in strides():
                for r, pl in ((0.0, R.Placement.STATIC_LAST), (0.25, R.Placement.STATIC_LAST), (0.3, R.Placement.STATIC_FIRST)):
                    for size in (100_000_000, 1000, 7_812_500):
                        plan = R.build_plan(n, s, r, pl)
                        tl = R.simulate_update_phase(plan, prof, size)
                        out[f"{prof_name}|{n}|{stride_key(s)}|{r}|{pl.value}|{size}"] = {
                            "makespan": tl.makespan_ns, "span": tl.span_ns, "spill": tl.spillover_ns,
                            "peak": tl.peak_fast_bytes, "events": sha(events_canon(tl.events)),
                            "busy": {k.value: v for k, v in tl.lane_busy_ns.items()},
                        }
        # capacity-gated plans
        import dataclasses
        for cap_w in (1, 2, 3):
            for s in (1, 2, 3):
                p2 = dataclasses.replace(prof, fast_capacity_bytes=12 * 1000 * cap_w)
                plan = R.build_plan(8, s)
                tl = R.simulate_update_phase(plan, p2, 1000)
                out[f"{prof_name}|cap{cap_w}|{s}"] = {"makespan": tl.makespan_ns, "span": tl.span_ns,
                                                      "peak": tl.peak_fast_bytes, "events": sha(events_canon(tl.events))}
        # ragged sizes
        plan = R.build_plan(4, 2)
        tl = R.simulate_update_phase(plan, prof, [1000, 1000, 1000, 500])
        out[f"{prof_name}|ragged"] = {"makespan": tl.makespan_ns, "events": sha(events_canon(tl.events))}
    return out


def gen_perfmodel():
    out = {}
    for name in ("v100-node", "h100-node"):
        prof = R.get_profile(name)
        r = R.optimal_stride(prof)
        out[name] = {"k_real": r.k_real, "k": stride_key(r.k),
                     "est": {f"{k}|{st}": R.estimate_update_time(prof, 40, 10**8, k if k != "all" else R.ALL_CPU, st)
                             for k in (1, 2, 3, 5, "all") for st in (0, 7)}}
    rng = np.random.default_rng(7)
    rand = []
    for _ in range(300):
        kw = dict(name="r", channel_params_per_s=float(10 ** rng.uniform(8.5, 11)),
                  fast_update_params_per_s=float(10 ** rng.uniform(10, 11.5)),
                  cpu_update_params_per_s=float(10 ** rng.uniform(8, 10.5)),
                  cpu_downscale_params_per_s=float(10 ** rng.uniform(9, 11)),
                  fast_convert_bytes_per_s=1e12, host_convert_bytes_per_s=3e10, host_alloc_bytes_per_s=4e9,
                  pageable_d2h_bytes_per_s=6e9, pageable_h2d_bytes_per_s=5.5e9,
                  host_contention=float(rng.choice([1.0, 1.0, 1.3, 2.0])))
        prof = R.SystemProfile(**kw)
        r = R.optimal_stride(prof)
        rand.append({"profile": kw, "k_real": r.k_real if math.isfinite(r.k_real) else "inf", "k": stride_key(r.k)})
    out["random"] = rand
    return out


def gen_kernel_vectors():
    """Adam vectors: inputs and reference outputs (numba backend)."""
    cases = []
    arrays = {}
    specs = [(16, 42, 5, (1e-3, 0.9, 0.999, 1e-8)), (1, 0, 1, (1e-3, 0.9, 0.999, 1e-8)),
             (7, 1, 3, (1e-3, 0.9, 0.999, 1e-8)), (1024, 2, 3, (1e-3, 0.9, 0.999, 1e-8)),
             (4097, 3, 3, (1e-3, 0.9, 0.999, 1e-8)), (2048, 4, 1, (3e-4, 0.8, 0.95, 1e-6)),
             (3001, 5, 1000, (1e-2, 0.95, 0.9995, 1e-9)), (999, 6, 2, (1e-4, 0.85, 0.98, 1e-7))]
    for ci, (n, seed, step, (lr, b1, b2, eps)) in enumerate(specs):
        rng = np.random.default_rng(seed)
        p = rng.normal(0, 0.02, n).astype(np.float32)
        m = rng.normal(0, 1e-3, n).astype(np.float32)
        v = (rng.random(n) * 1e-4).astype(np.float32)
        g = rng.normal(0, 1.0, n).astype(np.float32)
        arrays[f"c{ci}_in_p"], arrays[f"c{ci}_in_m"], arrays[f"c{ci}_in_v"], arrays[f"c{ci}_g"] = p, m, v, g
        p2, m2, v2 = p.copy(), m.copy(), v.copy()
        RK.adam_step_arrays(p2, m2, v2, g, lr, b1, b2, eps, step)
        arrays[f"c{ci}_out_p"], arrays[f"c{ci}_out_m"], arrays[f"c{ci}_out_v"] = p2, m2, v2
        cases.append({"n": n, "seed": seed, "step": step, "lr": lr, "beta1": b1, "beta2": b2, "eps": eps})
    np.savez_compressed(OUT / "adam_vectors.npz", **arrays)
    return {"backend": RK.active_backend(), "cases": cases}


def gen_fp16():
    rng = np.random.default_rng(20240901)
    u = rng.integers(0, 2**32, size=50_000, dtype=np.uint32)
    extra = np.array([0x7FC00000, 0x7F800001, 0xFFC00001, 0x7FABCDEF, 0xFF800001, 0, 0x80000000, 0x7F800000,
                      0x477FF000, 0x477FEFFF, 0x33000000, 0x33000001, 0x387FC000, 0x38800000], dtype=np.uint32)
    u = np.concatenate([u, extra])
    with np.errstate(over="ignore"):
        h = R.downscale_rne(u.view(np.float32)).view(np.uint16)
    np.savez_compressed(OUT / "fp16_vectors.npz", f32_bits=u, f16_bits=h)


def gen_states():
    """Digests of sequential_oracle / execute_plan results on seeded shards,
    including the acceptance suite's 236 instances (test_acceptance.py:121-175)."""
    out = {"oracle": {}, "acceptance": []}
    for total, sg, seed in ((10 * 1024, 1024, 11), (5000, 1024, 5), (2048, 512, 2), (1536, 256, 8),
                            (12 * 257, 257, 4242), (125_000, 7_813, 1)):
        opt = R.ShardedOptimizer.initialize(total, sg, seed=seed)
        out["oracle"][f"{total}|{sg}|{seed}|init"] = state_digest(opt)
        R.sequential_oracle(opt, R.AdamHyper())
        out["oracle"][f"{total}|{sg}|{seed}|1"] = state_digest(opt)
        R.sequential_oracle(opt, R.AdamHyper())
        out["oracle"][f"{total}|{sg}|{seed}|2"] = state_digest(opt)
    rng = np.random.default_rng(20250816)
    ratios = (0.0, 0.25, 0.5)
    placements = (R.Placement.STATIC_FIRST, R.Placement.STATIC_LAST)
    for _ in range(200):
        n = int(rng.integers(1, 65))
        sg_size = int(rng.integers(8, 4097))
        total = (n - 1) * sg_size + int(rng.integers(1, sg_size + 1))
        hyper = dict(lr=float(10 ** rng.uniform(-4, -2)), beta1=float(rng.uniform(0.8, 0.95)),
                     beta2=float(rng.uniform(0.95, 0.9995)), eps=float(10 ** rng.uniform(-9, -6)))
        stride = int(rng.integers(1, 7))
        seed = int(rng.integers(0, 2**31))
        ratio = ratios[rng.integers(0, len(ratios))]
        pl = placements[rng.integers(0, len(placements))]
        opt = R.ShardedOptimizer.initialize(total, sg_size, seed=seed)
        R.sequential_oracle(opt, R.AdamHyper(**hyper))
        out["acceptance"].append({"total": total, "sg": sg_size, "seed": seed, "stride": stride, "ratio": ratio,
                                  "placement": pl.value, "hyper": hyper, "digest": state_digest(opt)})
    opt = R.ShardedOptimizer.initialize(12 * 257, 257, seed=4242)
    R.sequential_oracle(opt, R.AdamHyper())
    out["fixed_4242"] = state_digest(opt)
    return out


def main():
    meta = {"generator": "tests/golden/make_goldens.py", "reference": str(REF), "numpy": np.__version__}
    (OUT / "plans.json").write_text(json.dumps(gen_plans(), sort_keys=True))
    (OUT / "sim.json").write_text(json.dumps(gen_sim(), sort_keys=True))
    (OUT / "perfmodel.json").write_text(json.dumps(gen_perfmodel(), sort_keys=True))
    kv = gen_kernel_vectors()
    gen_fp16()
    st = gen_states()
    (OUT / "kernel_meta.json").write_text(json.dumps({**meta, **kv}, sort_keys=True, indent=1))
    (OUT / "states.json").write_text(json.dumps(st, sort_keys=True))
    print("ok")


if __name__ == "__main__":
    main()
