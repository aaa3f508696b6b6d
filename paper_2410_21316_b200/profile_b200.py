"""Measure the ``b200-node`` SystemProfile on the machine at hand.

The performance model (Eq. 1) is only as good as its constants; the
reference ships hand-entered V100/H100 numbers (catalog.py:23-51).  Here
every constant the planner uses is measured on the B200 box, quickly enough
to re-fit per iteration:

* ``channel_params_per_s``       pinned H2D and D2H run *concurrently*
                                 (duplex, as in the interleaved phase), the
                                 slower direction / 4 B per fp32 param;
* ``fast_update_params_per_s``   K1 on one subgroup resident in HBM;
* ``cpu_update_params_per_s``    H1 (fused Adam + working-copy store) on the
                                 host team, while the link is busy (the
                                 contended rate, which is what the phase sees);
* ``cpu_downscale_params_per_s`` inf: the downscale is fused into H1;
* ``host_contention``            H1 alone / H1 under concurrent DMA (>= 1).
"""

from __future__ import annotations

import ctypes
import dataclasses
import json
import threading
import time
from pathlib import Path

import numpy as np

from . import _native as N
from .state import SystemProfile

_OUT = Path(__file__).resolve().parent.parent / "profiles" / "b200_node_profile.json"
LAST_RAW: dict = {}  # raw measurements behind the last measure_profile()


def _torch():
    import torch

    return torch


_LINK_BUFS: dict = {}  # nbytes -> probe buffers, allocated once per process and reused


def _wait(*streams) -> None:
    """Wait for ``streams`` on blocking-sync events: the waiting thread sleeps
    instead of spinning on a core (a spinning probe thread steals a core from
    the host team it runs next to and makes the team's static shares straggle)."""
    torch = _torch()
    for st in streams:
        ev = torch.cuda.Event(blocking=True)
        ev.record(st)
        ev.synchronize()


def _link_buffers(nbytes: int, numa_node: int = -1):
    """Pinned probe buffers of ``nbytes`` (pre-faulted huge pages, registered),
    allocated on first use and kept: a probe late in a run reuses the pages it
    got at start-up instead of fresh ones from a fragmented host (which
    measured the link 30-40% low in round 1).  The device twins are made per
    probe and freed after it, so they never hold HBM a capacity-aware
    residency could use."""
    torch = _torch()
    key = (nbytes, numa_node, torch.cuda.current_device())
    if key not in _LINK_BUFS:
        hb1, hb2 = N.HostBuffer(nbytes, numa_node=numa_node), N.HostBuffer(nbytes, numa_node=numa_node)
        h1 = torch.from_numpy(hb1.array(np.uint8, nbytes))
        h2 = torch.from_numpy(hb2.array(np.uint8, nbytes))
        _LINK_BUFS[key] = (hb1, hb2, h1, h2, torch.cuda.Stream(), torch.cuda.Stream())
    return _LINK_BUFS[key]


def measure_link(nbytes: int = 1 << 30, reps: int = 3, numa_node: int = -1) -> dict:
    """Pinned host<->device GB/s: each direction alone and both at once
    (best of ``reps``; buffers reused across calls, see ``_link_buffers``)."""
    torch = _torch()
    _, _, h1, h2, s1, s2 = _link_buffers(nbytes, numa_node)
    d1 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")

    def timed(fn) -> float:
        fn()
        _wait(s1, s2)
        best = float("inf")
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            _wait(s1, s2)
            best = min(best, time.perf_counter() - t0)
        return best

    def h2d():
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    t_h2d = timed(h2d)
    t_d2h = timed(d2h)
    t_dup = timed(lambda: (h2d(), d2h()))
    del d1, d2  # every copy has finished (timed() waits on both streams)
    torch.cuda.empty_cache()
    return {"h2d_GBs": nbytes / t_h2d / 1e9, "d2h_GBs": nbytes / t_d2h / 1e9,
            "duplex_GBs_per_dir": nbytes / t_dup / 1e9}


def measure_link_under_h1(nbytes: int = 1 << 28, n: int = 50_000_000) -> dict:
    """Duplex link GB/s while H1 runs on every host thread — the copy
    engines and the host team share the host DRAM, so the link slows."""
    hb = N.HostBuffer(n * 16)
    p, m, v = (hb.array(np.float32, n, k * 4 * n) for k in range(3))
    g, w = hb.array(np.uint16, n, 12 * n), hb.array(np.uint16, n, 14 * n)
    p[:] = np.float32(0.01)
    m[:] = 0
    v[:] = np.float32(1e-5)
    g[:] = 0x3F80
    sc = N.scalars(1e-3, 0.9, 0.999, 1e-8, np.float32(0.1), np.float32(0.001))
    lib = N.lib()
    stop = threading.Event()

    def hammer():
        while not stop.is_set():
            lib.dos_adam_step_host(p.ctypes.data, m.ctypes.data, v.ctypes.data, g.ctypes.data, N.DOS_BF16,
                                   w.ctypes.data, N.DOS_BF16, n, sc, 0)

    th = threading.Thread(target=hammer, daemon=True)
    th.start()
    time.sleep(0.05)
    try:
        res = measure_link(nbytes)
    finally:
        stop.set()
        th.join()
    return res


def measure_k1(n: int = 100_000_000, reps: int = 5, with_dma: bool = False) -> dict:
    """K1 params/s and achieved HBM GB/s (28 B/param) on one subgroup.

    ``with_dma``: also K1 and a plain device-to-device copy (the HBM
    roofline's own kernel) while duplex pinned DMA runs on two other streams,
    as inside a phase: the copy's rate there is the HBM ceiling the in-phase
    K1 can reach (host-link DMA costs HBM more than its own bytes;
    profiles/r02_k1_variants_dma.jsonl)."""
    torch = _torch()
    dev = torch.device("cuda")
    p = torch.randn(n, device=dev) * 0.02
    m = torch.randn(n, device=dev) * 1e-3
    v = torch.rand(n, device=dev) * 1e-4
    g = torch.randn(n, device=dev).to(torch.bfloat16)
    w = torch.empty(n, dtype=torch.bfloat16, device=dev)
    sc = N.scalars(1e-3, 0.9, 0.999, 1e-8, np.float32(0.1), np.float32(0.001))
    st = torch.cuda.current_stream()
    lib = N.lib()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def run():
        N.check(lib.dos_adam_step_cuda(p.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(), N.DOS_BF16,
                                       w.data_ptr(), N.DOS_BF16, n, sc, st.cuda_stream))

    for _ in range(3):
        run()
    times = []
    for _ in range(reps):
        e0.record(st)
        run()
        e1.record(st)
        e1.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
    t = float(np.median(times))
    out = {"k1_params_per_s": n / t, "k1_GBs": 28 * n / t / 1e9, "k1_ms": t * 1e3, "n": n}
    if with_dma:
        # 2 GB each way, less when the HBM is mostly taken (capacity-aware residency)
        nb = min(1 << 31, (torch.cuda.mem_get_info(dev)[0] - (2 << 30)) // 2) & ~((1 << 20) - 1)
        if nb < (256 << 20):
            out["under_duplex_dma_skipped"] = {"skipped": "no HBM left for the device-copy buffers"}
            return out
        src = torch.empty(nb, dtype=torch.uint8, device=dev)
        dst = torch.empty_like(src)

        def timed(fn) -> float:
            fn()
            ts = []
            for _ in range(reps):
                e0.record(st)
                fn()
                e1.record(st)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3)
            return float(np.median(ts))

        copy = lambda: dst.copy_(src)
        out["d2d_copy_GBs"] = 2 * src.numel() / timed(copy) / 1e9
        with _DuplexPump() as pump:
            t0, m0 = time.perf_counter(), pump.moved
            tk = timed(run)
            tc = timed(copy)
            dma = (pump.moved - m0) / (time.perf_counter() - t0)
        out["under_duplex_dma"] = {"k1_GBs": 28 * n / tk / 1e9, "d2d_copy_GBs": 2 * src.numel() / tc / 1e9,
                                   "dma_GBs": dma / 1e9}
        del src, dst
        torch.cuda.empty_cache()
    return out


def measure_h1(n: int = 100_000_000, with_dma: bool = False, reps: int = 3) -> dict:
    """H1 params/s (fused Adam + bf16 store) on the host team."""
    hb = N.HostBuffer(n * 16)
    p = hb.array(np.float32, n, 0)
    m = hb.array(np.float32, n, 4 * n)
    v = hb.array(np.float32, n, 8 * n)
    g = hb.array(np.uint16, n, 12 * n)
    w = hb.array(np.uint16, n, 14 * n)
    rng = np.random.default_rng(0)
    p[:] = rng.standard_normal(n, dtype=np.float32) * np.float32(0.02)
    m[:] = 0
    v[:] = np.float32(1e-5)
    g[:] = 0x3F80
    sc = N.scalars(1e-3, 0.9, 0.999, 1e-8, np.float32(0.1), np.float32(0.001))
    lib = N.lib()
    stop = threading.Event()
    dma = None
    if with_dma:
        torch = _torch()
        nb = 1 << 26  # 64 MB per direction per round: fine-grained byte accounting
        hx = torch.from_numpy(N.HostBuffer(nb).array(np.uint8, nb))
        hy = torch.from_numpy(N.HostBuffer(nb).array(np.uint8, nb))
        dx = torch.empty(nb, dtype=torch.uint8, device="cuda")
        dy = torch.empty(nb, dtype=torch.uint8, device="cuda")
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

        moved = [0]  # host bytes read + written by the copy engines

        def pump():
            while not stop.is_set():
                with torch.cuda.stream(s1):
                    dx.copy_(hx, non_blocking=True)
                with torch.cuda.stream(s2):
                    hy.copy_(dy, non_blocking=True)
                _wait(s1, s2)
                moved[0] += 2 * nb

        dma = threading.Thread(target=pump, daemon=True)
        dma.start()
        time.sleep(0.05)
    run = lambda: N.check(lib.dos_adam_step_host(p.ctypes.data, m.ctypes.data, v.ctypes.data, g.ctypes.data,
                                                  N.DOS_BF16, w.ctypes.data, N.DOS_BF16, n, sc, 0))
    t0 = time.perf_counter()
    run()
    if dma is not None:  # a window of >= 0.4 s, so the DMA byte count (64 MB grains) is fine enough
        reps = max(reps, int(0.4 / max(1e-3, time.perf_counter() - t0)) + 1)
    best = float("inf")
    t_all0 = time.perf_counter()
    moved0 = moved[0] if dma is not None else 0
    for _ in range(reps):
        t0 = time.perf_counter()
        run()
        best = min(best, time.perf_counter() - t0)
    t_all = time.perf_counter() - t_all0
    out = {"h1_params_per_s": n / best, "h1_GBs": 28 * n / best / 1e9, "threads": lib.dos_host_threads()}
    if dma is not None:
        dma_bytes = moved[0] - moved0
        stop.set()
        dma.join()
        # host DRAM bytes per second while H1 and duplex DMA share the memory
        out["dma_GBs"] = dma_bytes / t_all / 1e9
        out["host_dram_GBs_combined"] = (28 * n * reps + dma_bytes) / t_all / 1e9
    return out


class _DuplexPump:
    """Pinned duplex DMA in a background thread (64 MB per direction per
    round); ``moved`` counts the host bytes the copy engines read + wrote."""

    def __init__(self, nb: int = 1 << 26) -> None:
        torch = _torch()
        self.hx = torch.from_numpy(N.HostBuffer(nb).array(np.uint8, nb))
        self.hy = torch.from_numpy(N.HostBuffer(nb).array(np.uint8, nb))
        self.dx = torch.empty(nb, dtype=torch.uint8, device="cuda")
        self.dy = torch.empty(nb, dtype=torch.uint8, device="cuda")
        self.s1, self.s2 = torch.cuda.Stream(), torch.cuda.Stream()
        self.nb, self.moved = nb, 0
        self.stop = threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self) -> None:
        torch = _torch()
        while not self.stop.is_set():
            with torch.cuda.stream(self.s1):
                self.dx.copy_(self.hx, non_blocking=True)
            with torch.cuda.stream(self.s2):
                self.hy.copy_(self.dy, non_blocking=True)
            _wait(self.s1, self.s2)
            self.moved += 2 * self.nb

    def __enter__(self):
        self.th.start()
        time.sleep(0.05)
        return self

    def __exit__(self, *exc):
        self.stop.set()
        self.th.join()


def measure_host_dram(nbytes: int = 1 << 31, reps: int = 3, with_dma: bool = True) -> dict:
    """Host DRAM throughput of the whole team: a read pass and a copy pass
    (memcpy, non-temporal stores), alone and with duplex pinned DMA running
    (bytes the copy engines move count too).  ``peak_GBs`` — the best of
    these — is the host-DRAM roofline's denominator."""
    src = N.HostBuffer(nbytes)
    dst = N.HostBuffer(nbytes)
    lib = N.lib()
    secs = ctypes.c_double()
    out: dict = {}

    def one(mode: int) -> tuple[float, int]:
        N.check(lib.dos_host_membw(src.address, dst.address, nbytes, mode, 0, ctypes.byref(secs)))
        return secs.value, nbytes * (1 if mode == 0 else 2)

    for mode, name in ((0, "read"), (1, "copy")):
        one(mode)
        out[f"{name}_GBs"] = max(b / t for t, b in (one(mode) for _ in range(reps))) / 1e9
        if with_dma:
            with _DuplexPump() as pump:
                t0, m0, cpu = time.perf_counter(), pump.moved, 0
                for _ in range(reps):
                    cpu += one(mode)[1]
                dt, dma = time.perf_counter() - t0, pump.moved - m0
            out[f"{name}_with_dma_GBs_combined"] = (cpu + dma) / dt / 1e9
            out[f"{name}_with_dma_dma_GBs"] = dma / dt / 1e9
    out["peak_GBs"] = max(v for k, v in out.items() if k.endswith("_GBs") or k.endswith("_combined"))
    return out


def host_rates():
    """``policy.HostRates`` from the last ``measure_profile`` in this process,
    else from the committed measurement (``profiles/b200_node_profile.json``),
    else None."""
    from .policy import HostRates

    raw = LAST_RAW
    if not raw and _OUT.exists():
        try:
            raw = json.loads(_OUT.read_text()).get("raw", {})
        except (OSError, ValueError):
            raw = {}
    if not raw or "link" not in raw or "h1_alone" not in raw or "k1" not in raw:
        return None
    return HostRates(link_bytes_per_s=raw["link"]["duplex_GBs_per_dir"] * 1e9,
                     host_params_per_s=raw["h1_alone"]["h1_params_per_s"],
                     fast_params_per_s=raw["k1"]["k1_params_per_s"],
                     host_dram_bytes_per_s=max(raw.get("host_dram", {}).get("peak_GBs", 0.0),
                                               raw.get("h1_with_dma", {}).get("host_dram_GBs_combined", 0.0),
                                               raw["h1_alone"]["h1_GBs"]) * 1e9)


def measure_profile(fast_capacity_bytes: int | None = None, save: bool = False, quick: bool = False) -> SystemProfile:
    """Measure all planner constants on this box; returns a SystemProfile."""
    n = 25_000_000 if quick else 100_000_000
    link = measure_link(1 << 28 if quick else 1 << 30)
    k1 = measure_k1(n)
    h1_alone = measure_h1(n)
    h1_busy = measure_h1(100_000_000, with_dma=True)
    channel = min(link["duplex_GBs_per_dir"], link["h2d_GBs"], link["d2h_GBs"]) * 1e9 / 4.0
    contention = max(1.0, h1_alone["h1_params_per_s"] / h1_busy["h1_params_per_s"])
    prof = SystemProfile(
        name="b200-node",
        channel_params_per_s=channel,
        fast_update_params_per_s=k1["k1_params_per_s"],
        cpu_update_params_per_s=h1_alone["h1_params_per_s"],
        cpu_downscale_params_per_s=float("inf"),
        fast_convert_bytes_per_s=2.0 * k1["k1_params_per_s"],
        host_convert_bytes_per_s=2.0 * h1_alone["h1_params_per_s"],
        host_alloc_bytes_per_s=4e9,
        pageable_d2h_bytes_per_s=link["d2h_GBs"] * 1e9 / 3.0,
        pageable_h2d_bytes_per_s=link["h2d_GBs"] * 1e9 / 5.0,
        fast_capacity_bytes=fast_capacity_bytes,
        host_contention=contention,
        caveat="measured by profile_b200.measure_profile",
    )
    link_h1 = measure_link_under_h1(1 << 28)
    dram = measure_host_dram(1 << 30 if quick else 1 << 31)
    LAST_RAW.clear()
    LAST_RAW.update({"link": link, "k1": k1, "h1_alone": h1_alone, "h1_with_dma": h1_busy, "link_under_h1": link_h1,
                     "host_dram": dram,
                     "link_slowdown_under_h1": max(1.0, link["duplex_GBs_per_dir"] / link_h1["duplex_GBs_per_dir"])})
    if save:
        d = dataclasses.asdict(prof)
        d["raw"] = {"link": link, "k1": k1, "h1_alone": h1_alone, "h1_with_dma": h1_busy, "host_dram": dram,
                    "link_under_h1": link_h1, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
        _OUT.parent.mkdir(exist_ok=True)
        _OUT.write_text(json.dumps(d, indent=1))
    return prof


if __name__ == "__main__":
    import sys

    prof = measure_profile(save="--save" in sys.argv, quick="--quick" in sys.argv)
    print(json.dumps(dataclasses.asdict(prof), indent=1))
