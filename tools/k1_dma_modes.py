"""K1 and a plain device-to-device copy (the HBM roofline's own kernel) while
the copy engines run nothing / H2D / D2H / both (pinned, 256 MiB chunks in a
loop): is the in-phase K1 slowdown specific to K1 or a property of HBM under
host-link DMA?"""
import json, sys, threading, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2410_21316_b200 import _native as N, profile_b200

nb = 1 << 28
hx = torch.from_numpy(N.HostBuffer(nb).array(np.uint8, nb))
hy = torch.from_numpy(N.HostBuffer(nb).array(np.uint8, nb))
dx = torch.empty(nb, dtype=torch.uint8, device="cuda")
dy = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
src = torch.empty(1 << 31, dtype=torch.uint8, device="cuda")
dst = torch.empty_like(src)


def d2d_GBs(reps=10):
    dst.copy_(src)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dst.copy_(src)
    e1.record()
    torch.cuda.synchronize()
    return 2 * src.numel() * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


def run(mode):
    stop = threading.Event()
    moved = [0]

    def pump():
        while not stop.is_set():
            if mode in ("h2d", "duplex"):
                with torch.cuda.stream(s1):
                    dx.copy_(hx, non_blocking=True)
            if mode in ("d2h", "duplex"):
                with torch.cuda.stream(s2):
                    hy.copy_(dy, non_blocking=True)
            s1.synchronize()
            s2.synchronize()
            moved[0] += nb * (2 if mode == "duplex" else 1)

    th = None
    if mode != "none":
        th = threading.Thread(target=pump, daemon=True)
        th.start()
        time.sleep(0.2)
    t0 = time.perf_counter()
    k1 = profile_b200.measure_k1(100_000_000, reps=20)["k1_GBs"]
    cp = d2d_GBs()
    dt = time.perf_counter() - t0
    if th:
        stop.set()
        th.join()
    return {"mode": mode, "k1_GBs": k1, "d2d_copy_GBs": cp, "dma_GBs_total": moved[0] / dt / 1e9}


out = [run(m) for m in ("none", "h2d", "d2h", "duplex", "none")]
for r in out:
    print(json.dumps(r), flush=True)
