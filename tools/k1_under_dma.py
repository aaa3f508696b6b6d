"""K1 alone vs K1 while the copy engines run duplex pinned DMA (as in the
phase): does host-link traffic slow the HBM-bound kernel?"""
import json, sys, threading, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2410_21316_b200 import _native as N, profile_b200

alone = profile_b200.measure_k1(100_000_000, reps=10)
nb = 1 << 28
hx = torch.from_numpy(N.HostBuffer(nb).array(np.uint8, nb))
hy = torch.from_numpy(N.HostBuffer(nb).array(np.uint8, nb))
dx = torch.empty(nb, dtype=torch.uint8, device="cuda")
dy = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
stop = threading.Event()


def pump():
    while not stop.is_set():
        with torch.cuda.stream(s1):
            dx.copy_(hx, non_blocking=True)
        with torch.cuda.stream(s2):
            hy.copy_(dy, non_blocking=True)
        s1.synchronize()
        s2.synchronize()


th = threading.Thread(target=pump, daemon=True)
th.start()
time.sleep(0.2)
busy = profile_b200.measure_k1(100_000_000, reps=10)
stop.set()
th.join()
print(json.dumps({"alone_GBs": alone["k1_GBs"], "with_duplex_dma_GBs": busy["k1_GBs"]}))
