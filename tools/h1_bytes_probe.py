"""Where could the host lane save DRAM bytes?  (round-2 A/B probe)

H1 (host Adam, 16 threads) on 1e8-param subgroups of a 2 GB-per-array pinned
pool, alone and next to pinned DMA, in variants that differ only in host-DRAM
bytes per param:

* ``w_nt``   the product: bf16 working copy written with non-temporal stores
             into the big host image (2 B of DRAM write per param);
* ``no_w``   no working copy at all (the bound for a cache-resident ring:
             what H1 costs if its 2 B store never reaches DRAM).

and DMA patterns that differ in where the copy engine reads/writes host
memory:

* ``dma_cold``  H2D from / D2H into 1 GiB buffers (always DRAM);
* ``dma_hot``   the same byte rate from / into one 4 MiB buffer reused over
                and over (LLC-resident: does the copy engine read the cache,
                and do its writes stay there, on this host?).

If ``no_w`` under DMA is clearly faster than ``w_nt``, and H1 runs faster
next to ``dma_hot`` than next to ``dma_cold``, a chunked cache-resident
staging ring for the working copy (and for the in-phase grad flush) would buy
host-DRAM bandwidth; otherwise it cannot.
"""
from __future__ import annotations

import json
import sys
import threading
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2410_21316_b200 import _native as N  # noqa: E402

SG = 100_000_000
NSUB = 4  # distinct subgroups cycled (8 GB of p/m/v, far above the LLC)


def pool():
    hb = N.HostBuffer(NSUB * SG * 16)
    arrs = []
    for k in range(NSUB):
        base = k * SG * 16
        p = hb.array(np.float32, SG, base)
        m = hb.array(np.float32, SG, base + 4 * SG)
        v = hb.array(np.float32, SG, base + 8 * SG)
        g = hb.array(np.uint16, SG, base + 12 * SG)
        w = hb.array(np.uint16, SG, base + 14 * SG)
        p[:] = np.float32(0.01)
        m[:] = 0
        v[:] = np.float32(1e-5)
        g[:] = 0x3F80
        arrs.append((p, m, v, g, w))
    return hb, arrs


class Dma:
    """Duplex pinned DMA from a host buffer of `nbytes` (cycled in 4 MiB
    pieces so hot and cold move the same bytes per call)."""

    def __init__(self, nbytes: int, piece: int = 4 << 20, same: bool = False) -> None:
        # same=True: both directions on one buffer (the D2H writes land in the
        # LLC, if the host's DMA allocates there, and the H2D reads find them)
        self.hb = [N.HostBuffer(nbytes)] + ([] if same else [N.HostBuffer(nbytes)])
        self.hx = torch.from_numpy(self.hb[0].array(np.uint8, nbytes))
        self.hy = self.hx if same else torch.from_numpy(self.hb[1].array(np.uint8, nbytes))
        self.dx = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
        self.dy = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
        self.s1, self.s2 = torch.cuda.Stream(), torch.cuda.Stream()
        self.n, self.piece = nbytes, piece
        self.moved = 0
        self.stop = threading.Event()
        self.th = threading.Thread(target=self.run, daemon=True)

    def run(self) -> None:
        off = 0
        k = 16  # pieces per round (64 MiB each way)
        while not self.stop.is_set():
            for j in range(k):
                a = (off + j * self.piece) % self.n
                d = (j * self.piece) % (64 << 20)
                with torch.cuda.stream(self.s1):
                    self.dx[d:d + self.piece].copy_(self.hx[a:a + self.piece], non_blocking=True)
                with torch.cuda.stream(self.s2):
                    self.hy[a:a + self.piece].copy_(self.dy[d:d + self.piece], non_blocking=True)
            off = (off + k * self.piece) % self.n
            self.s1.synchronize()
            self.s2.synchronize()
            self.moved += 2 * k * self.piece

    def __enter__(self):
        self.th.start()
        time.sleep(0.1)
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join()


def h1_rate(arrs, with_w: bool, reps: int = 8) -> float:
    sc = N.scalars(1e-3, 0.9, 0.999, 1e-8, np.float32(0.1), np.float32(0.001))
    lib = N.lib()

    def one(k):
        p, m, v, g, w = arrs[k % NSUB]
        N.check(lib.dos_adam_step_host(p.ctypes.data, m.ctypes.data, v.ctypes.data, g.ctypes.data, N.DOS_BF16,
                                       w.ctypes.data if with_w else None, N.DOS_BF16 if with_w else N.DOS_NONE,
                                       SG, sc, 0))

    one(0)
    t0 = time.perf_counter()
    for k in range(reps):
        one(k)
    return reps * SG / (time.perf_counter() - t0)


def main() -> None:
    hb, arrs = pool()
    out = {"threads": N.lib().dos_host_threads()}
    for with_w, tag in ((True, "w_nt"), (False, "no_w")):
        out[f"{tag}_alone_Gps"] = h1_rate(arrs, with_w) / 1e9
    for dma_bytes, dtag in ((1 << 30, "dma_cold"), (4 << 20, "dma_hot")):
        dma = Dma(dma_bytes, same=dtag == "dma_hot")
        for with_w, tag in ((True, "w_nt"), (False, "no_w")):
            with dma as d:
                m0, t0 = d.moved, time.perf_counter()
                r = h1_rate(arrs, with_w)
                dt = time.perf_counter() - t0
                out[f"{tag}_{dtag}_Gps"] = r / 1e9
                out[f"{tag}_{dtag}_dma_GBs"] = (d.moved - m0) / dt / 1e9
            dma.stop.clear()
            dma.th = threading.Thread(target=dma.run, daemon=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
