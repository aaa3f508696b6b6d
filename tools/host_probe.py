"""Host-side probe on the GPU box: H1 scaling with threads, alone and under
full-duplex DMA, plus the C oracle port's scaling."""
import json, os, sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2410_21316_b200 import _native as N, profile_b200
out = {"cores": len(os.sched_getaffinity(0))}
for t in (1, 2, 4, 8, 12, 16):
    N.lib().dos_set_host_threads(t)
    a = profile_b200.measure_h1(100_000_000, reps=2)
    b = profile_b200.measure_h1(100_000_000, with_dma=True, reps=2)
    out[f"h1_t{t}"] = {"alone_Gps": round(a["h1_params_per_s"] / 1e9, 3), "dma_Gps": round(b["h1_params_per_s"] / 1e9, 3)}
    print(t, out[f"h1_t{t}"], flush=True)
N.lib().dos_set_host_threads(0)
link = profile_b200.measure_link(1 << 30)
out["link"] = link
# link while H1 runs on all cores
import threading
stop = threading.Event()
def hammer():
    while not stop.is_set():
        profile_b200.measure_h1(50_000_000, reps=1)
th = threading.Thread(target=hammer, daemon=True); th.start(); time.sleep(1.0)
out["link_under_h1"] = profile_b200.measure_link(1 << 30)
stop.set(); th.join()
from oracle import c_oracle
c_oracle.build()
for t in (1, 4, 8, 16):
    n = 100_000_000
    p = np.full(n, 0.01, np.float32); m = np.zeros(n, np.float32); v = np.full(n, 1e-5, np.float32)
    g = np.full(n, 0x3F80, np.uint16); w = np.empty(n, np.uint16)
    c_oracle.adam_mt(p, m, v, g, "bf16", w, "bf16", 1e-3, 0.9, 0.999, 1e-8, 1, nthreads=t)
    t0 = time.perf_counter()
    for s in range(3):
        c_oracle.adam_mt(p, m, v, g, "bf16", w, "bf16", 1e-3, 0.9, 0.999, 1e-8, 2 + s, nthreads=t)
    out[f"oracle_t{t}_Gps"] = round(3 * n / (time.perf_counter() - t0) / 1e9, 3)
    print(t, out[f"oracle_t{t}_Gps"], flush=True)
print(json.dumps(out))
json.dump(out, open("gpurun_out/host_probe.json", "w"), indent=1)
