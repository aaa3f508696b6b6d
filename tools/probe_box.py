"""One-off probe of the GPU box: topology, host RAM/cores, pinned link bandwidth."""
import os, subprocess, time, json
def sh(c):
    try: return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e: return str(e)
out = {}
for c in ["nvidia-smi", "nvidia-smi topo -m", "lscpu", "free -g", "cat /sys/fs/cgroup/cpu.max", "cat /sys/fs/cgroup/memory.max",
          "ls /sys/devices/system/node/", "cat /proc/meminfo | head -20", "ulimit -l", "cat /sys/kernel/mm/transparent_hugepage/enabled",
          "nproc", "python -c 'import numba; print(numba.__version__)'"]:
    out[c] = sh(c)
out["affinity"] = len(os.sched_getaffinity(0))
import torch
out["gpu_numa"] = sh("cat /sys/bus/pci/devices/*/numa_node | sort | uniq -c")
dev = torch.device("cuda:0")
torch.cuda.init()
p = torch.cuda.get_device_properties(0)
out["props"] = str(p)
out["mem_get_info"] = torch.cuda.mem_get_info()
res = {}
for gb in (1, 4):
    n = gb << 30
    t0 = time.time(); h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h.fill_(1); res[f"pin_{gb}GB_s"] = time.time() - t0
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True); d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(2):
        d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    def timed(fn, reps=5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(reps): fn()
        torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
    res[f"h2d_{gb}GB_GBs"] = n / timed(lambda: d.copy_(h, non_blocking=True)) / 1e9
    res[f"d2h_{gb}GB_GBs"] = n / timed(lambda: h.copy_(d, non_blocking=True)) / 1e9
    def duplex():
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    res[f"duplex_{gb}GB_GBs_per_dir"] = n / timed(duplex) / 1e9
    del h, d, h2, d2
# pageable
n = 1 << 30
hp = torch.empty(n, dtype=torch.uint8); hp.fill_(1); d = torch.empty(n, dtype=torch.uint8, device=dev)
torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(hp); torch.cuda.synchronize(); res["pageable_h2d_GBs"] = n / (time.perf_counter() - t0) / 1e9
t0 = time.perf_counter(); hp.copy_(d); torch.cuda.synchronize(); res["pageable_d2h_GBs"] = n / (time.perf_counter() - t0) / 1e9
# host memcpy bandwidth single thread (numpy)
import numpy as np
a = np.ones(1 << 28, dtype=np.float32); b = np.empty_like(a)
t0 = time.perf_counter(); np.copyto(b, a); res["host_copy_1thread_GBs"] = 2 * a.nbytes / (time.perf_counter() - t0) / 1e9
# big pin timing
t0 = time.time(); big = torch.empty(32 << 30, dtype=torch.uint8, pin_memory=True); res["pin_32GB_alloc_s"] = time.time() - t0
t0 = time.time(); big.fill_(0); res["pin_32GB_touch_s"] = time.time() - t0
del big
out["bw"] = res
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1, default=str)
print(json.dumps(res, indent=1))
