"""Summaries of ncu outputs for profiles/ (run here, on the CPU box)."""
import collections
import csv
import io
import json
import sys


def launches(path):
    text = open(path).read()
    text = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(text)))
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        import re

        if re.search(r"(^|::|\s)k_(adam|down|up|reduce|coherence|shuttle)", name):
            mt = re.search(r"(k_[a-z_]+)(<[^>]*>)?", name)
            short = "libdos:" + (mt.group(1) + (mt.group(2) or "") if mt else name[:60])
        else:
            short = "torch:" + name.split("(")[0][-70:]
        tot[short][0] += 1
        tot[short][1] += float(r["Metric Value"])
    all_ns = sum(v[1] for v in tot.values())
    return {k: {"launches": v[0], "total_us": round(v[1] / 1e3, 1), "share": round(v[1] / all_ns, 4)}
            for k, v in sorted(tot.items(), key=lambda x: -x[1][1])}


def full(path, n_params):
    raw = list(csv.reader(open(path)))
    h, u, v = raw[0], raw[1], raw[2]
    g = lambda k: v[h.index(k)]
    stalls = sorted(((float(v[i]), hh.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                     for i, hh in enumerate(h) if hh.startswith("smsp__average_warps_issue_stalled") and hh.endswith("ratio")),
                    reverse=True)[:4]
    d = {
        "kernel": g("Kernel Name")[:120],
        "grid": g("launch__grid_size"), "block": g("launch__block_size"),
        "registers": g("launch__registers_per_thread"),
        "gpu_time_us": float(g("gpu__time_duration.sum")),
        "dram_bytes_read": float(g("dram__bytes_read.sum")) * (1e9 if u[h.index("dram__bytes_read.sum")] == "Gbyte" else 1e6),
        "dram_bytes_write": float(g("dram__bytes_write.sum")) * (1e9 if u[h.index("dram__bytes_write.sum")] == "Gbyte" else 1e6),
        "dram_pct_of_peak_elapsed": float(g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")),
        "warps_active_pct": float(g("sm__warps_active.avg.pct_of_peak_sustained_active")),
        "issue_active_pct": float(g("smsp__issue_active.avg.pct_of_peak_sustained_active")),
        "top_stalls_warps_per_issue": stalls,
        "params_per_launch": n_params,
        "algorithmic_bytes_per_launch": 28 * n_params,
    }
    d["dram_bytes_per_launch"] = d["dram_bytes_read"] + d["dram_bytes_write"]
    d["traffic_over_algorithmic"] = d["dram_bytes_per_launch"] / d["algorithmic_bytes_per_launch"]
    d["dram_GBs_under_ncu"] = d["dram_bytes_per_launch"] / (d["gpu_time_us"] * 1e-6) / 1e9
    return d


if __name__ == "__main__":
    kind, path, out = sys.argv[1], sys.argv[2], sys.argv[3]
    res = launches(path) if kind == "launches" else full(path, int(float(sys.argv[4])))
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:2500])
