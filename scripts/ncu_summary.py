"""Summarise an ncu --set full report: per kernel launch, time, DRAM bytes,
throughput vs the measured peak, tensor-pipe %, top stall reasons."""
import csv
import json
import subprocess
import sys

rep = sys.argv[1]
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if len(sys.argv) < 3 else float(sys.argv[2])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
units = rows[1]


def g(r, key):
    i = hdr.index(key)
    v = r[i].replace(",", "")
    u = units[i]
    try:
        x = float(v)
    except ValueError:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
    return x * scale


print("| kernel | time (us) | DRAM read+write (MB) | DRAM GB/s | frac of measured peak | tensor pipe active % | top stalls (per issue) |")
print("|---|---|---|---|---|---|---|")
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")[:40]
    t = g(r, "gpu__time_duration.sum")
    rd = g(r, "dram__bytes_read.sum") or 0
    wr = g(r, "dram__bytes_write.sum") or 0
    tp = g(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
    stalls = []
    for h in hdr:
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            v = g(r, h)
            if v:
                stalls.append((v, h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
    stalls = ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)[:3] if n != "selected")
    gbs = (rd + wr) / t / 1e9
    print(f"| {name} | {t*1e6:.1f} | {(rd+wr)/1e6:.1f} | {gbs:.0f} | {gbs/peak:.3f} | {tp:.1f} | {stalls} |")
