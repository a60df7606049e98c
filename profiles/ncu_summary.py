"""Summarize an ncu report: per-kernel time, DRAM bytes, throughput, occupancy, top stalls."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "rdMB", "dram__bytes_write.sum": "wrMB",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "warps%",
        "launch__registers_per_thread": "regs", "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
        "launch__grid_size": "grid", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64%"}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0]
    vals = []
    for k, lab in want.items():
        v = d.get(k, "")
        try:
            f = float(v)
            if lab == "us":
                unit = rows[1][hdr.index(k)]
                f = f / 1000.0 if unit == "ns" else (f * 1000.0 if unit == "ms" else f)
            vals.append(f"{lab}={f:.1f}")
        except ValueError:
            vals.append(f"{lab}=?")
    stalls = sorted(((float(v), h.split("issue_stalled_")[1].split("_per")[0]) for h, v in d.items()
                     if "average_warps_issue_stalled" in h and "per_issue_active" in h and v.replace('.', '', 1).isdigit()),
                    reverse=True)[:4]
    print(f"{name:14s} " + " ".join(vals) + " | " + ", ".join(f"{n}:{v:.1f}" for v, n in stalls))
