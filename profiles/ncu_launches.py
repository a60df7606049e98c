"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file):
per kernel name the launch count, mean duration and share of the libhsx kernel time.

    python profiles/ncu_launches.py gpurun_out/TAG_launches.csv "header line" > profiles/TAG_ncu_launches_summary.txt
"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
acc = OrderedDict()
for r in rows[1:]:
    name = r[ik].split("(")[0][:45]
    us = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    n, t = acc.get(name, (0, 0.0))
    acc[name] = (n + 1, t + us)
hsx = sum(t for k, (n, t) in acc.items() if "hsx::" in k) or 1.0
if len(sys.argv) > 2:
    print(sys.argv[2])
for k, (n, t) in acc.items():
    share = t / hsx if "hsx::" in k else 0.0
    print(f"{k:45s}  n={n:3d} mean={t / n:8.1f} us  share_of_hsx={share:.3f}")
