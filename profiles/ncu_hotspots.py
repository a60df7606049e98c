"""Top SASS lines of one kernel by a stall reason: python profiles/ncu_hotspots.py REP KERNEL_REGEX [stall_col]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
col = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data = rows[1], rows[2:]
i_src, i_s = hdr.index("Source"), hdr.index(col)
seen = set()
data = [r for r in data if len(r) == len(hdr) and not (r[0] in seen or seen.add(r[0]))]
tot = sum(int(r[i_s]) for r in data if r[i_s].isdigit())
print(f"{col}: total {tot}")
for k, r in sorted(enumerate(data), key=lambda kr: -int(kr[1][i_s]) if kr[1][i_s].isdigit() else 0)[:22]:
    print(f"{k:5d} {r[i_s]:>6} {r[i_src][:90]}")
