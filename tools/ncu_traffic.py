"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the libhsx
kernels in an ncu --set full report -> profiles/ncu_traffic.json[model][bench kernel name]
(bench.py puts the dominant kernel's figure in roofline.traffic).

    python tools/ncu_traffic.py REPORT.ncu-rep [model=rn18_224]
"""
import csv
import json
import os
import subprocess
import sys

NAMES = {"k_candidate": "K1_candidate", "k_project": "K3_project", "k_compact": "K6_compact_dual",
         "k_decompact": "K7_decompact_dual", "k_dual": "K6f_dual_intra", "k_add": "K0_pack_theta_u",
         "k_select": "K2_select", "k_keep_fixup": "K5_keep_fixup", "k_keep_sets": "K5_keep_sets",
         "k_local_sync": "K67_local_sync"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

rep = sys.argv[1]
model = sys.argv[2] if len(sys.argv) > 2 else "rn18_224"
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
seen = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    base = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").replace("hsx::", "").strip()
    name = NAMES.get(base)
    if name is None or name in seen:
        continue
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(m)
        tot += float(d[m].replace(",", "")) * SCALE.get(units[i], 1)
    seen[name] = int(tot)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
db = json.load(open(path)) if os.path.exists(path) else {}
db.setdefault(model, {}).update(seen)
db.setdefault("_source", {})[model] = os.path.basename(rep)
json.dump(db, open(path, "w"), indent=1, sort_keys=True)
print(json.dumps(seen, indent=1))
