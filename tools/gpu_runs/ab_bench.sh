#!/bin/bash
# A/B of bench.py under env settings: tools/gpu_runs/ab_bench.sh "NAME=ENV ..." ...
# prints ms/step, frozen ms/step and per-kernel us for each setting
for cfg in "$@"; do
  env $cfg python bench.py --no-cpu-baseline --steps ${AB_STEPS:-40} > gpurun_out/ab.json 2>/dev/null
  python - "$cfg" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
print(f"{sys.argv[1]:30s} dyn {d['ms_per_step']:.4f} p50 {d['step_ms_spread']['p50']:.4f} min {d['step_ms_spread']['min']:.4f} frozen {d['frozen_ms_per_step']:.4f} e2e {d['e2e']['ms_per_step']:.3f}",
      {k: round(v["us"], 1) for k, v in d["kernels"].items()})
PY
done
