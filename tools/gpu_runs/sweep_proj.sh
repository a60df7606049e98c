#!/bin/bash
# K3 projection tile-height sweep (HSX_PROJ_TILE_ROWS); one line per (model, rows)
for m in rn18_224 rn50_224; do for t in 16 32 64 128; do
  echo "$m proj_rows=$t $(HSX_PROJ_TILE_ROWS=$t timeout 180 python bench.py --model $m --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(round(d["ms_per_step"],4), {k: (v["us"], v.get("frac")) for k, v in d["kernels"].items()})')"
done; done
