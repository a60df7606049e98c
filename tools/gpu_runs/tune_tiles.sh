#!/bin/bash
# tuning sweep over quad-tile heights (K1 / stream kernels); one bench line per setting
for c in 32 64 128; do for t in 32 64; do
  echo "cand=$c stream=$t $(HSX_CAND_TILE_ROWS=$c HSX_STREAM_TILE_ROWS=$t timeout 120 python bench.py --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(round(d["ms_per_step"],4), round(d["frozen_ms_per_step"],4), {k: v["us"] for k, v in d["kernels"].items()})')"
done; done
