#!/bin/bash
# K2 select block size sweep (HSX_SELECT_THREADS); one line per (model, threads)
for m in rn18_224 rn50_224; do for t in 128 256 512 1024; do
  echo "$m select_threads=$t $(HSX_SELECT_THREADS=$t timeout 180 python bench.py --model $m --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.readline()); print(round(d["ms_per_step"],4), {k: (v["us"], v.get("frac")) for k, v in d["kernels"].items()})')"
done; done
