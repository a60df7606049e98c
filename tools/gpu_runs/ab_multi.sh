#!/bin/bash
# tools/gpu_runs/ab_multi.sh N TRANSPORT "ENV=.." ...: multi-rank bench per env setting (peer/nccl)
N=$1; TR=$2; shift; shift
port=29700
for cfg in "$@"; do
  port=$((port + 1))
  env $cfg timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $N --transport $TR --no-cpu-baseline > gpurun_out/abm.json 2> gpurun_out/abm.err
  python - "$cfg" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/abm.json").readline())
    print(f"{sys.argv[1]:34s} {d['config']['grouping']} dyn {d['ms_per_step']:.4f} frozen {d['frozen_ms_per_step']:.4f} e2e {d['e2e']['ms_per_step']:.3f}",
          {k: round(v["us"], 1) for k, v in d["kernels"].items()})
except Exception as e:
    print(sys.argv[1], "failed", e, open("gpurun_out/abm.err").read()[-500:])
PY
done
