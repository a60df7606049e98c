#!/bin/bash
# usage: tools/gpu_runs/bench_multi.sh N [grouping] [extra bench args...]  -> gpurun_out/bench{N}_{grouping}_{transport}.json
N=$1; G=${2:-default}; shift; shift
port=29600
for tr in nccl peer; do
  port=$((port + 1))
  gargs=""; [ "$G" != "default" ] && gargs="--grouping $G"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $N --transport $tr $gargs "$@" \
    > gpurun_out/bench${N}_${G}_${tr}.json 2> gpurun_out/bench${N}_${G}_${tr}.err
  echo "bench N=$N $G $tr rc=$? $(python -c "
import json; d=json.loads(open('gpurun_out/bench${N}_${G}_${tr}.json').readline())
print(d['config']['grouping'], round(d['ms_per_step'],4), round(d['frozen_ms_per_step'],4), round(d['value']), {k: v['us'] for k, v in d['kernels'].items()})" 2>&1 | tail -1)"
done
