#!/bin/bash
# usage: tools/gpu_runs/bench_models.sh N GROUPING MODEL [transport=peer] -> gpurun_out/bench{N}_{MODEL}_{GROUPING}_{transport}.json
N=$1; G=$2; M=$3; TR=${4:-peer}
port=$((29700 + RANDOM % 200))
out=gpurun_out/bench${N}_${M}_${G}_${TR}.json
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port $port bench.py --gpus $N --grouping $G --model $M --transport $TR --steps 10 --warmup 3 \
  > $out 2> ${out%.json}.err
echo "bench N=$N $M $G $TR rc=$? $(python -c "
import json; d=json.loads(open('$out').readline())
print(round(d['ms_per_step'],4), round(d['frozen_ms_per_step'],4), round(d['value']), round(d['leader_bytes']['ratio_vs_dense'],3))" 2>&1 | tail -1)"
