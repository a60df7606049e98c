#!/bin/bash
# old vs new checkout, 2-rank peer bench
for d in _old .; do
  (cd $d && timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29811 bench.py --gpus 2 --transport peer --no-cpu-baseline > /tmp/on.json 2>/tmp/on.err)
  python -c "
import json; d=json.loads(open('/tmp/on.json').readline())
print('$d', round(d['ms_per_step'],4), round(d['frozen_ms_per_step'],4), {k: round(v['us'],1) for k, v in d['kernels'].items()})" || tail -5 /tmp/on.err
done
