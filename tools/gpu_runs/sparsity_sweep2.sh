#!/bin/bash
# configs[4] at 2 GPUs, 2x1 (two leaders): the compaction K6 runs on its own, the leader
# all-reduce moves the compact buffer -> gpurun_out/sweep2_<model>_<transport>.jsonl
model=${1:-rn50_224}; tr=${2:-nccl}
out=gpurun_out/sweep2_${model}_${tr}.jsonl
: > $out
for keep in 1.0 0.9 0.8 0.7 0.6 0.5 0.4 0.3 0.2 0.1; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701 \
    bench.py --gpus 2 --grouping 2x1 --transport $tr --model $model --keep $keep --no-cpu-baseline --steps 10 --warmup 3 >> $out 2>/dev/null
  echo "keep=$keep rc=$?"
done
python - $out <<'PY'
import json, sys
for line in open(sys.argv[1]):
    d = json.loads(line)
    k6 = d["kernels"].get("K6_compact_dual", {})
    c = d.get("collectives", {})
    zs = c.get("K8_leader_avg") or c.get("C:z_sync") or {}
    bw = zs.get("busbw_gbs", zs.get("nvlink_gbs"))
    print(f"keep {d['config']['keep_rate']:.1f}: dyn {d['ms_per_step']:.3f} ms frozen {d['frozen_ms_per_step']:.3f} ms "
          f"K6 {k6.get('us')} us {k6.get('gbs')} GB/s ({k6.get('frac')}) leader {d['leader_bytes']['z_sync_bytes']/1e6:.1f} MB "
          f"({d['leader_bytes']['ratio_vs_dense']:.3f} of dense) leader avg {zs.get('us')} us {bw} GB/s")
PY
