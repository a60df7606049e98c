#!/bin/bash
# configs[4]: channel-sparsity sweep on ResNet-50 (1 B200): step time, K6 compaction GB/s,
# leader bytes vs dense -> gpurun_out/sweep_rn50.jsonl (one bench line per keep rate)
out=gpurun_out/sweep_${1:-rn50_224}.jsonl
: > $out
for keep in 1.0 0.9 0.8 0.7 0.6 0.5 0.4 0.3 0.2 0.1; do
  timeout 300 python bench.py --model ${1:-rn50_224} --keep $keep --no-cpu-baseline --steps 10 --warmup 3 >> $out 2>/dev/null
  echo "keep=$keep rc=$?"
done
python - $out <<'PY'
import json, sys
for line in open(sys.argv[1]):
    d = json.loads(line)
    kn = "K6_compact_dual" if "K6_compact_dual" in d["kernels"] else "K67_local_sync"  # one node: K6+K7 fused
    k6 = d["kernels"].get(kn, {})
    print(f"keep {d['config']['keep_rate']:.1f}: dyn {d['ms_per_step']:.3f} ms frozen {d['frozen_ms_per_step']:.3f} ms "
          f"{kn} {k6.get('us')} us {k6.get('gbs')} GB/s leader bytes {d['leader_bytes']['z_sync_bytes']/1e6:.1f} MB "
          f"({d['leader_bytes']['ratio_vs_dense']:.3f} of dense)")
PY
