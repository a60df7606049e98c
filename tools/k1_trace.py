"""Timeline of the K1 candidate launch (trace build): per item start / tile-done /
tail-done times and SM. Usage (GPU box): make trace && HSX_LIB_PATH=paper_2512_14628_b200/libhsx_trace.so
python tools/k1_trace.py [model] [keep]"""
import collections
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_14628_b200 as H  # noqa: E402
from paper_2512_14628_b200 import _lib  # noqa: E402
from paper_2512_14628_b200.synthetic import (channel_keep_constraints, model_layers, synthetic_base,  # noqa: E402
                                             synthetic_rank_state)

model = sys.argv[1] if len(sys.argv) > 1 else "rn18_224"
keep = float(sys.argv[2]) if len(sys.argv) > 2 else 0.4
torch.cuda.set_device(0)
layers = model_layers(model)
names = [ls.name for ls in layers]
topo = H.Topology(1, 1)
cluster = H.LocalCluster(topo)
sched = H.PenaltySchedule.uniform(names, 1.5e-3, 1.5e-4, adapt=False)
settings = H.ConsensusSettings(t_freeze=10**9, drift_window=0, weight_decay=1e-4)
eng = H.HSADMMSync(0, cluster, layers, channel_keep_constraints(layers, keep), sched, settings)
eng.load(**synthetic_rank_state(layers, 0, 1, 0, synthetic_base(layers, 0)))
for k in range(1, 6):
    H.run_local([eng], k)
torch.cuda.synchronize()
n = 16384
buf = np.zeros(n * 4, dtype=np.uint64)
lib = _lib.load()
lib.hsx_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
rc = lib.hsx_debug_trace(buf.ctypes.data, n)
assert rc == 0, rc
tr = buf.reshape(n, 4)
used = tr[:, 0] > 0
tr = tr[used].astype(np.int64)
t0 = tr[:, 0].min()
start, tile, end = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3
sm = tr[:, 3] & 0xFFFF
lay = tr[:, 3] >> 16
print(f"{model}: {len(tr)} items, span {end.max():.1f} us; last tile done {tile.max():.1f} us")
tail = end - np.maximum(tile, start)
dur = tile - start
print(f"item tile time us: mean {dur.mean():.1f} p50 {np.median(dur):.1f} max {dur.max():.1f}")
big = tail > 0.5
print(f"tails (>0.5us): {big.sum()} items, mean {tail[big].mean() if big.any() else 0:.1f} us, "
      f"max {tail.max():.1f} us")
busy = collections.defaultdict(float)
for s, e, m in zip(start, end, sm):
    busy[m] += e - s
b = np.array(list(busy.values()))
print(f"SMs used {len(b)}; per-SM busy CTA-us mean {b.mean():.1f} min {b.min():.1f} max {b.max():.1f}")
# concurrency over time (CTAs in flight), 20 buckets
edges = np.linspace(0, end.max(), 21)
conc = [int(((start < hi) & (end > lo)).sum()) for lo, hi in zip(edges[:-1], edges[1:])]
print("CTAs in flight per 5% of span:", conc)
per_layer = collections.defaultdict(list)
for l, s, t, e in zip(lay, start, tile, end):
    per_layer[int(l)].append((s, t, e))
print("layer  items  first_start  last_tile  tail_end  (us)  name")
for l in sorted(per_layer):
    v = np.array(per_layer[l])
    print(f"{l:5d} {len(v):6d} {v[:, 0].min():11.1f} {v[:, 1].max():10.1f} {v[:, 2].max():9.1f}  {names[l]}")
