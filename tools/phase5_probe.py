"""Per-kernel CUDA-event times of the dynamic step with phase 5 on (RN18-224, 1x1).
Usage (GPU box): python tools/phase5_probe.py [model] [adapt 0|1]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_14628_b200 as H  # noqa: E402
from paper_2512_14628_b200 import plan as plan_mod  # noqa: E402
from paper_2512_14628_b200.synthetic import (channel_keep_constraints, model_layers, synthetic_base,  # noqa: E402
                                             synthetic_rank_state)

model = sys.argv[1] if len(sys.argv) > 1 else "rn18_224"
adapt = (sys.argv[2] != "0") if len(sys.argv) > 2 else True
torch.cuda.set_device(0)
layers = model_layers(model)
names = [ls.name for ls in layers]
cluster = H.LocalCluster(H.Topology(1, 1))
sched = H.PenaltySchedule.uniform(names, 1.5e-3, 1.5e-4, adapt=adapt)
settings = H.ConsensusSettings(t_freeze=10**9, drift_window=0, weight_decay=1e-4)
eng = H.HSADMMSync(0, cluster, layers, channel_keep_constraints(layers, 0.4), sched, settings, residuals=True)
eng.load(**synthetic_rank_state(layers, 0, 1, 0, synthetic_base(layers, 0)))
for k in range(1, 4):
    H.run_local([eng], k)
torch.cuda.synchronize()
timer = plan_mod.KernelTimer()
evs = []
for k in range(4, 14):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    plan_mod.TIMER = timer
    H.run_local([eng], k)
    plan_mod.TIMER = None
    e.record()
    evs.append((s, e))
torch.cuda.synchronize()
print(f"{model} adapt={adapt}: step with events {statistics.mean(a.elapsed_time(b) for a, b in evs):.3f} ms")
for name, d in timer.durations_ms().items():
    print(f"  {name:28s} {statistics.mean(d) * 1e3:8.1f} us  x{len(d) / 10:.0f}")
