"""Per-step device times of the bench's dynamic step (graph replay, L2 flushed), to see
the spread. Usage (GPU box): python tools/step_times.py [steps] [sampler 0|1]"""
import os
import subprocess
import sys
import threading

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_14628_b200 as H  # noqa: E402
from paper_2512_14628_b200.synthetic import (channel_keep_constraints, model_layers, synthetic_base,  # noqa: E402
                                             synthetic_rank_state)

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
sampler = len(sys.argv) > 2 and sys.argv[2] == "1"
torch.cuda.set_device(0)
layers = model_layers("rn18_224")
names = [ls.name for ls in layers]
cluster = H.LocalCluster(H.Topology(1, 1))
sched = H.PenaltySchedule.uniform(names, 1.5e-3, 1.5e-4, adapt=False)
settings = H.ConsensusSettings(t_freeze=10**9, drift_window=0, weight_decay=1e-4)
eng = H.HSADMMSync(0, cluster, layers, channel_keep_constraints(layers, 0.4), sched, settings, residuals=False)
eng.load(**synthetic_rank_state(layers, 0, 1, 0, synthetic_base(layers, 0)))
eng.defer_host = True
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
stop = threading.Event()


def smi():
    while not stop.is_set():
        subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader"], capture_output=True)
        stop.wait(0.2)


if sampler:
    threading.Thread(target=smi, daemon=True).start()
for k in range(1, 6):
    eng.graph_step(k)
torch.cuda.synchronize()
import time  # noqa: E402

evs, host = [], []
for i in range(steps):
    flush.fill_(float(i))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    t0 = time.perf_counter()
    eng.graph_step(6 + i)
    host.append((time.perf_counter() - t0) * 1e3)
    e.record()
    evs.append((s, e))
torch.cuda.synchronize()
print(f"host ms per graph_step: mean {sum(host) / len(host):.4f} min {min(host):.4f} max {max(host):.4f}")
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for i in range(20):
    flush.fill_(float(i))
    eng.graph_step(100 + i)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
stop.set()
t = [a.elapsed_time(b) for a, b in evs]
print(f"sampler={sampler} mean {sum(t) / len(t):.4f} min {min(t):.4f} max {max(t):.4f}")
print(" ".join(f"{x:.3f}" for x in t))
