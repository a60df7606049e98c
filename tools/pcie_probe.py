"""PCIe copy rates of one arena-sized buffer: H2D alone, D2H alone, both at once
(separate streams), and host time per HSADMMSync.step_host call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

n = 11689512
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_in = torch.empty(n, dtype=torch.float32, device="cuda")
d_out = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


gb = 4 * n / 1e9
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = timeit(fn)
    print(f"{name:5s} {ms:.3f} ms  {gb / (ms / 1e3):.1f} GB/s per direction", flush=True)

import paper_2512_14628_b200 as H  # noqa: E402
from paper_2512_14628_b200.synthetic import channel_keep_constraints, model_layers, synthetic_rank_state  # noqa: E402

layers = model_layers("rn18_224")
cons = channel_keep_constraints(layers, 0.4)
sched = H.PenaltySchedule.uniform([ls.name for ls in layers], 1.5e-3, 1.5e-4, adapt=False)
settings = H.ConsensusSettings(t_freeze=10**9, drift_window=0, weight_decay=1e-4)
eng = H.HSADMMSync(0, H.LocalCluster(H.Topology.parse("1x1")), layers, cons, sched, settings)
eng.load(**synthetic_rank_state(layers, 0, 1, 0))
th = eng.theta.cpu().pin_memory()
zh = torch.empty(eng.plan.arena, dtype=torch.float32).pin_memory()
for k in range(1, 4):
    eng.step_host(k, th, zh)
torch.cuda.synchronize()
eng.settle()
host = []
t0 = time.perf_counter()
for k in range(4, 24):
    t1 = time.perf_counter()
    done = eng.step_host(k, th, zh)
    host.append(time.perf_counter() - t1)
done.synchronize()
wall = (time.perf_counter() - t0) / 20 * 1e3
print(f"step_host: wall {wall:.3f} ms/step, host per call {sum(host) / len(host) * 1e3:.3f} ms "
      f"(max {max(host) * 1e3:.3f})", flush=True)
# device-resident steps: host time per call
host = []
for k in range(24, 44):
    t1 = time.perf_counter()
    H.run_local([eng], k)
    host.append(time.perf_counter() - t1)
torch.cuda.synchronize()
print(f"run_local: host per call {sum(host) / len(host) * 1e3:.3f} ms", flush=True)
