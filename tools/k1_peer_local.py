"""K1 in peer mode with both 'peers' local (one GPU): separates the kernel's own cost
from NVLink. Prints K1 us for sum mode, theta+u mode and peer mode (2 and 4 local
sends) on RN50-224 / RN18-224 (python tools/k1_peer_local.py)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2512_14628_b200 as H  # noqa: E402
from paper_2512_14628_b200.synthetic import channel_keep_constraints, model_layers  # noqa: E402
from paper_2512_14628_b200.sparsity import resolve_plan  # noqa: E402
from paper_2512_14628_b200.plan import Plan  # noqa: E402


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush.fill_(1.0)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        ts.append((s, e))
    torch.cuda.synchronize()
    return sorted(s.elapsed_time(e) for s, e in ts)[iters // 2] * 1e3


flush = torch.empty(256 << 18, device="cuda")
for model in ("rn18_224", "rn50_224"):
    layers = model_layers(model)
    cons = channel_keep_constraints(layers, 0.4)
    groups = {ls.name: resolve_plan(ls.shape, cons[ls.name]) for ls in layers if cons.get(ls.name)}
    rho = {ls.name: 1.5e-3 for ls in layers}
    pl = Plan(layers, groups, rho, {ls.name: 1.5e-4 for ls in layers})
    pl.set_penalties(None, None, 1e-4, 1, 2)
    a = [torch.randn(pl.arena, device="cuda") for _ in range(8)]
    zn = torch.empty(pl.arena, device="cuda")
    r = {}
    r["sum"] = timeit(lambda: pl.candidate(a[0], None, None, a[1], a[2], zn))
    r["theta_u"] = timeit(lambda: pl.candidate(None, a[0], a[3], a[1], a[2], zn))
    r["peers2_local"] = timeit(lambda: pl.candidate_peers([a[0].data_ptr(), a[3].data_ptr()], a[1], a[2], zn))
    r["peers4_local"] = timeit(lambda: pl.candidate_peers([x.data_ptr() for x in (a[0], a[3], a[4], a[5])], a[1], a[2], zn))
    print(model, {k: round(v, 1) for k, v in r.items()}, flush=True)
