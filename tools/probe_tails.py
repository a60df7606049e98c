"""Back-to-back launch timing of the latency-bound kernels (K2 select, K5 keep
sets, fused K3+K5) per launch and per layer, free of host submission gaps.

    HSX_FUSE_SELECT=0 python tools/probe_tails.py [model]
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2512_14628_b200 as H  # noqa: E402
from paper_2512_14628_b200.synthetic import channel_keep_constraints, model_layers, synthetic_rank_state  # noqa: E402

REPS = 50


def bench(fn, reps=REPS):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3  # us


def engine(layers, keep=0.4):
    topo = H.Topology.parse("1x1")
    cons = channel_keep_constraints(layers, keep)
    sched = H.PenaltySchedule.uniform([ls.name for ls in layers], 1.5e-3, 1.5e-4, adapt=False)
    settings = H.ConsensusSettings(t_freeze=10**9, drift_window=0, weight_decay=1e-4)
    eng = H.HSADMMSync(0, H.LocalCluster(topo), layers, cons, sched, settings)
    eng.load(**synthetic_rank_state(layers, 0, 1, 0))
    H.run_local([eng], 1)
    torch.cuda.synchronize()
    return eng


def probe(eng, label):
    pl = eng.plan
    out = {}
    out["K1"] = bench(lambda: pl.candidate(None, eng.theta, eng.u, eng.z, eng.v, eng.z_node))
    out["K2"] = bench(lambda: pl.select(0))
    out["K3"] = bench(lambda: pl.project(eng.z_node, eng.local_mask))
    out["K5"] = bench(lambda: pl.keep_sets(eng.union, eng.masks))
    out["K3+K5"] = bench(lambda: pl.project_keep_sets(eng.z_node, eng.union, eng.masks))
    out["K6"] = bench(lambda: pl.compact_dual(eng.theta, eng.u, eng.z_node, eng.v, eng.flat))
    out["K7"] = bench(lambda: pl.decompact_dual(eng.flat, 1.0, eng.z_node, eng.v, eng.z))
    print(f"{label:40s} " + " ".join(f"{k}={v:7.2f}" for k, v in out.items()), flush=True)


def main():
    model = sys.argv[1] if len(sys.argv) > 1 else "rn18_224"
    torch.cuda.set_device(0)
    layers = model_layers(model)
    probe(engine(layers), f"{model} all layers")
    seen = set()
    for ls in layers:
        if ls.kind is not H.LayerKind.CONV or ls.shape in seen:
            continue
        seen.add(ls.shape)
        probe(engine([ls]), f"{ls.name} {ls.shape}")


if __name__ == "__main__":
    main()
