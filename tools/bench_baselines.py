"""Fig. 6-style comparison on B200: one sync step of the hierarchical
H-SADMM engine vs the reference's flat consensus and dense synchronous SGD
(baselines.py), same synthetic ResNet state, same timing rules as bench.py (CUDA
events per step, L2 flushed between steps, max over ranks).

    python tools/bench_baselines.py [--model rn18_224] [--grouping 2x1]            # 1 GPU
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/bench_baselines.py --grouping 2x1

Prints one JSON line per system: dynamic / frozen ms per step and the bytes the
reference ledger books per sync (hierarchical: leaders' compact z_sync; flat: the
dense all-rank SUM; dense: the gradient AVG), per rank.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="rn18_224")
    ap.add_argument("--grouping", default=None)
    ap.add_argument("--keep", type=float, default=0.4)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--transport", default="auto")
    ap.add_argument("--systems", default="hsadmm,flat,dense,topk")
    ap.add_argument("--topk-rate", type=float, default=0.01)
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    import bench
    import paper_2512_14628_b200 as H
    from paper_2512_14628_b200.synthetic import channel_keep_constraints, model_layers, synthetic_base, \
        synthetic_rank_state

    world, rank, local = bench.dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    topo = bench.topology_for(world, args.grouping)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    layers = model_layers(args.model)
    N = sum(ls.elements for ls in layers)
    cons = channel_keep_constraints(layers, args.keep)
    names = [ls.name for ls in layers]
    base = synthetic_base(layers, 0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(run, k0, n):
        evs = []
        barrier()
        torch.cuda.synchronize()
        for i in range(n):
            flush.fill_(float(i))
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            run(k0 + i)
            e.record()
            evs.append((s, e))
        torch.cuda.synchronize()
        barrier()
        ts = sorted(s.elapsed_time(e) for s, e in evs)
        return max_over_ranks(sum(ts) / len(ts)), max_over_ranks(ts[len(ts) // 2])

    for system in args.systems.split(","):
        cluster = H.DistCluster(topo) if world > 1 else H.LocalCluster(topo)
        line = {"system": system, "model": args.model, "n_gpus": world, "params_per_rank": N,
                "keep_rate": args.keep, "steps": args.steps, "warmup": args.warmup,
                "l2": "flushed between timed steps (256 MiB write)"}
        class Solver:
            lr, momentum, weight_decay = 0.05, 0.9, 1e-4

        if system == "topk":
            eng = H.TopKSync(rank, cluster, layers, Solver, args.topk_rate, device=dev)
            eng.init_from(base)
            eng.grad.normal_(0.0, 0.1)
            run = (lambda k: eng.step(k)) if world > 1 else (lambda k: H.run_topk_local([eng], k))
            for k in range(1, args.warmup + 1):
                run(k)
            mean, p50 = timed(run, args.warmup + 1, args.steps)
            line.update(grouping=f"1x{world}", transport="nccl", rate=args.topk_rate, ms_per_step=mean, p50_ms=p50,
                        bytes_per_rank_per_sync=8 * eng.K)
        elif system == "dense":
            eng = H.DenseSync(rank, cluster, layers, Solver, device=dev, transport=args.transport)
            eng.init_from(base)
            eng.grad.normal_(0.0, 0.1)
            run = (lambda k: eng.step(k)) if world > 1 else (lambda k: H.run_dense_local([eng], k))
            for k in range(1, args.warmup + 1):
                run(k)
            mean, p50 = timed(run, args.warmup + 1, args.steps)
            line.update(grouping=f"1x{world}", transport=eng.transport, ms_per_step=mean, p50_ms=p50,
                        bytes_per_rank_per_sync=4 * N)
        else:
            sched = H.PenaltySchedule.uniform(names, 1.5e-3, 1.5e-4, adapt=False)
            for mode in ("dynamic", "frozen"):
                settings = H.ConsensusSettings(t_freeze=(1 if mode == "frozen" else 10**9), drift_window=0,
                                               weight_decay=1e-4)
                cls = H.FlatConsensusSync if system == "flat" else H.HSADMMSync
                eng = cls(rank, cluster, layers, cons, sched, settings, device=dev, transport=args.transport,
                          residuals=False)
                eng.load(**synthetic_rank_state(layers, rank, topo.accels_per_node, 0, base))
                if system == "flat":
                    eng.v.zero_()
                eng.defer_host = True
                run = (lambda k: eng.step(k)) if world > 1 else (lambda k: H.run_local([eng], k))
                for k in range(1, args.warmup + 1):
                    run(k)
                if mode == "frozen":
                    assert eng.frozen
                mean, p50 = timed(run, args.warmup + 1, args.steps)
                eng.settle()
                line[f"{mode}_ms_per_step"] = mean
                line[f"{mode}_p50_ms"] = p50
                line["transport"] = eng.transport
                if mode == "dynamic":
                    if system == "flat":
                        line.update(grouping=f"1x{world}", bytes_per_rank_per_sync=4 * N)
                    else:
                        line.update(grouping=f"{topo.num_nodes}x{topo.accels_per_node}",
                                    leader_bytes_per_sync=4 * eng.payload_elements,
                                    intra_bytes_per_rank_per_sync=4 * N if topo.accels_per_node > 1 else 0)
                del eng
                torch.cuda.synchronize()
                barrier()
        if rank == 0:
            print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
