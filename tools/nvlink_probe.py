"""NVLink / NCCL bandwidth probe on one B200 box (run under torchrun, N ranks).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/nvlink_probe.py [out.json]

Measures, with CUDA events and the max over ranks:
* NCCL all-reduce (SUM, AVG), all-gather, reduce-scatter, broadcast on the world
  group and on pairs {0,1}, {2,3}, ... — algbw and busbw in nccl-tests convention;
* peer-memory reads and writes through torch symmetric memory (a copy kernel
  that loads from / stores to the peer's mapping), all ranks at once (both link
  directions loaded) and one rank alone;
* one copy-engine peer copy (rank 0 -> rank 1).
The result is the measured NVLink peak the bench's collectives block reports
against.
"""

from __future__ import annotations

import json
import os
import sys

import torch
import torch.distributed as dist

MiB = 1 << 20


def timed(fn, iters=20, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    t = torch.tensor([s.elapsed_time(e) / iters], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()) / 1e3   # seconds


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else None
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    res = {"world": world, "nccl": torch.cuda.nccl.version(), "collectives": [], "peer": []}
    groups = {"world": (None, world)}
    pairs = [dist.new_group([2 * i, 2 * i + 1]) for i in range(world // 2)] if world >= 2 else []
    if world > 2:
        groups["pair"] = (pairs[rank // 2], 2)
    big = torch.ones(256 * MiB // 4, device=dev)
    outbuf = torch.empty(256 * MiB // 4 * world, device=dev)
    for gname, (g, gs) in groups.items():
        for mb in (4, 16, 32, 64, 128, 256):
            n = mb * MiB // 4
            x = big[:n]
            S = mb * MiB
            t = timed(lambda: dist.all_reduce(x, op=dist.ReduceOp.SUM, group=g))
            res["collectives"].append(dict(group=gname, ranks=gs, op="all_reduce_sum", MiB=mb, us=t * 1e6,
                                           algbw=S / t / 1e9, busbw=S / t / 1e9 * 2 * (gs - 1) / gs))
            if mb in (32, 64, 128):
                t = timed(lambda: dist.all_reduce(x, op=dist.ReduceOp.AVG, group=g))
                res["collectives"].append(dict(group=gname, ranks=gs, op="all_reduce_avg", MiB=mb, us=t * 1e6,
                                               algbw=S / t / 1e9, busbw=S / t / 1e9 * 2 * (gs - 1) / gs))
                t = timed(lambda: dist.broadcast(x, src=0 if g is None else 2 * (rank // 2), group=g))
                res["collectives"].append(dict(group=gname, ranks=gs, op="broadcast", MiB=mb, us=t * 1e6,
                                               algbw=S / t / 1e9, busbw=S / t / 1e9))
                per = n // gs
                t = timed(lambda: dist.all_gather_into_tensor(outbuf[:per * gs], x[:per], group=g))
                res["collectives"].append(dict(group=gname, ranks=gs, op="all_gather", MiB=mb, us=t * 1e6,
                                               algbw=S / t / 1e9, busbw=S / t / 1e9 * (gs - 1) / gs))
                t = timed(lambda: dist.reduce_scatter_tensor(outbuf[:per], x[:per * gs], group=g))
                res["collectives"].append(dict(group=gname, ranks=gs, op="reduce_scatter", MiB=mb, us=t * 1e6,
                                               algbw=S / t / 1e9, busbw=S / t / 1e9 * (gs - 1) / gs))
    # peer memory (symmetric memory mappings): copy kernels loading from / storing to the peer
    try:
        import torch.distributed._symmetric_memory as symm

        n = 256 * MiB // 4
        buf = symm.empty(n, dtype=torch.float32, device=dev)
        buf.fill_(1.0)
        h = symm.rendezvous(buf, dist.group.WORLD)
        peer_rank = rank ^ 1 if world > 1 else rank
        peer = h.get_buffer(peer_rank, (n,), torch.float32)
        local = torch.empty(n, device=dev)
        S = n * 4
        t = timed(lambda: local.copy_(peer))
        res["peer"].append(dict(mode="read, all ranks", MiB=256, us=t * 1e6, gbs=S / t / 1e9))
        t = timed(lambda: peer.copy_(local))
        res["peer"].append(dict(mode="write, all ranks", MiB=256, us=t * 1e6, gbs=S / t / 1e9))

        def only0(fn):
            return (lambda: fn()) if rank == 0 else (lambda: None)

        t = timed(only0(lambda: local.copy_(peer)))
        res["peer"].append(dict(mode="read, rank 0 alone", MiB=256, us=t * 1e6, gbs=S / t / 1e9))
        t = timed(only0(lambda: peer.copy_(local)))
        res["peer"].append(dict(mode="write, rank 0 alone", MiB=256, us=t * 1e6, gbs=S / t / 1e9))
        h.barrier()
    except Exception as exc:  # noqa: BLE001
        res["peer_error"] = repr(exc)
    # copy engine (cudaMemcpyPeerAsync), rank 0 -> device 1
    if world > 1:
        try:
            if rank == 0:
                src = torch.ones(256 * MiB // 4, device=dev)
                dst = torch.empty(256 * MiB // 4, device="cuda:1")
            t = timed((lambda: dst.copy_(src, non_blocking=True)) if rank == 0 else (lambda: None))
            res["peer"].append(dict(mode="copy engine 0->1", MiB=256, us=t * 1e6, gbs=256 * MiB / t / 1e9))
        except Exception as exc:  # noqa: BLE001
            res["copy_engine_error"] = repr(exc)
    if rank == 0:
        text = json.dumps(res, indent=1)
        print(text, flush=True)
        if out_path:
            with open(out_path, "w") as fh:
                fh.write(text)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
