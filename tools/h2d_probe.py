"""Concurrent H2D rates of N ranks (torchrun): each rank copies one arena-sized pinned
buffer to its GPU repeatedly, all ranks at once; with HSX_PROBE_AFFINITY=1 the rank
first binds itself to its GPU's CPU set (NVML) so its pinned pages are NUMA-local."""
import os
import sys
import time

import torch
import torch.distributed as dist


def bind_gpu_cpus(dev_index):
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
    words = pynvml.nvmlDeviceGetCpuAffinity(h, 64)
    cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
    os.sched_setaffinity(0, cpus)
    return len(cpus)


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    ncpu = bind_gpu_cpus(local) if os.environ.get("HSX_PROBE_AFFINITY") == "1" else 0
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    n = 11689512
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    h.fill_(1.0)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    reps = 30
    for _ in range(reps):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / reps * 1e3
    out = [None] * world
    dist.all_gather_object(out, (rank, round(ms, 3), round(4 * n / ms / 1e6, 1), ncpu, sorted(os.sched_getaffinity(0))[:2]))
    if rank == 0:
        print(f"world {world} affinity {os.environ.get('HSX_PROBE_AFFINITY', '0')}: {out}", flush=True)


main()
