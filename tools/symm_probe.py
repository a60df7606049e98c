"""Probe torch symmetric memory on the box: rendezvous on sub-groups, barrier, peer reads."""
import os
import time

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
g_all = dist.new_group(list(range(world)))
t = symm.empty(1 << 20, dtype=torch.float32, device="cuda")
t.fill_(rank + 1)
h = symm.rendezvous(t, g_all)
print(rank, "ptrs", [hex(p) for p in h.buffer_ptrs], "mc", h.multicast_ptr, flush=True)
h.barrier(channel=0)
peer = h.get_buffer((rank + 1) % world, (1 << 20,), torch.float32)
torch.cuda.synchronize()
print(rank, "peer value", float(peer[0]), float(peer[-1]), flush=True)
# barrier latency
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(100):
    h.barrier(channel=0)
e.record()
torch.cuda.synchronize()
print(rank, "barrier us", s.elapsed_time(e) * 10, flush=True)
# peer copy bandwidth
n = 1 << 26
a = symm.empty(n, dtype=torch.float32, device="cuda")
ha = symm.rendezvous(a, g_all)
a.fill_(rank)
ha.barrier()
src = ha.get_buffer((rank + 1) % world, (n,), torch.float32)
dst = torch.empty(n, device="cuda")
torch.cuda.synchronize()
s.record()
for _ in range(10):
    dst.copy_(src)
e.record()
torch.cuda.synchronize()
print(rank, "peer read GB/s", 10 * 4 * n / (s.elapsed_time(e) / 1e3) / 1e9, flush=True)
dist.barrier()
dist.destroy_process_group()
