"""One process, two GPUs: K1 (peer mode) on cuda:0 reading the second rank's send
buffer from cuda:1 over NVLink (peer access enabled), so ncu can profile it
(a multi-rank job must not run under ncu). python tools/k1_remote_1proc.py [model]"""
import ctypes as C
import glob
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2512_14628_b200.synthetic import channel_keep_constraints, model_layers  # noqa: E402
from paper_2512_14628_b200.sparsity import resolve_plan  # noqa: E402
from paper_2512_14628_b200.plan import Plan  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "rn50_224"
torch.cuda.set_device(0)
torch.empty(1, device="cuda:1")   # context on device 1
rt = C.CDLL(sorted(glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) +
                   glob.glob("/usr/local/cuda/lib64/libcudart.so*"))[0])
for d, peer in ((0, 1), (1, 0)):
    rt.cudaSetDevice(d)
    print("enable peer", d, "->", peer, rt.cudaDeviceEnablePeerAccess(peer, 0))
rt.cudaSetDevice(0)
torch.cuda.set_device(0)
layers = model_layers(model)
cons = channel_keep_constraints(layers, 0.4)
groups = {ls.name: resolve_plan(ls.shape, cons[ls.name]) for ls in layers if cons.get(ls.name)}
pl = Plan(layers, groups, {ls.name: 1.5e-3 for ls in layers}, {ls.name: 1.5e-4 for ls in layers})
pl.set_penalties(None, None, 1e-4, 1, 2)
s0, z, v = (torch.randn(pl.arena, device="cuda:0") for _ in range(3))
s1 = torch.randn(pl.arena, device="cuda:1")
zn = torch.empty(pl.arena, device="cuda:0")
flush = torch.empty(256 << 18, device="cuda:0")
ts = []
for i in range(23):
    flush.fill_(1.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    pl.candidate_peers([s0.data_ptr(), s1.data_ptr()], z, v, zn)
    b.record()
    ts.append((a, b))
torch.cuda.synchronize()
t = sorted(x.elapsed_time(y) for x, y in ts[3:])[10] * 1e3
print(f"{model} K1 peer, remote send on cuda:1 (one direction loaded): {t:.1f} us, "
      f"{4 * pl.arena / t / 1e3:.1f} GB/s remote", flush=True)
