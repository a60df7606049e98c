"""Drive tools/nvl_micro.cu on 2 GPUs (torchrun): every rank streams its peer's
symmetric buffer into a local one, all at once; prints GB/s per variant (rank 0).

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -o tools/libnvl_micro.so tools/nvl_micro.cu
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/nvl_micro.py
"""
import ctypes as C
import json
import os
import sys

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

ROOT = os.path.dirname(os.path.abspath(__file__))


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    lib = C.CDLL(os.path.join(ROOT, "libnvl_micro.so"))
    ld, rows = 4608, 13824
    n = ld * rows
    buf = symm.empty(n, dtype=torch.float32, device=dev)
    buf.copy_(torch.arange(n, device=dev, dtype=torch.float32))
    h = symm.rendezvous(buf, dist.group.WORLD)
    peer = h.buffer_ptrs[rank ^ 1]
    out = torch.empty(n, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    nbytes = n * 4
    res = {}

    def timed(name, fn, iters=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / iters / 1e3], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[name] = round(nbytes / float(t.item()) / 1e9, 1)
        # correctness: the peer's buffer holds arange
        want = torch.arange(1024, device=dev, dtype=torch.float32) + (3 if name.startswith("mix") else 0)
        assert torch.equal(out[:1024], want) or name.startswith("torch"), name

    peer_t = h.get_buffer(rank ^ 1, (n,), torch.float32)
    timed("torch_copy", lambda: out.copy_(peer_t))
    for g in (148 * 4, 148 * 8, 148 * 16):
        timed(f"v4_grid{g}", lambda g=g: lib.nvl_copy_v4(C.c_void_p(peer), C.c_void_p(out.data_ptr()), C.c_longlong(nbytes), g, C.c_void_p(stream)))
    for g in (148 * 2, 148 * 3, 148 * 4):
        timed(f"ring_tile_grid{g}", lambda g=g: lib.nvl_copy_ring(C.c_void_p(peer), C.c_void_p(out.data_ptr()), rows, ld, g, C.c_void_p(stream)))
    stages = nbytes // 16384
    for g in (148, 148 * 2, 148 * 3):
        timed(f"bulk_contig_grid{g}", lambda g=g: lib.nvl_copy_bulk(C.c_void_p(peer), C.c_void_p(out.data_ptr()), C.c_longlong(stages), 0, ld, g, C.c_void_p(stream)))
        timed(f"bulk_rows_grid{g}", lambda g=g: lib.nvl_copy_bulk(C.c_void_p(peer), C.c_void_p(out.data_ptr()), C.c_longlong(stages), 1, ld, g, C.c_void_p(stream)))
    # K1-like mix: remote + 3 local streams -> 1 local stream
    la, lb, lc = (torch.ones(n, device=dev) for _ in range(3))
    for mode in (0, 1):
        for g in (148 * 2, 148 * 3):
            timed(f"mix_mode{mode}_grid{g}", lambda g=g, mode=mode: lib.nvl_mix(
                C.c_void_p(peer), C.c_void_p(la.data_ptr()), C.c_void_p(lb.data_ptr()), C.c_void_p(lc.data_ptr()),
                C.c_void_p(out.data_ptr()), rows, ld, g, mode, C.c_void_p(stream)))
    # the same kernels on local memory (HBM) for reference
    loc = buf.data_ptr()
    timed("local_v4_grid1184", lambda: lib.nvl_copy_v4(C.c_void_p(loc), C.c_void_p(out.data_ptr()), C.c_longlong(nbytes), 1184, C.c_void_p(stream)))
    timed("local_ring_tile_grid444", lambda: lib.nvl_copy_ring(C.c_void_p(loc), C.c_void_p(out.data_ptr()), rows, ld, 444, C.c_void_p(stream)))
    timed("local_bulk_rows_grid444", lambda: lib.nvl_copy_bulk(C.c_void_p(loc), C.c_void_p(out.data_ptr()), C.c_longlong(stages), 1, ld, 444, C.c_void_p(stream)))
    if rank == 0:
        print(json.dumps({"bytes": nbytes, "GBps_read_each_rank_all_at_once": res}, indent=1), flush=True)
        if len(sys.argv) > 1:
            open(sys.argv[1], "w").write(json.dumps(res, indent=1))
    h.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
