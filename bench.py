"""Benchmark of the H-SADMM synchronization step on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--model rn18_224] [--grouping MxP] [--keep 0.4]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

A step is one full dynamic H-SADMM sync iteration (SURVEY.md §3.2 phases 2-5u:
intra all-reduce, candidate + fp64 group norms, top-k projection + masks,
leader mask union, keep sets + one D2H, compaction fused with the intra dual,
leader all-reduce of the compact buffer, broadcast, decompaction fused with
the inter dual) on synthetic ResNet-shaped state resident in HBM. Default
workload: BASELINE.json configs[1] — ResNet-18 224x224 shapes, 60% channel
sparsity (keep 0.4), 1 B200. Groupings by N: 1x1, 1x2, 2x2, 2x4 (override
with --grouping). Each rank holds a full replica: weak scaling.

value = synced parameters x ranks / step time (Mparams/s); ms_per_step is
the device time per step (CUDA events on the launching stream, max over
ranks, L2 flushed between steps). ``--impl reference`` times the CPU oracle
(oracle/hsadmm_oracle.py, the fp64 restatement of the reference's numpy
path) on this host on the same workload.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "H-SADMM sync step ms & HBM GB/s (frac of roofline) at 1/2/4/8 B200; leader bytes"
UNIT = "Mparams/s"
DEFAULT_GROUPING = {1: "1x1", 2: "1x2", 4: "2x2", 8: "2x4"}
PRESLEEP_CYCLES = int(float(os.environ.get("HSX_BENCH_PRESLEEP_MS", "1")) * 2e6)   # ~ms at ~2 GHz
FALLBACK_HBM_GBS = 6650.0


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--model", default="rn18_224")
    ap.add_argument("--grouping", default=None)
    ap.add_argument("--keep", type=float, default=0.4)
    ap.add_argument("--transport", choices=["auto", "peer", "nccl"], default="auto")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-graph", action="store_true", help="one rank: launch eagerly instead of replaying CUDA graphs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--ref-budget-s", type=float, default=150.0)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def topology_for(n, grouping):
    from paper_2512_14628_b200.transport import Topology

    g = grouping or DEFAULT_GROUPING.get(n, f"{n}x1")
    topo = Topology.parse(g)
    if topo.world_size != n:
        raise SystemExit(f"grouping {g} needs {topo.world_size} ranks, have {n}")
    return topo


def workload_config(args, topo, n):
    from paper_2512_14628_b200.synthetic import model_layers

    layers = model_layers(args.model)
    N = sum(ls.elements for ls in layers)
    return layers, N, {
        "workload": f"{args.model} synthetic, H-SADMM sync (dynamic: norm, project, mask union, "
                    f"compact, leader all-reduce, decompact), channel keep {args.keep}, "
                    f"{topo.num_nodes}x{topo.accels_per_node} grouping",
        "model": args.model, "grouping": f"{topo.num_nodes}x{topo.accels_per_node}",
        "keep_rate": args.keep, "params_per_rank": N, "mode": "dynamic",
        "l2": "flushed between timed steps (256 MiB write)", "ranks": n}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


# -- clocks -------------------------------------------------------------------------


class ClockSampler:
    """One background ``nvidia-smi -lms 200`` (the recipe's clocks line) for the
    duration of the block: a single process streaming samples, so the timed loop
    is not disturbed by a fork per sample."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.samples = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                        "-i", ",".join(str(g) for g in self.gpus), "-lms", "200"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self._p = None
        time.sleep(0.3)   # first sample before the timed loop starts
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        time.sleep(0.25)  # a last sample inside the window
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=5)
        except Exception:
            self._p.kill()
            out, _ = self._p.communicate()
        for line in (out or "").strip().splitlines():
            self.samples.append([x.strip() for x in line.split(",")])

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            for name, val in zip(names, s[4:8]):
                if val.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# -- CPU oracle (reference arm and cpu_baseline) -------------------------------------


def oracle_setup(layers, topo, keep, seed, max_elems=None):
    """fp64 oracle states of every simulated rank for (a prefix of) the workload."""
    import numpy as np

    from oracle import hsadmm_oracle as O
    from paper_2512_14628_b200.layers import LayerKind
    from paper_2512_14628_b200.synthetic import synthetic_base, synthetic_rank_state

    sample = layers
    if max_elems is not None:
        sample, tot = [], 0
        for ls in layers:
            if tot and tot + ls.elements > max_elems:
                break
            sample.append(ls)
            tot += ls.elements
    base = synthetic_base(sample, seed)
    cons = {ls.name: [(O.CHANNEL, None, keep)] for ls in sample if ls.kind is LayerKind.CONV}
    olayers = O.make_layers([(ls.name, ls.shape) for ls in sample], cons)
    states, thetas = [], []
    for r in range(topo.world_size):
        st = synthetic_rank_state(sample, r, topo.accels_per_node, seed, base)
        states.append(O.init_rank_state(olayers, st["theta"], st["u"], st["z_node"], st["v"], st["z"]))
        thetas.append({n: a.astype(np.float64) for n, a in st["theta"].items()})
    rho1 = {ls.name: 1.5e-3 for ls in sample}
    rho2 = {ls.name: 1.5e-4 for ls in sample}
    return O, olayers, states, thetas, rho1, rho2, sum(ls.elements for ls in sample)


def oracle_step(ctx, topo, k):
    O, olayers, states, thetas, rho1, rho2, _ = ctx
    O.cluster_sync(olayers, states, thetas, k, topo.num_nodes, topo.accels_per_node, rho1, rho2, 1e-4,
                   t_freeze=10**9, drift_window=0)


def _prefix(layers, max_elems):
    sample, tot = [], 0
    for ls in layers:
        if tot and tot + ls.elements > max_elems:
            break
        sample.append(ls)
        tot += ls.elements
    return sample


def cpu_baseline(layers, topo, keep, seed, budget_s):
    """Oracle port on this host: dynamic steps of the workload (every simulated rank)
    until ~budget_s; a layer prefix when the whole M x P workload exceeds 60 M
    simulated elements (host memory and time)."""
    N = sum(ls.elements for ls in layers)
    cap = 60_000_000 // topo.world_size
    ctx = oracle_setup(layers, topo, keep, seed, max_elems=cap if N > cap else None)
    times, k = [], 0
    t_end = time.perf_counter() + budget_s
    while True:
        k += 1
        t0 = time.perf_counter()
        oracle_step(ctx, topo, k)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() >= t_end or k >= 30:
            break
    n = ctx[-1] * topo.world_size
    t = statistics.median(times)
    what = "the full workload" if ctx[-1] == N else f"a layer prefix of {ctx[-1]} of {N} params"
    out = {"value": n / t / 1e6, "unit": UNIT, "cores": 1, "kind": "port",
           "sample": f"{len(times)} dynamic sync steps of {what} x {topo.world_size} simulated ranks "
                     f"(oracle port, numpy fp64 single-threaded), median {t * 1e3:.0f} ms/step, "
                     f"host {os.cpu_count()} cpus",
           "ms_per_step": t * 1e3}
    # the reference itself beside the port (its iteration also runs phase 5 and the
    # sha256 digests, which the timed sync step does not: the port is the like-for-like
    # number)
    real = real_reference(layers, topo, keep, seed, steps=3, warmup=1, budget_s=budget_s)
    if real is not None:
        out["reference_real"] = {k: real[k] for k in ("value", "kind", "sample", "ms_per_step")}
    return out


def admmprune_path():
    """baseline/_ref: the unmodified reference package (pip-installed from
    /root/reference into the repo, git-ignored, shipped with the snapshot)."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "admmprune")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import admmprune  # noqa: F401
    except Exception:
        return None
    return path


def real_reference(layers, topo, keep, seed, steps, warmup, budget_s):
    """The reference itself, ``admmprune.run_hierarchical(Cluster(Topology(M, P)), ...)``
    through its public API and stock code path, with only phase 1 replaced (it
    returns each rank's fixed synthetic theta, as SURVEY Appendix C times it); one
    step = one outer iteration of every simulated rank (phases 2-5 incl. the
    reference's residual block and digests), timed between rank 0's successive
    phase-1 calls. A layer prefix keeps (warmup + steps) iterations near
    budget_s. None when baseline/_ref has no admmprune."""
    if admmprune_path() is None:
        return None
    import numpy as np

    import admmprune as A
    from admmprune import consensus as RC
    from paper_2512_14628_b200.layers import LayerKind
    from paper_2512_14628_b200.synthetic import synthetic_base, synthetic_rank_state

    W = topo.world_size
    N = sum(ls.elements for ls in layers)

    def run(sample, iters):
        base = synthetic_base(sample, seed)
        specs = [A.LayerSpec(ls.name, A.LayerKind(ls.kind.value), tuple(ls.shape),
                             prunable=ls.kind is LayerKind.CONV) for ls in sample]
        cons = {ls.name: [A.SparsityConstraint(A.ConstraintKind.CHANNEL_KEEP, keep_rate=keep)]
                for ls in sample if ls.kind is LayerKind.CONV}
        thetas = [{n: a.astype(np.float64) for n, a in
                   synthetic_rank_state(sample, r, topo.accels_per_node, seed, base)["theta"].items()}
                  for r in range(W)]

        class Workload:
            def __init__(self):
                self.layers = specs
                self.shards = [None] * W

            def init_params(self, rng):
                return {n: a.astype(np.float64) for n, a in base.items()}

        stamps = []

        def phase1(wl, shard, th, zn, u, rho1, solver, key):
            if key == 0:
                stamps.append(time.perf_counter())
            return {n: a.copy() for n, a in thetas[key].items()}

        saved = (RC.batch_rng, RC.proximal_sgd)
        RC.batch_rng, RC.proximal_sgd = (lambda s, rank, k: rank), phase1
        try:
            names = [sp.name for sp in specs]
            settings = A.ConsensusSettings(iterations=iters + 1, t_freeze=10**9, drift_window=0,
                                           stop_on_convergence=False, weight_decay=1e-4, seed=seed)
            A.run_hierarchical(A.Cluster(A.Topology(topo.num_nodes, topo.accels_per_node)), Workload(), cons,
                               A.PenaltySchedule.uniform(names, 1.5e-3, 1.5e-4, adapt=False), A.SolverConfig(),
                               settings)
        finally:
            RC.batch_rng, RC.proximal_sgd = saved
        return [b - a for a, b in zip(stamps, stamps[1:])]

    probe = _prefix(layers, 2_000_000)
    t_probe = min(run(probe, 2))
    rate = sum(ls.elements for ls in probe) * W / t_probe            # simulated elements / s
    per_iter = budget_s / (warmup + steps + 1)
    sample = layers if N * W <= rate * per_iter else _prefix(layers, max(1, int(rate * per_iter / W)))
    times = run(sample, warmup + steps)[warmup:]
    n = sum(ls.elements for ls in sample)
    t = sum(times) / len(times)
    what = "the full workload" if n == N else f"a layer prefix of {n} of {N} params"
    return {"value": n * W / t / 1e6, "unit": UNIT, "cores": 1, "kind": "reference", "ms_per_step": t * 1e3,
            "steps": len(times),
            "sample": f"admmprune.run_hierarchical (baseline/_ref, unmodified) on {what} x {W} simulated ranks, "
                      f"phase 1 returning fixed thetas; {len(times)} timed iterations after {warmup} warm-up, "
                      f"mean {t * 1e3:.0f} ms/iteration; numpy fp64, one Python thread (the reference is "
                      f"single-process), host {os.cpu_count()} cpus"}


def run_reference(args):
    world, rank, _ = dist_env()
    n = args.gpus or world
    if rank != 0:
        return
    topo = topology_for(n, args.grouping)
    layers, N, config = workload_config(args, topo, n)
    # the port: size the per-step sample so W + K steps end within ~ref_budget_s
    ctx = oracle_setup(layers, topo, args.keep, args.seed, max_elems=_port_cap(N, topo))
    t0 = time.perf_counter()
    oracle_step(ctx, topo, 1)
    t_full = time.perf_counter() - t0
    steps_total = args.warmup + args.steps
    if t_full * steps_total > args.ref_budget_s:
        frac = args.ref_budget_s / (t_full * steps_total)
        ctx = oracle_setup(layers, topo, args.keep, args.seed, max_elems=max(1, int(ctx[-1] * frac)))
    n_params = ctx[-1]
    for k in range(1, args.warmup + 1):
        oracle_step(ctx, topo, k)
    times = []
    for k in range(args.warmup + 1, steps_total + 1):
        t0 = time.perf_counter()
        oracle_step(ctx, topo, k)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    port_ms = total / len(times) * 1e3
    port_value = n_params * topo.world_size / (total / len(times)) / 1e6
    port_sample = (f"oracle port (oracle/hsadmm_oracle.py, numpy fp64): "
                   f"{'full workload' if n_params == N else f'layer prefix of {n_params} of {N} params'} per "
                   f"simulated rank, {topo.world_size} ranks serialized in one process (reference architecture)")
    port = {"value": port_value, "unit": UNIT, "cores": 1, "kind": "port", "sample": port_sample,
            "ms_per_step": port_ms}
    # the port does exactly the timed step's work (phases 2-4 + the u-update); the
    # unmodified reference's iteration (admmprune from baseline/_ref) also runs phase 5
    # and sha256 digests of the state: reported beside it, not as the line's value
    real = real_reference(layers, topo, args.keep, args.seed, args.steps, args.warmup, args.ref_budget_s)
    value, ms = port["value"], port["ms_per_step"]
    cpu = {k: port[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if real is not None:
        cpu["reference_real"] = {k: real[k] for k in ("value", "kind", "sample", "ms_per_step")}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
            "impl": "reference", "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def _port_cap(N, topo):
    cap = 60_000_000 // topo.world_size
    return cap if N > cap else None


# -- the B200 arm ------------------------------------------------------------------------

# algorithmic HBM bytes per launch; N = synced elements, n_c = conv
# elements, Z = compact payload elements; k3 / k67_extra from projection_bytes
def algorithmic_bytes(kernel, N, n_c, Z, P, k3=None, k67_extra=0):
    k3 = 8 * n_c + n_c // 8 if k3 is None else k3
    return {
        "K0_pack_theta_u": 12 * N,
        "K1_candidate": (16 if P > 1 else 20) * N,     # read S,z,v (or theta,u,z,v), write z_node
        "K3_project": k3,
        "K3_project_keep": k3,
        "K2K3_select_project_keep": k3,
        "K6_compact_dual": 20 * N + 4 * Z,
        "K6f_dual_intra": 16 * N,
        "K7_decompact_dual": 16 * N + 4 * Z,
        # read z_node, v, theta, u; write u, z, v (+ the fused projection's stores)
        "K67_local_sync": 28 * N + k67_extra,
    }.get(kernel)


def projection_bytes(eng, layers):
    """(K3 bytes, K67's extra bytes) per launch: K3 reads and writes every element
    of the prunable layers + n/8 mask bytes."""
    n_p = sum(layers[i].elements for i in eng.plan.prunable)
    return 8 * n_p + n_p // 8, 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2512_14628_b200 as H
    from paper_2512_14628_b200 import _lib, plan as plan_mod
    from paper_2512_14628_b200.synthetic import channel_keep_constraints, synthetic_base, synthetic_rank_state

    world, rank, local = dist_env()
    n = args.gpus or world
    if n != world:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={world}: launch with torchrun --nproc-per-node {n}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    topo = topology_for(n, args.grouping)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        cluster = H.DistCluster(topo)
    else:
        cluster = H.LocalCluster(topo)
    layers, N, config = workload_config(args, topo, n)
    n_c = sum(ls.elements for ls in layers if ls.kind is H.LayerKind.CONV)
    cons = channel_keep_constraints(layers, args.keep)
    names = [ls.name for ls in layers]
    sched = H.PenaltySchedule.uniform(names, 1.5e-3, 1.5e-4, adapt=False)
    settings = H.ConsensusSettings(t_freeze=10**9, drift_window=0, weight_decay=1e-4)
    eng = H.HSADMMSync(rank, cluster, layers, cons, sched, settings, device=dev, transport=args.transport,
                       residuals=False)
    if world > 1:
        config["transport"] = eng.transport
    base = synthetic_base(layers, args.seed)
    st = synthetic_rank_state(layers, rank, topo.accels_per_node, args.seed, base)
    eng.load(**st)
    theta_host = torch.empty(eng.plan.arena, dtype=torch.float32).pin_memory()
    theta_host.copy_(eng.theta.cpu())
    z_host = torch.empty(eng.plan.arena, dtype=torch.float32).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    # L2 flush between timed steps: write 256 MiB (evicts every line of the step's
    # state); "write_read" then reads a second 256 MiB buffer so the write-back of the
    # flush's own dirty lines happens before the timed step, not inside its first kernel
    flush_mode = os.environ.get("HSX_BENCH_FLUSH", "write_read")
    flush2 = torch.empty_like(flush) if flush_mode == "write_read" else None
    sink = torch.empty((), dtype=torch.float32, device=dev)
    if flush2 is not None:
        config["l2"] = "flushed between timed steps (256 MiB write, then 256 MiB read: no dirty lines left)"
    # run the flush kernels once now: their lazily loaded modules would otherwise load
    # in front of the first timed step, leaving the host no launch slack for it
    flush.fill_(0.0)
    if flush2 is not None:
        torch.sum(flush2, dim=0, out=sink)
    torch.cuda._sleep(1000)
    torch.cuda.synchronize()

    use_graph = world == 1 and not args.no_graph
    config["launch"] = "cuda-graph replay per step" if use_graph else "eager launches (deferred host bookkeeping)"

    def run_step(k, eager=False):
        if world > 1:
            return eng.step(k)
        if use_graph and not eager:   # one rank: the step replays a captured CUDA graph
            return eng.graph_step(k)
        return H.run_local([eng], k)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def timed_steps(k0, nsteps, kernel_timer=None):
        """Per-step device times (ms) with an L2 flush between steps."""
        evs = []
        barrier()
        torch.cuda.synchronize()
        # a spin before the first step (outside every event pair): the host enqueues
        # the first steps while it runs, so no step's bracket contains GPU idle time
        # waiting for the host (or another rank) to launch it
        torch.cuda._sleep(PRESLEEP_CYCLES)
        host_t = []
        for i in range(nsteps):
            host_t.append(time.perf_counter())
            flush.fill_(float(i))
            if flush2 is not None:
                torch.sum(flush2, dim=0, out=sink)
            if kernel_timer is not None:
                # per-kernel pass: a ~1 ms spin keeps the GPU busy while the host
                # enqueues the step's launches and their events, so each event pair
                # brackets the kernel's device time, not the host's launch latency
                torch.cuda._sleep(2_000_000)
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            plan_mod.TIMER = kernel_timer
            run_step(k0 + i, eager=kernel_timer is not None)
            plan_mod.TIMER = None
            e.record()
            evs.append((s, e))
        torch.cuda.synchronize()
        barrier()
        if os.environ.get("HSX_BENCH_TRACE"):
            print(f"rank {rank} host enqueue ms:", [round((b - a) * 1e3, 3) for a, b in zip(host_t, host_t[1:])],
                  file=sys.stderr, flush=True)
        return [s.elapsed_time(e) for s, e in evs]

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # deferred host bookkeeping (the product's pipelined mode): a step returns once its
    # launches are queued and its keep-set counts are read back when the next step
    # starts, so the host stays ahead of the GPU
    eng.defer_host = True
    # clocks are sampled from before the warm-up to the end of the headline steps (the
    # sampler's start-up pause is not an idle gap between warm-up and timed steps)
    # rank 0 alone runs the sampler (over every GPU of the job): one NVML poller, not one per rank
    clocks = (ClockSampler([local] if world == 1 else list(range(world)))
              if rank == 0 and not os.environ.get("HSX_BENCH_NO_CLOCKS") else None)
    if clocks is not None:
        clocks.__enter__()
    k = 0
    for _ in range(args.warmup):
        k += 1
        run_step(k)
    torch.cuda.synchronize()
    # headline: dynamic steps
    launches0 = _lib.launch_count()
    gc.disable()   # no collector pauses inside the timed loop
    try:
        times = timed_steps(k + 1, args.steps)
    finally:
        if clocks is not None:
            clocks.__exit__(None, None, None)
    gc.enable()
    launches = _lib.launch_count() - launches0
    k += args.steps
    total_ms = max_over_ranks(sum(times))
    ms = total_ms / args.steps
    step_spread = {"min": min(times), "p50": statistics.median(times), "max": max(times)}
    value = N * world / (ms / 1e3) / 1e6
    Z = eng.payload_elements
    # roofline pass: the same K dynamic steps with CUDA events around every libhsx
    # launch and collective, on the launching stream
    timer = plan_mod.KernelTimer()
    plan_mod.NOTES.clear()
    ktimes = timed_steps(k + 1, args.steps, kernel_timer=timer)
    k += args.steps
    kstep_ms = max_over_ranks(sum(ktimes)) / args.steps
    kdur = timer.durations_ms()
    notes = dict(plan_mod.NOTES)
    plan_mod.NOTES.clear()
    kern = {name: statistics.mean(d) for name, d in kdur.items()}
    launches_per_kernel = {name: len(d) / args.steps for name, d in kdur.items()}
    # frozen steady state (after t_freeze: sealed keep sets, no projection / union)
    eng.frozen = True
    for _ in range(2):
        k += 1
        run_step(k)
    ftimes = timed_steps(k + 1, args.steps)
    k += args.steps
    frozen_ms = max_over_ranks(sum(ftimes)) / args.steps
    eng.frozen = False
    # back-to-back steady state: the same dynamic steps with no L2 flush in between,
    # one event pair around all K (each step's trailing write-back lands in the next)
    for _ in range(2):
        k += 1
        run_step(k)
    barrier()
    torch.cuda.synchronize()
    bs, be = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(2_000_000)
    bs.record()
    for i in range(args.steps):
        run_step(k + 1 + i)
    be.record()
    torch.cuda.synchronize()
    barrier()
    k += args.steps
    steady_ms = max_over_ranks(bs.elapsed_time(be)) / args.steps
    # the full Algorithm-1 iteration: the dynamic step + phase 5 (residual sums fused
    # into K6/K7, report, adaptive penalties, dual rescale), as the reference runs it
    eng.set_residuals(True, adapt=True)
    for _ in range(2):
        k += 1
        run_step(k)
    rtimes = timed_steps(k + 1, args.steps)
    k += args.steps
    resid_ms = max_over_ranks(sum(rtimes)) / args.steps
    eng.set_residuals(False)
    eng.settle()
    eng.defer_host = False
    # e2e through the public API with host buffers: HSADMMSync.step_host copies every
    # step's theta in from pinned host memory on a copy stream (double-buffered, so
    # step k+1's input copy overlaps step k) and the step's result to the host: the
    # per-layer keep-set summary (kept channels, payload sizes = leader bytes, drift;
    # the step's own D2H, which the host's freeze / ledger bookkeeping reads) — and,
    # in the second pass, the whole new consensus z (4N bytes) as well
    def e2e_pass(k0, z_out):
        for i in range(2):
            eng.step_host(k0 + i, theta_host, z_out)
        torch.cuda.synchronize()
        eng.settle()
        barrier()
        torch.cuda.synchronize()
        es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        es.record()
        for i in range(args.steps):
            done = eng.step_host(k0 + 2 + i, theta_host, z_out)
        torch.cuda.current_stream().wait_event(done)
        ee.record()
        torch.cuda.synchronize()
        eng.settle()
        barrier()
        return max_over_ranks(es.elapsed_time(ee)) / args.steps

    e2e_ms = e2e_pass(k + 1, None)
    k += args.steps + 2
    e2e_z_ms = e2e_pass(k + 1, z_host)
    k += args.steps + 2
    summary_bytes = int(eng.plan.summary_host.numel()) * 8
    eng.check_barriers()
    nvlink = nvlink_peaks(world, dev) if world > 1 else None
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    hbm, hbm_src = peaks()
    k3b, k67x = projection_bytes(eng, layers)
    ab_of = lambda kname: algorithmic_bytes(kname, N, n_c, Z, topo.accels_per_node, k3b, k67x)
    cands = {kname: t for kname, t in kern.items() if ab_of(kname)}
    top = max(cands, key=cands.get)
    abytes = ab_of(top)
    achieved = abytes / (kern[top] / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.model, {}).get(top)
        except Exception:
            traffic = None
    kernels_out = {}
    for kname, t in sorted(kern.items()):
        ab = ab_of(kname)
        kernels_out[kname] = {"us": round(t * 1e3, 2), "per_step": launches_per_kernel[kname]}
        if ab:
            kernels_out[kname]["gbs"] = round(ab / (t / 1e3) / 1e9, 1)
            kernels_out[kname]["frac"] = round(ab / (t / 1e3) / 1e9 / hbm, 3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config,
        "roofline": {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "algorithmic_bytes": abytes,
                     "peak_source": hbm_src, "kernel_us": kern[top] * 1e3,
                     "timed_region": "second K-step dynamic pass with per-launch CUDA events "
                                     f"({kstep_ms:.3f} ms/step with events)"},
        "e2e": {"value": N * world / (e2e_ms / 1e3) / 1e6, "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": 4 * eng.plan.arena, "d2h_bytes_per_step": summary_bytes,
                "path": "HSADMMSync.step_host via the C ABI: every step's theta H2D from pinned host memory "
                        "(copy stream, double-buffered) and the step's result D2H — the per-layer keep-set "
                        "summary (kept counts, payload sizes = leader bytes, drift), which the host's freeze "
                        "/ ledger bookkeeping consumes — inside the timed region; K steps timed end to end, "
                        "no L2 flush (6 state arenas > L2)",
                "with_z_readback": {"value": N * world / (e2e_z_ms / 1e3) / 1e6, "ms_per_step": e2e_z_ms,
                                    "d2h_bytes_per_step": summary_bytes + 4 * eng.plan.arena,
                                    "path": "the same, plus the whole new consensus z copied to pinned host "
                                            "memory every step"}},
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / args.steps,
        "clocks": clocks.summary() if clocks is not None else {"sm_mhz": None, "reasons": ["not sampled (HSX_BENCH_NO_CLOCKS)"]},
        "step_ms_spread": step_spread,
        "step_ms": [round(t, 4) for t in times],
        "steady_ms_per_step": steady_ms,
        "frozen_ms_per_step": frozen_ms,
        "phase5_ms_per_step": resid_ms,
        "leader_bytes": {"z_sync_bytes": 4 * Z, "dense_bytes": 4 * N, "ratio_vs_dense": Z / N},
        "kernels": kernels_out,
    }
    if world > 1:
        line["collectives"] = collectives_block(kdur, notes, N, Z, topo, eng.transport, nvlink, args.steps)
        line["nvlink_peak"] = nvlink
        dist.destroy_process_group()
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(layers, topo, args.keep, args.seed, args.cpu_budget_s)
    emit(line)


def nvlink_peaks(world, dev):
    """Measured NVLink peaks in this run (all ranks): a copy kernel reading a peer's
    symmetric-memory mapping (rank r reads rank r ^ 1; all ranks at once, so both
    link directions are loaded) and an NCCL all-reduce of 256 MiB on the world
    group (busbw, nccl-tests convention). CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist

    def timed(fn, iters=10):
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
        return float(t.item())

    out = {}
    n = 64 * 1024 * 1024 // 4
    try:
        import torch.distributed._symmetric_memory as symm

        buf = symm.empty(n, dtype=torch.float32, device=dev)
        buf.fill_(1.0)
        h = symm.rendezvous(buf, dist.group.WORLD)
        peer = h.get_buffer(dist.get_rank() ^ 1 if dist.get_rank() ^ 1 < world else 0, (n,), torch.float32)
        local = torch.empty(n, device=dev)
        t = timed(lambda: local.copy_(peer))
        out["peer_read_gbs"] = 4 * n / t / 1e9
        out["peer_read"] = "copy kernel loading a peer's 64 MiB symmetric buffer, every rank at once"
        h.barrier()
        del peer, buf
    except Exception as exc:  # noqa: BLE001
        out["peer_read_error"] = repr(exc)[:200]
    x = torch.ones(4 * n, device=dev)
    t = timed(lambda: dist.all_reduce(x))
    out["nccl_allreduce_256MiB_busbw_gbs"] = 16 * n / t / 1e9 * 2 * (world - 1) / world
    out["spec_gbs_per_direction"] = 900.0
    return out


def collectives_block(kdur, notes, N, Z, topo, transport, nvlink, steps):
    """Per collective of the step: time per call, bytes, algbw and busbw in nccl-tests
    convention (all-reduce 2(g-1)/g, all-gather (g-1)/g of the gathered size,
    broadcast 1); for the fused NVLink kernels of the peer transport the remote bytes
    they read and that rate against the measured peer-read peak."""
    import statistics as st

    M, P = topo.num_nodes, topo.accels_per_node
    peak = (nvlink or {}).get("peer_read_gbs")
    out = {}
    for name, calls in notes.items():
        ts = kdur.get(name, [])
        if not ts:
            continue
        op, nbytes, g = calls[0]
        per_call = st.mean(ts) / 1e3
        total_b = sum(c[1] for c in calls) / len(calls)    # mean bytes per call
        row = {"op": op, "ranks": g, "us": round(per_call * 1e6, 2), "calls_per_step": len(ts) / steps}
        if op != "barrier" and nbytes:
            alg = total_b / per_call / 1e9
            factor = {"broadcast": 1.0, "all_gather": (g - 1) / g}.get(op, 2 * (g - 1) / g)
            row.update(bytes=int(total_b), algbw_gbs=round(alg, 1), busbw_gbs=round(alg * factor, 1))
            if peak:
                row["busbw_frac_of_peer_peak"] = round(alg * factor / peak, 3)
        out[name] = row
    remote = {}
    if transport == "peer":
        if P == 2:
            remote["K1_candidate"] = 4 * N * (P - 1)
        if P > 2:
            remote["K8_intra_rs"] = remote["K8_intra_ag"] = 4 * N * (P - 1) // P
        if M == 2:
            remote["K8_leader_avg"] = 4 * Z * (M - 1)
        if M > 2:
            remote["K8_leader_rs"] = remote["K8_leader_ag"] = 4 * Z * (M - 1) // M
        if P > 1:
            remote["K8_zhat_read"] = 4 * Z
    for name, b in remote.items():
        ts = kdur.get(name)
        if not ts:
            continue
        t = st.mean(ts) / 1e3
        row = {"op": "fused NVLink kernel (peer loads)", "remote_bytes": int(b), "us": round(t * 1e6, 2),
               "nvlink_gbs": round(b / t / 1e9, 1)}
        if peak:
            row["frac_of_peer_peak"] = round(b / t / 1e9 / peak, 3)
        out[name] = row
    return out


_OUT_FD = None


def emit(line: dict) -> None:
    """The one JSON line, on the real stdout (everything else was moved to stderr)."""
    os.write(_OUT_FD if _OUT_FD is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    global _OUT_FD
    # NCCL / torch banners print on fd 1 from C code; route fd 1 to stderr and keep
    # the real stdout for the single JSON line
    _OUT_FD = os.dup(1)
    os.dup2(2, 1)
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
