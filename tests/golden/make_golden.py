"""Generate golden vectors by running the REAL reference (admmprune 0.1.0).

Run in the build container (the reference is mounted read-only at
/root/reference; it does not exist on the GPU box):

    python tests/golden/make_golden.py

Writes small ``.npz`` / ``.json`` fixtures next to this file. They pin the CPU
oracle (oracle/hsadmm_oracle.py, tests/test_oracle.py) and the GPU path
(tests/test_gpu_*.py). Inputs are fp32-representable so the fp32 CUDA path and
the fp64 reference see identical values.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)

import admmprune.consensus as ref_consensus  # noqa: E402
from admmprune.consensus import ConsensusSettings, PenaltySchedule, node_candidate, run_hierarchical  # noqa: E402
from admmprune.shrinkage import compress, decompress, derive_keep_sets  # noqa: E402
from admmprune.sparsity import ConstraintKind, SparsityConstraint, extract_mask, project, project_composite  # noqa: E402
from admmprune.tensors import GroupBy, LayerKind, LayerSpec, group_norms  # noqa: E402
from admmprune.transport import Cluster, Topology, bucketize  # noqa: E402
from admmprune.workloads import SolverConfig  # noqa: E402

KINDS = {"filter": ConstraintKind.FILTER_KEEP, "channel": ConstraintKind.CHANNEL_KEEP,
         "shape": ConstraintKind.SHAPE_KEEP}
GROUPS = {"filter": GroupBy.FILTER, "channel": GroupBy.CHANNEL, "shape": GroupBy.SHAPE_POSITION}


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def gen_projection():
    """Single-constraint and composite projections incl. exact ties and zeros."""
    rng = np.random.default_rng(1234)
    out = {}
    shapes = [(4, 3, 1, 2), (6, 5, 3, 3), (8, 16, 1, 1), (5, 3, 7, 7), (16, 8, 3, 3)]
    idx = 0
    for shape in shapes:
        for kind in KINDS:
            g = {"filter": shape[0], "channel": shape[1]}.get(kind, int(np.prod(shape[1:])))
            for keep in sorted({1, max(1, g // 3), max(1, g // 2), g}):
                for variant in ("normal", "ties", "zeros"):
                    t = f32(rng.normal(size=shape))
                    if variant == "ties":     # duplicate a group so norms tie exactly
                        if kind == "filter" and shape[0] > 1:
                            t[shape[0] - 1] = t[0]
                        elif kind == "channel" and shape[1] > 1:
                            t[:, shape[1] - 1] = t[:, 0]
                        elif kind == "shape":
                            flat = t.reshape(shape[0], -1)
                            flat[:, -1] = flat[:, 0]
                    if variant == "zeros":    # exact zeros inside groups, one all-zero group
                        t[rng.random(shape) < 0.2] = 0.0
                        if kind == "channel":
                            t[:, 0] = 0.0
                    c = SparsityConstraint(KINDS[kind], keep_count=keep)
                    z = project(t, c)
                    out[f"c{idx}_in"] = t
                    out[f"c{idx}_meta"] = np.array([list(KINDS).index(kind), keep])
                    out[f"c{idx}_norms"] = group_norms(t, GROUPS[kind])
                    out[f"c{idx}_out"] = z
                    out[f"c{idx}_mask"] = extract_mask(z)
                    idx += 1
    # composite projections (sequential, listed order)
    comp = [[("filter", 0.5), ("channel", 0.5)], [("channel", 0.5), ("filter", 0.5)],
            [("channel", 0.4), ("shape", 0.5)], [("filter", 0.75), ("channel", 0.4), ("shape", 0.6)]]
    cidx = 0
    for shape in [(8, 6, 3, 3), (16, 12, 1, 1), (6, 4, 3, 3)]:
        for plan in comp:
            t = f32(rng.normal(size=shape))
            cons = [SparsityConstraint(KINDS[k], keep_rate=r) for k, r in plan]
            z = project_composite(t, cons)
            out[f"p{cidx}_in"] = t
            out[f"p{cidx}_plan"] = np.array([[list(KINDS).index(k), c.resolve(
                {"filter": shape[0], "channel": shape[1]}.get(k, int(np.prod(shape[1:]))))]
                for (k, _), c in zip(plan, cons)])
            out[f"p{cidx}_out"] = z
            cidx += 1
    out["n_single"] = np.array(idx)
    out["n_composite"] = np.array(cidx)
    np.savez_compressed(os.path.join(HERE, "projection.npz"), **out)


def gen_shrinkage():
    rng = np.random.default_rng(99)
    out = {}
    idx = 0
    for shape in [(3, 2, 3, 3), (5, 4, 2, 3), (16, 8, 1, 1), (8, 3, 7, 7), (12, 10, 3, 3)]:
        layer = LayerSpec("c", LayerKind.CONV, shape, prunable=True)
        for variant in ("ones", "zeros", "rect", "elem", "sparse"):
            if variant == "ones":
                m = np.ones(shape, bool)
            elif variant == "zeros":
                m = np.zeros(shape, bool)
            elif variant == "rect":
                ko = rng.choice(shape[0], size=rng.integers(1, shape[0] + 1), replace=False)
                ki = rng.choice(shape[1], size=rng.integers(1, shape[1] + 1), replace=False)
                m = np.zeros(shape, bool)
                m[np.ix_(np.sort(ko), np.sort(ki))] = True
            elif variant == "elem":
                m = rng.random(shape) < 0.5
            else:
                m = rng.random(shape) < 0.02
            keep = derive_keep_sets(m, layer)
            t = f32(rng.normal(size=shape))
            cb = compress(t, keep)
            out[f"s{idx}_mask"] = m
            out[f"s{idx}_t"] = t
            out[f"s{idx}_kout"] = np.array(keep.k_out, dtype=np.int64)
            out[f"s{idx}_kin"] = np.array(keep.k_in, dtype=np.int64)
            out[f"s{idx}_compact"] = cb.data
            out[f"s{idx}_restored"] = decompress(cb, keep, shape)
            idx += 1
    out["n"] = np.array(idx)
    np.savez_compressed(os.path.join(HERE, "shrinkage.npz"), **out)


def gen_bucketize():
    rng = np.random.default_rng(5)
    cases = []
    for cap, count in [(256, 12), (100, 6), (3200, 8), (32 * 1024 * 1024, 4)]:
        sizes = [int(s) for s in rng.integers(1, 90, size=count)]
        if cap == 100:
            sizes[2] = 50                     # oversize payload
        if cap == 32 * 1024 * 1024:
            sizes = [4_000_000, 5_000_000, 2_359_296, 9_000_000]
        named = [(f"t{i}", np.zeros(s)) for i, s in enumerate(sizes)]
        layout = [list(map(list, b.layout)) for b in bucketize(named, cap_bytes=cap)]
        cases.append({"cap": cap, "sizes": sizes, "layout": layout})
    with open(os.path.join(HERE, "bucketize.json"), "w") as fh:
        json.dump(cases, fh, indent=1)


def gen_candidate():
    rng = np.random.default_rng(7)
    out = {}
    params = [(1.5e-3, 1.5e-4, 1e-4, 2, 2), (0.3, 0.1, 0.01, 2, 4), (0.7, 0.0, 0.0, 3, 1),
              (1.5e-3, 1.5e-4, 1e-4, 4, 2), (2.0, 5.0, 1e-4, 1, 8)]
    for i, (r1, r2, wd, m, p) in enumerate(params):
        s, z, v = (f32(rng.normal(size=(64, 33))) for _ in range(3))
        out[f"k{i}_svz"] = np.stack([s, z, v])
        out[f"k{i}_par"] = np.array([r1, r2, wd, m, p], dtype=np.float64)
        out[f"k{i}_out"] = node_candidate(s, z, v, r1, r2, wd, m, p)
    out["n"] = np.array(len(params))
    np.savez_compressed(os.path.join(HERE, "candidate.npz"), **out)


# -- end-to-end runs of run_hierarchical with phase 1 replaced ------------------

E2E_LAYERS = [
    ("stem", LayerKind.CONV, (8, 3, 3, 3), [("channel", 0.5)]),
    ("bn1.w", LayerKind.FULLY_CONNECTED, (1, 8), []),
    ("conv_a", LayerKind.CONV, (16, 8, 3, 3), [("channel", 0.5)]),
    ("conv_b", LayerKind.CONV, (32, 16, 1, 1), [("channel", 0.4)]),
    ("conv_c", LayerKind.CONV, (8, 32, 3, 3), [("filter", 0.75), ("channel", 0.5)]),
    ("conv_d", LayerKind.CONV, (12, 8, 1, 1), [("shape", 0.5)]),
    ("conv_e", LayerKind.CONV, (8, 12, 3, 3), []),
    ("fc.w", LayerKind.FULLY_CONNECTED, (10, 8), []),
    ("fc.b", LayerKind.FULLY_CONNECTED, (1, 10), []),
]
E2E_ITERS = 5
E2E_T_FREEZE = 4


class _FixedWorkload:
    kind = "fixed"

    def __init__(self, layers, params0, world):
        self.layers = layers
        self.shards = [None] * world
        self._p0 = params0

    def init_params(self, rng):
        return {k: v.copy() for k, v in self._p0.items()}


def gen_e2e(num_nodes, per_node, seed=3, adapt=False):
    world = num_nodes * per_node
    rng = np.random.default_rng([seed, 777, num_nodes, per_node])
    specs = [LayerSpec(n, kind, shape, prunable=bool(c)) for n, kind, shape, c in E2E_LAYERS]
    constraints = {n: [SparsityConstraint(KINDS[k], keep_rate=r) for k, r in c]
                   for n, _, _, c in E2E_LAYERS if c}
    params0 = {}
    for ls in specs:
        t = rng.normal(0.0, 0.5, size=ls.shape)
        if ls.kind is LayerKind.CONV:
            t = t * rng.uniform(0.2, 1.0, size=(1, ls.shape[1], 1, 1))
        params0[ls.name] = f32(t)
    thetas = {(r, k): {n: f32(params0[n] + rng.normal(0, 0.05, size=params0[n].shape))
                       for n in params0}
              for k in range(1, E2E_ITERS + 1) for r in range(world)}
    names = [ls.name for ls in specs]
    sched = PenaltySchedule.uniform(names, 1.5e-3, 1.5e-4, adapt=adapt)
    solver = SolverConfig()
    out = {"meta": np.array([num_nodes, per_node, E2E_ITERS, E2E_T_FREEZE])}
    for n in names:  # inputs are fp32-representable: stored as float32 (exact)
        out[f"p0/{n}"] = params0[n].astype(np.float32)
        for k in range(1, E2E_ITERS + 1):
            for r in range(world):
                out[f"theta/{k}/{r}/{n}"] = thetas[(r, k)][n].astype(np.float32)
    saved = (ref_consensus.batch_rng, ref_consensus.proximal_sgd)
    try:
        ref_consensus.batch_rng = lambda s, rank, k: (rank, k)
        ref_consensus.proximal_sgd = lambda wl, shard, th, zn, u, rho1, solver, key: {
            n: a.copy() for n, a in thetas[key].items()}
        for iters in range(1, E2E_ITERS + 1):
            settings = ConsensusSettings(iterations=iters, t_freeze=E2E_T_FREEZE,
                                         stop_on_convergence=False, weight_decay=1e-4, seed=seed)
            cluster = Cluster(Topology(num_nodes, per_node))
            res = run_hierarchical(cluster, _FixedWorkload(specs, params0, world), constraints,
                                   sched, solver, settings)
            if adapt and iters == E2E_ITERS:  # phase 5 per iteration, from the trace rows
                for row in res[0].trace:
                    k = row["k"]
                    out[f"report/{k}"] = ref_consensus.pack_report(row["report"], names)
                    out[f"rho1/{k}"] = np.array([row["rho1"][n] for n in names])
                    out[f"rho2/{k}"] = np.array([row["rho2"][n] for n in names])
                for r in range(world):
                    for row in res[r].trace:
                        out[f"r_intra/{row['k']}/{r}"] = np.array([row["r_intra"][n] for n in names])
                out["rho_final"] = np.array([[res[0].state.schedule.rho1[n] for n in names],
                                             [res[0].state.schedule.rho2[n] for n in names]])
            for r in range(world):
                st = res[r].state
                for n in names:
                    out[f"u/{iters}/{r}/{n}"] = st.u[n]
                out[f"cache/{iters}/{r}"] = np.array([res[r].cache_derive, res[r].cache_hits])
            # z_node, v, z and the masks are bitwise identical on every rank of a
            # node (checked here); store them once per node.
            for i in range(num_nodes):
                lead = res[i * per_node].state
                for r in range(i * per_node, (i + 1) * per_node):
                    st = res[r].state
                    assert st.frozen == lead.frozen
                    for grp in ("z_node", "v", "z", "masks"):
                        for n, a in getattr(lead, grp).items():
                            assert np.array_equal(getattr(st, grp)[n], a), (grp, n, r)
                for grp in ("z_node", "v", "z"):
                    for n in names:
                        out[f"{grp}/{iters}/{i}/{n}"] = getattr(lead, grp)[n]
                for n, m in lead.masks.items():
                    out[f"mask/{iters}/{i}/{n}"] = m
                out[f"frozen/{iters}/{i}"] = np.array(lead.frozen)
            zs = [e.to_dict() for e in cluster.ledger.entries
                  if e.iteration == iters and e.label.startswith("z_sync")]
            out[f"zsync/{iters}"] = np.array(json.dumps(zs))
            if adapt:  # the whole ledger of the iteration (phase 5 included)
                out[f"ledger/{iters}"] = np.array(json.dumps([e.to_dict() for e in cluster.ledger.entries
                                                               if e.iteration == iters]))
    finally:
        ref_consensus.batch_rng, ref_consensus.proximal_sgd = saved
    tag = "e2e_adapt" if adapt else "e2e"
    np.savez_compressed(os.path.join(HERE, f"{tag}_{num_nodes}x{per_node}.npz"), **out)


# -- phase-1 boundary: the proximal-SGD update rule (workloads.py:296-321) ------

PROX_STEPS = 6   # 2 epochs x 3 mini-batches


def gen_prox(seed=5):
    """proximal_sgd with a stub workload whose loss_and_grad returns recorded
    gradients in call order: pins the fused update (combined gradient, momentum,
    lr) independent of any model."""
    from admmprune.workloads import Shard, proximal_sgd

    rng = np.random.default_rng([seed, 919])
    shapes = {n: shape for n, _, shape, _ in E2E_LAYERS}
    names = list(shapes)
    w0 = {n: f32(rng.normal(0, 0.5, size=sh)) for n, sh in shapes.items()}
    z = {n: f32(w0[n] + rng.normal(0, 0.05, size=sh)) for n, sh in shapes.items()}
    u = {n: f32(rng.normal(0, 0.01, size=sh)) for n, sh in shapes.items()}
    rho1 = {n: float(r) for n, r in zip(names, rng.choice([1.5e-3, 0.024, 0.75, 10.0], size=len(names)))}
    grads = [{n: f32(rng.normal(0, 0.1, size=sh)) for n, sh in shapes.items()} for _ in range(PROX_STEPS)]
    calls = iter(grads)

    class _Stub:
        def loss_and_grad(self, params, features, targets):
            return 0.0, next(calls)

    cfg = SolverConfig(lr=0.05, epochs=2, batch_size=4, momentum=0.9)
    shard = Shard(np.zeros((12, 1)), np.zeros(12))
    out = proximal_sgd(_Stub(), shard, w0, z, u, rho1, cfg, np.random.default_rng(0))
    fx = {"meta": np.array([cfg.lr, cfg.momentum, PROX_STEPS]), "rho1": np.array([rho1[n] for n in names])}
    for n in names:
        fx[f"w0/{n}"] = w0[n].astype(np.float32)
        fx[f"z/{n}"] = z[n].astype(np.float32)
        fx[f"u/{n}"] = u[n].astype(np.float32)
        fx[f"out/{n}"] = out[n]
        for i, g in enumerate(grads):
            fx[f"g/{i}/{n}"] = g[n].astype(np.float32)
    np.savez_compressed(os.path.join(HERE, "prox_sgd.npz"), **fx)


# -- comparison baselines (baselines.py) ---------------------------


def _spy(gen, on_yield):
    """Drive ``gen`` transparently; on_yield(gen, request) sees every request while the
    generator is suspended at it (its frame locals are the program state)."""
    try:
        req = next(gen)
        while True:
            on_yield(gen, req)
            try:
                res = yield req
            except BaseException as exc:        # noqa: BLE001 — forward into the program
                req = gen.throw(exc)
                continue
            req = gen.send(res)
    except StopIteration as stop:
        return stop.value


def gen_flat(world, adapt, seed=3):
    """run_flat_consensus (baselines.py:151-293) with phase 1 replaced by recorded thetas.
    The state after iteration k (z, u post-rescale, masks, frozen, rho1) is read from the
    program's frame at the first collective of iteration k + 1; the report / drift / r_intra
    from the trace rows; the ledger per iteration."""
    import admmprune.baselines as ref_base

    rng = np.random.default_rng([seed, 778, world, int(adapt)])
    specs = [LayerSpec(n, kind, shape, prunable=bool(c)) for n, kind, shape, c in E2E_LAYERS]
    constraints = {n: [SparsityConstraint(KINDS[k], keep_rate=r) for k, r in c]
                   for n, _, _, c in E2E_LAYERS if c}
    names = [ls.name for ls in specs]
    params0 = {}
    for ls in specs:
        t = rng.normal(0.0, 0.5, size=ls.shape)
        if ls.kind is LayerKind.CONV:
            t = t * rng.uniform(0.2, 1.0, size=(1, ls.shape[1], 1, 1))
        params0[ls.name] = f32(t)
    iters = E2E_ITERS
    thetas = {(r, k): {n: f32(params0[n] + rng.normal(0, 0.05, size=params0[n].shape)) for n in names}
              for k in range(1, iters + 2) for r in range(world)}
    sched = PenaltySchedule.uniform(names, 1.5e-3, 1.5e-4, adapt=adapt)
    settings = ConsensusSettings(iterations=iters + 1, t_freeze=E2E_T_FREEZE, stop_on_convergence=False,
                                 weight_decay=1e-4, seed=seed)
    out = {"meta": np.array([world, iters, E2E_T_FREEZE, int(adapt)])}
    for n in names:
        out[f"p0/{n}"] = params0[n].astype(np.float32)
        for k in range(1, iters + 1):
            for r in range(world):
                out[f"theta/{k}/{r}/{n}"] = thetas[(r, k)][n].astype(np.float32)

    def capture(rank):
        def on_yield(gen, req):
            if req.tag != f"z_sync/{names[0]}" or req.iteration < 2:
                return
            k, f = req.iteration - 1, gen.gi_frame.f_locals
            for n in names:
                out[f"z/{k}/{rank}/{n}"] = f["z_prev"][n].copy()
                out[f"u/{k}/{rank}/{n}"] = f["u"][n].copy()
            for n, m in f["masks"].items():
                out[f"mask/{k}/{rank}/{n}"] = m.copy()
            out[f"frozen/{k}/{rank}"] = np.array(f["frozen"])
            out[f"rho1_after/{k}/{rank}"] = np.array([f["sched"].rho1[n] for n in names])
        return on_yield

    saved = (ref_base.batch_rng, ref_base.proximal_sgd)
    try:
        ref_base.batch_rng = lambda s, rank, k: (rank, k)
        ref_base.proximal_sgd = lambda wl, shard, th, z, u, rho1, solver, key: {
            n: a.copy() for n, a in thetas[key].items()}
        cluster = Cluster(Topology(1, world))
        wl = _FixedWorkload(specs, params0, world)
        progs = {r: _spy(ref_base.flat_consensus_program(r, cluster, wl, constraints, sched, SolverConfig(),
                                                          settings), capture(r))
                 for r in range(world)}
        res = cluster.run(progs)
    finally:
        ref_base.batch_rng, ref_base.proximal_sgd = saved
    for row in res[0].trace[:iters]:
        k = row["k"]
        out[f"report/{k}"] = ref_consensus.pack_report(row["report"], names)
        out[f"rho1/{k}"] = np.array([row["rho1"][n] for n in names])
        out[f"drift/{k}"] = np.array(json.dumps(row["drift"]))
        out[f"popcount/{k}"] = np.array(json.dumps(row["mask_popcount"]))
    for r in range(world):
        for row in res[r].trace[:iters]:
            out[f"r_intra/{row['k']}/{r}"] = np.array([row["r_intra"][n] for n in names])
    for k in range(1, iters + 1):
        out[f"ledger/{k}"] = np.array(json.dumps([e.to_dict() for e in cluster.ledger.entries
                                                   if e.iteration == k]))
    np.savez_compressed(os.path.join(HERE, f"flat_{'adapt_' if adapt else ''}{world}.npz"), **out)


DENSE_STEPS = 4


def gen_dense(world, seed=3):
    """run_dense_sync (baselines.py:77-98, 260-266) with a stub workload whose
    loss_and_grad returns recorded per-rank gradients: pins the all-rank gradient AVG
    (weight decay folded in), momentum and lr, and the bit-identical parameters."""
    import admmprune.baselines as ref_base
    from admmprune.workloads import Shard

    rng = np.random.default_rng([seed, 779, world])
    specs = [LayerSpec(n, kind, shape, prunable=False) for n, kind, shape, _ in E2E_LAYERS]
    names = [ls.name for ls in specs]
    params0 = {ls.name: f32(rng.normal(0.0, 0.5, size=ls.shape)) for ls in specs}
    grads = {(r, s): {n: f32(rng.normal(0, 0.1, size=params0[n].shape)) for n in names}
             for s in range(1, DENSE_STEPS + 1) for r in range(world)}
    calls = {r: 0 for r in range(world)}

    class _Stub(_FixedWorkload):
        def loss_and_grad(self, params, features, targets):
            r = int(features[0, 0])
            calls[r] += 1
            return float(r), {n: g.copy() for n, g in grads[(r, calls[r])].items()}

    wl = _Stub(specs, params0, world)
    wl.shards = [Shard(np.full((8, 1), float(r)), np.zeros(8)) for r in range(world)]
    solver = SolverConfig(lr=0.05, momentum=0.9, weight_decay=1e-4, batch_size=4)
    cluster = Cluster(Topology(1, world))
    res = ref_base.run_dense_sync(cluster, wl, solver, DENSE_STEPS, seed)
    out = {"meta": np.array([world, DENSE_STEPS]), "solver": np.array([solver.lr, solver.momentum,
                                                                       solver.weight_decay])}
    for n in names:
        out[f"p0/{n}"] = params0[n].astype(np.float32)
        out[f"out/{n}"] = res[0].params[n]
        for (r, s), g in grads.items():
            out[f"g/{s}/{r}/{n}"] = g[n].astype(np.float32)
    out["ledger"] = np.array(json.dumps([e.to_dict() for e in cluster.ledger.entries]))
    np.savez_compressed(os.path.join(HERE, f"dense_{world}.npz"), **out)


TOPK_RATE = 0.1


def gen_topk(world, rate=TOPK_RATE, seed=3):
    """run_topk (baselines.py:101-148, 269-275) with recorded per-rank gradients: the
    final parameters, every rank's selected indices per step and layer (read from the
    program frame at its all-gather), the ledger. Layer fc.b starts at zero with
    gradients of equal magnitude (exact ties: the lower index must win)."""
    import admmprune.baselines as ref_base
    from admmprune.workloads import Shard

    rng = np.random.default_rng([seed, 780, world])
    specs = [LayerSpec(n, kind, shape, prunable=False) for n, kind, shape, _ in E2E_LAYERS]
    names = [ls.name for ls in specs]
    params0 = {ls.name: f32(rng.normal(0.0, 0.5, size=ls.shape)) for ls in specs}
    params0["fc.b"][:] = 0.0
    grads = {}
    for s in range(1, DENSE_STEPS + 1):
        for r in range(world):
            g = {n: f32(rng.normal(0, 0.1, size=params0[n].shape)) for n in names}
            g["fc.b"] = f32(rng.choice([-0.25, 0.25, 0.5, -0.5], size=params0["fc.b"].shape))
            grads[(r, s)] = g
    calls = {r: 0 for r in range(world)}

    class _Stub(_FixedWorkload):
        def loss_and_grad(self, params, features, targets):
            r = int(features[0, 0])
            calls[r] += 1
            return float(r), {n: g.copy() for n, g in grads[(r, calls[r])].items()}

    wl = _Stub(specs, params0, world)
    wl.shards = [Shard(np.full((8, 1), float(r)), np.zeros(8)) for r in range(world)]
    solver = SolverConfig(lr=0.05, momentum=0.9, weight_decay=1e-4, batch_size=4)
    cluster = Cluster(Topology(1, world))
    out = {"meta": np.array([world, DENSE_STEPS]), "solver": np.array([solver.lr, solver.momentum,
                                                                       solver.weight_decay, rate])}

    def capture(rank):
        def on_yield(gen, req):
            f = gen.gi_frame.f_locals
            out[f"sel/{req.iteration}/{rank}/{f['n']}"] = np.asarray(f["sel"], dtype=np.int64)
        return on_yield

    progs = {r: _spy(ref_base.topk_program(r, cluster, wl, solver, DENSE_STEPS, seed, rate), capture(r))
             for r in range(world)}
    res = cluster.run(progs)
    ref_base._check_divergence(res)
    for n in names:
        out[f"p0/{n}"] = params0[n].astype(np.float32)
        out[f"out/{n}"] = res[0].params[n]
        for (r, s), g in grads.items():
            out[f"g/{s}/{r}/{n}"] = g[n].astype(np.float32)
    out["ledger"] = np.array(json.dumps([e.to_dict() for e in cluster.ledger.entries]))
    np.savez_compressed(os.path.join(HERE, f"topk_{world}.npz"), **out)


if __name__ == "__main__":
    gen_projection()
    gen_shrinkage()
    gen_bucketize()
    gen_candidate()
    for m, p in [(1, 1), (2, 1), (1, 2), (2, 2), (2, 4), (4, 2), (1, 4), (4, 1)]:
        gen_e2e(m, p)
    for m, p in [(1, 1), (2, 1), (1, 2), (2, 2), (2, 4), (4, 2)]:
        gen_e2e(m, p, adapt=True)
    gen_prox()
    gen_flat(2, False)
    for w in (1, 2, 4):
        gen_flat(w, True)
        gen_dense(w)
        gen_topk(w)
    print("golden fixtures written to", HERE)
