"""Multi-GPU parity, one rank per GPU over NCCL (run under torchrun).

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tests/mp_parity.py 2x2

1) The reference's run_hierarchical golden vectors for this topology
   (tests/golden/e2e_MxP.npz): every rank steps HSADMMSync through DistCluster
   (intra all-reduce, leader all-gather of mask bits + OR, leader all-reduce of
   the compact buffer, intra broadcast) and checks masks bit-exact and z_node /
   u / v / z within 1e-5 of the reference at every iteration.
2) A synthetic ResNet-18 (CIFAR shapes) state at full size: after dynamic and
   frozen iterations every rank of a node holds bitwise-identical z_node, v, z
   and every rank holds the same union masks; the leader payload matches the
   keep sets.
Exit code 0 on success on every rank.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2512_14628_b200 as H  # noqa: E402
from tests import golden_io as G  # noqa: E402

TOL = 1e-5


def rel_err(got, ref, *ops):
    scale = max([np.abs(ref).max()] + [np.abs(o).max() for o in ops] + [1e-30])
    return float(np.abs(np.asarray(got, np.float64) - ref).max() / scale)


def golden_check(topo, rank, transport, residuals=True):
    ref = G.E2E(topo.num_nodes, topo.accels_per_node)
    kinds = {"filter": H.ConstraintKind.FILTER_KEEP, "channel": H.ConstraintKind.CHANNEL_KEEP,
             "shape": H.ConstraintKind.SHAPE_KEEP}
    layers = [H.LayerSpec(n, H.LayerKind.CONV if k == "conv" else H.LayerKind.FULLY_CONNECTED, s,
                          prunable=bool(c)) for n, k, s, c in G.E2E_LAYERS]
    cons = {n: [H.SparsityConstraint(kinds[g], keep_rate=r) for g, r in c] for n, _, _, c in G.E2E_LAYERS if c}
    sched = H.PenaltySchedule.uniform(ref.names, G.E2E_RHO1, G.E2E_RHO2, adapt=False)
    settings = H.ConsensusSettings(t_freeze=ref.t_freeze, weight_decay=G.E2E_WD)
    cluster = H.DistCluster(topo)
    eng = H.HSADMMSync(rank, cluster, layers, cons, sched, settings, transport=transport, residuals=residuals)
    assert eng.transport == transport
    eng.init_from(ref.p0())
    node = topo.node_of(rank)
    worst = 0.0
    for k in range(1, ref.iters + 1):
        th = ref.theta(k, rank)
        eng.load(theta=th)
        eng.step(k)
        assert eng.frozen == ref.frozen(k, node), (k, rank)
        for n, m in ref.masks(k, node).items():
            assert np.array_equal(eng.mask_dict()[n].cpu().numpy(), m), (k, rank, n)
        for key, want in (("z_node", ref.node_state("z_node", k, node)), ("v", ref.node_state("v", k, node)),
                          ("z", ref.node_state("z", k, node)), ("u", ref.u(k, rank))):
            for n, t in eng.views(key).items():
                err = rel_err(t.cpu().numpy(), want[n], th[n])
                worst = max(worst, err)
                assert err <= TOL, (k, rank, key, n, err)
        if eng.is_leader:
            assert (eng.cache_derive, eng.cache_hits) == ref.cache(k, rank)
            zs = [e.to_dict() for e in cluster.ledger.entries if e.iteration == k and e.label.startswith("z_sync")]
            assert zs == ref.zsync(k), (zs, ref.zsync(k))
    eng.check_barriers()
    return worst


def adaptive_check(topo, rank, transport):
    """Phase 5 over the real collectives: run_hierarchical(adapt=True) goldens —
    penalties exact every iteration, report within 1e-5, state within 1e-5."""
    ref = G.E2E(topo.num_nodes, topo.accels_per_node, adapt=True)
    kinds = {"filter": H.ConstraintKind.FILTER_KEEP, "channel": H.ConstraintKind.CHANNEL_KEEP,
             "shape": H.ConstraintKind.SHAPE_KEEP}
    layers = [H.LayerSpec(n, H.LayerKind.CONV if k == "conv" else H.LayerKind.FULLY_CONNECTED, s,
                          prunable=bool(c)) for n, k, s, c in G.E2E_LAYERS]
    cons = {n: [H.SparsityConstraint(kinds[g], keep_rate=r) for g, r in c] for n, _, _, c in G.E2E_LAYERS if c}
    sched = H.PenaltySchedule.uniform(ref.names, G.E2E_RHO1, G.E2E_RHO2, adapt=True)
    settings = H.ConsensusSettings(t_freeze=ref.t_freeze, weight_decay=G.E2E_WD)
    eng = H.HSADMMSync(rank, H.DistCluster(topo), layers, cons, sched, settings, transport=transport)
    eng.init_from(ref.p0())
    node = topo.node_of(rank)
    for k in range(1, ref.iters + 1):
        r1, r2 = ref.rho(k)
        s = eng.current_schedule()
        assert [s.rho1[n] for n in ref.names] == list(r1) and [s.rho2[n] for n in ref.names] == list(r2), k
        th = ref.theta(k, rank)
        eng.load(theta=th)
        eng.step(k)
        rep = eng.last_report()
        got = np.array([x for n in ref.names for x in (
            rep.layers[n].r_intra, rep.layers[n].s_intra, rep.layers[n].r_inter, rep.layers[n].s_inter,
            rep.layers[n].eps_pri_intra, rep.layers[n].eps_dual_intra, rep.layers[n].eps_pri_inter,
            rep.layers[n].eps_dual_inter)] + [rep.r_pri, rep.r_dual, rep.eps_pri, rep.eps_dual, float(rep.converged)])
        want = ref.report(k)
        assert got[-1] == want[-1], (k, rank)
        assert float((np.abs(got - want) / np.maximum(np.abs(want), 1e-30)).max()) <= TOL, (k, rank)
        for key, w in (("z_node", ref.node_state("z_node", k, node)), ("v", ref.node_state("v", k, node)),
                       ("z", ref.node_state("z", k, node)), ("u", ref.u(k, rank))):
            for n, t in eng.views(key).items():
                err = rel_err(t.cpu().numpy(), w[n], th[n])
                assert err <= TOL, (k, rank, key, n, err)
    return True


def replica_check(topo, rank, world, transport, residuals=True, steps=4):
    from paper_2512_14628_b200.synthetic import channel_keep_constraints, model_layers, synthetic_rank_state

    layers = model_layers("rn18_cifar")
    cons = channel_keep_constraints(layers, 0.5)
    sched = H.PenaltySchedule.uniform([ls.name for ls in layers], 1.5e-3, 1.5e-4, adapt=False)
    settings = H.ConsensusSettings(t_freeze=3, weight_decay=1e-4)
    cluster = H.DistCluster(topo)
    eng = H.HSADMMSync(rank, cluster, layers, cons, sched, settings, transport=transport, residuals=residuals)
    eng.load(**synthetic_rank_state(layers, rank, topo.accels_per_node, seed=5))
    # steps back to back with no host sync in between (residuals off: no NCCL call
    # orders the ranks, only the device barriers and the double-buffered sends)
    for k in range(1, steps + 1):
        eng.step(k)
    eng.check_barriers()
    assert eng.frozen
    # every rank of a node: identical z_node, v, z; every rank: identical masks
    for key in ("z_node", "v", "z", "masks"):
        t = getattr(eng, key).contiguous()
        buf = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(buf, t)
        for r in range(world):
            if key == "masks" or topo.node_of(r) == topo.node_of(rank):
                assert torch.equal(buf[r], t), (key, r, rank)
    ratio = eng.payload_elements / sum(ls.elements for ls in layers)
    assert 0.45 < ratio < 0.6, ratio
    return ratio


def baselines_check(topo, rank, world, transport):
    """Flat consensus and dense sync (baselines.py) over the real collectives: the
    run_flat_consensus(adapt) / run_dense_sync goldens for W ranks, any topology."""
    if world in [w for w, adapt in G.FLAT_CASES if adapt]:
        ref = G.Flat(world, True)
        kinds = {"filter": H.ConstraintKind.FILTER_KEEP, "channel": H.ConstraintKind.CHANNEL_KEEP,
                 "shape": H.ConstraintKind.SHAPE_KEEP}
        layers = [H.LayerSpec(n, H.LayerKind.CONV if k == "conv" else H.LayerKind.FULLY_CONNECTED, s,
                              prunable=bool(c)) for n, k, s, c in G.E2E_LAYERS]
        cons = {n: [H.SparsityConstraint(kinds[g], keep_rate=r) for g, r in c] for n, _, _, c in G.E2E_LAYERS if c}
        sched = H.PenaltySchedule.uniform(ref.names, G.E2E_RHO1, G.E2E_RHO2, adapt=True)
        settings = H.ConsensusSettings(t_freeze=ref.t_freeze, weight_decay=G.E2E_WD)
        eng = H.FlatConsensusSync(rank, H.DistCluster(topo), layers, cons, sched, settings, transport=transport)
        eng.init_from(ref.p0())
        for k in range(1, ref.iters + 1):
            assert [eng.current_schedule().rho1[n] for n in ref.names] == list(ref.rho1(k)), k
            th = ref.theta(k, rank)
            eng.load(theta=th)
            eng.step(k)
            rep = eng.last_report()
            assert float(rep.converged) == ref.report(k)[-1], k
            assert abs(rep.r_pri - ref.report(k)[-5]) <= TOL * ref.report(k)[-5], k
            for key in ("z", "u"):
                w = ref.state(key, k, rank)
                for n, t in eng.views(key).items():
                    err = rel_err(t.cpu().numpy(), w[n], th[n])
                    assert err <= TOL, ("flat", k, rank, key, n, err)
            for n, m in ref.masks(k, rank).items():
                assert np.array_equal(eng.mask_dict()[n].cpu().numpy(), m), (k, rank, n)
    if world in G.DENSE_WORLDS:
        ref = G.Dense(world)
        layers = [H.LayerSpec(n, H.LayerKind.CONV if k == "conv" else H.LayerKind.FULLY_CONNECTED, s)
                  for n, k, s, _ in G.E2E_LAYERS]

        class Solver:
            lr, momentum, weight_decay = ref.lr, ref.momentum, ref.weight_decay

        eng = H.DenseSync(rank, H.DistCluster(topo), layers, Solver, transport=transport)
        eng.init_from(ref.p0())
        for s in range(1, ref.steps + 1):
            eng.load_grads(ref.grads(s, rank))
            eng.step(s)
        out = ref.out()
        for n, t in eng.views("params").items():
            err = rel_err(t.cpu().numpy(), out[n], ref.p0()[n])
            assert err <= TOL, ("dense", rank, n, err)
        buf = [torch.empty_like(eng.params) for _ in range(world)]
        dist.all_gather(buf, eng.params)
        assert all(torch.equal(b, eng.params) for b in buf), "dense params diverged across ranks"
        ref = G.TopK(world)
        Solver.lr, Solver.momentum, Solver.weight_decay = ref.lr, ref.momentum, ref.weight_decay
        eng = H.TopKSync(rank, H.DistCluster(topo), layers, Solver, ref.rate)
        eng.init_from(ref.p0())
        for s in range(1, ref.steps + 1):
            eng.load_grads(ref.grads(s, rank))
            eng.step(s)
            for n, t in eng.selections().items():
                assert np.array_equal(t.cpu().numpy(), ref.sel(s, rank, n)), ("topk", s, rank, n)
        out = ref.out()
        for n, t in eng.views("params").items():
            err = rel_err(t.cpu().numpy(), out[n], ref.p0()[n])
            assert err <= TOL, ("topk", rank, n, err)
        dist.all_gather(buf, eng.params)
        assert all(torch.equal(b, eng.params) for b in buf), "top-k params diverged across ranks"
    return True


def main():
    import faulthandler

    faulthandler.dump_traceback_later(int(os.environ.get("MP_PARITY_DUMP_S", "240")), exit=False)
    topo = H.Topology.parse(sys.argv[1])
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        for transport in os.environ.get("MP_PARITY_TRANSPORTS", "nccl,peer").split(","):
            worst = golden_check(topo, rank, transport)
            print(f"rank {rank} golden {transport} done", file=sys.stderr, flush=True)
            if (topo.num_nodes, topo.accels_per_node) in G.E2E_ADAPT_TOPOLOGIES:
                adaptive_check(topo, rank, transport)
                print(f"rank {rank} adaptive {transport} done", file=sys.stderr, flush=True)
            baselines_check(topo, rank, world, transport)
            print(f"rank {rank} baselines {transport} done", file=sys.stderr, flush=True)
            ratio = replica_check(topo, rank, world, transport)
            if transport == "peer":
                # the send / leader buffers are reused across back-to-back steps
                golden_check(topo, rank, transport, residuals=False)
                replica_check(topo, rank, world, transport, residuals=False, steps=12)
                print(f"rank {rank} peer residuals-off done", file=sys.stderr, flush=True)
            dist.barrier()
            if rank == 0:
                print(f"mp_parity {sys.argv[1]} {transport} ok: worst rel err {worst:.2e}, "
                      f"rn18_cifar leader payload ratio {ratio:.3f}", flush=True)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
