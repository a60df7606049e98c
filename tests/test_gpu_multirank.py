"""Full-size multi-rank parity against the CPU oracle on identical inputs.

All ranks of an M x P topology run in one process on cuda:0 (LocalCluster), so
the multi-node path — leader mask union (K4), keep sets from mask bits (K5),
compaction into the flat buffer (K6), the bucketed leader average (the
scheduler's rank-order fold, or K8 over "peer" pointers), the intra broadcast
and decompaction (K7) — runs at BASELINE sizes (ResNet-18 / ResNet-50 224, keep
0.4) against oracle/hsadmm_oracle.py's ``cluster_sync``
(/root/reference/pkg/src/admmprune/consensus.py:436-606).

Stage-wise: before every iteration the oracle's per-rank state is set to the
GPU's fp32 state (upcast exactly), so each iteration is compared on identical
inputs. Bars: masks, K_out / K_in, payload sizes and bucket layouts bit-exact;
z_node / u / v / z within 1e-5 (per-tensor relative error).
Iteration 1 is dynamic; t_freeze = 1 makes iteration 2 frozen (sealed keep
sets, frozen-mask candidate).
"""

import numpy as np
import pytest
import torch

from oracle import hsadmm_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-5


def rel_err(got, ref, *operands):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = max([np.max(np.abs(ref))] + [np.max(np.abs(np.asarray(o, dtype=np.float64))) for o in operands]
                + [1e-30])
    return float(np.max(np.abs(got - ref)) / scale)


def cpu(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


CASES = [("rn18_224", "2x2"), ("rn18_224", "2x4"), ("rn18_224", "4x2"),
         ("rn50_224", "2x2"), ("rn50_224", "2x4"), ("rn50_224", "4x2")]


@pytest.mark.parametrize("transport", ["nccl", "peer"])
@pytest.mark.parametrize("model,grouping", CASES)
def test_full_size_multirank_against_oracle(model, grouping, transport):
    import paper_2512_14628_b200 as H
    from paper_2512_14628_b200.synthetic import (channel_keep_constraints, model_layers, synthetic_base,
                                                 synthetic_rank_state)

    keep = 0.4
    topo = H.Topology.parse(grouping)
    M, P, W = topo.num_nodes, topo.accels_per_node, topo.world_size
    layers = model_layers(model)
    names = [ls.name for ls in layers]
    cons = channel_keep_constraints(layers, keep)
    sched = H.PenaltySchedule.uniform(names, 1.5e-3, 1.5e-4, adapt=False)
    settings = H.ConsensusSettings(t_freeze=1, weight_decay=1e-4)
    cluster = H.LocalCluster(topo)
    engines = [H.HSADMMSync(r, cluster, layers, cons, sched, settings, transport=transport, residuals=False)
               for r in range(W)]
    base = synthetic_base(layers, seed=7)
    thetas = []
    for e in engines:
        st = synthetic_rank_state(layers, e.rank, P, seed=7, base=base)
        e.load(**st)
        thetas.append(st["theta"])
    ocons = {n: [(O.CHANNEL, None, keep)] for n in cons}
    olayers = O.make_layers([(ls.name, ls.shape) for ls in layers], ocons)
    ost = [O.init_rank_state(olayers, {}, {}, {}, {}, {}) for _ in range(W)]
    rho1 = {n: 1.5e-3 for n in names}
    rho2 = {n: 1.5e-4 for n in names}
    leaders = [i * P for i in range(M)]
    for k in (1, 2):
        # stage-wise: the oracle starts from the GPU's fp32 state after iteration k - 1
        for e, o in zip(engines, ost):
            for key in ("u", "v", "z", "z_node"):
                setattr(o, key, {n: cpu(t).astype(np.float64) for n, t in e.views(key).items()})
            o.masks = {n: cpu(m) for n, m in e.mask_dict().items()}
        frozen_before = engines[0].frozen
        assert frozen_before == (k == 2)
        ledger = []
        H.run_local(engines, k)
        O.cluster_sync(olayers, ost, thetas, k, M, P, rho1, rho2, 1e-4, t_freeze=1, ledger=ledger)
        torch.cuda.synchronize()
        # the leader average's buckets: sizes and per-layer detail (payload offsets)
        want_z = [d for d in ledger if d["label"].startswith("z_sync")]
        got_z = [d.to_dict() for d in cluster.ledger.entries if d.iteration == k and d.label.startswith("z_sync")]
        assert got_z == want_z, (k, got_z[:1], want_z[:1])
        for e in engines:
            o = ost[e.rank]
            assert e.frozen == o.frozen, (k, e.rank)
            gm = e.mask_dict()
            for n, m in o.masks.items():
                assert np.array_equal(cpu(gm[n]), m), ("mask", k, e.rank, n)
            for key in ("z_node", "u", "v", "z"):
                for n in names:
                    err = rel_err(cpu(e.views(key)[n]), getattr(o, key)[n], thetas[e.rank][n])
                    assert err <= TOL, (key, k, e.rank, n, err, frozen_before)
            assert e.payload_elements == sum(d["elements"] for d in want_z), (k, e.rank)
        # keep sets (compaction indices) on every rank vs the leader's KeepSetCache
        ocache = ost[leaders[0]].keep_cache
        for e in engines:
            pos_out, pos_in = (cpu(t) for t in e.plan.keep_positions(e.device))
            for i in e.plan.prunable:
                ls = layers[i]
                po = pos_out[e.plan.keep_offset(i, 0):e.plan.keep_offset(i, 0) + ls.shape[0]]
                pi = pos_in[e.plan.keep_offset(i, 1):e.plan.keep_offset(i, 1) + ls.shape[1]]
                ko, ki = ocache[ls.name][1:]
                assert np.array_equal(np.flatnonzero(po >= 0), ko), ("K_out", k, e.rank, ls.name)
                assert np.array_equal(np.flatnonzero(pi >= 0), ki), ("K_in", k, e.rank, ls.name)
                assert np.array_equal(po[ko], np.arange(len(ko))) and np.array_equal(pi[ki], np.arange(len(ki)))
        # leader bytes vs dense: the north_star's ~60% reduction at keep 0.4
        ratio = engines[0].payload_elements / sum(ls.elements for ls in layers)
        assert 0.40 < ratio < 0.50, ratio
    for e, o in zip(engines, ost):
        if e.is_leader:
            assert (e.cache_derive, e.cache_hits) == (o.derive_calls, o.hits), e.rank
    for e in engines:
        e.check_barriers()
