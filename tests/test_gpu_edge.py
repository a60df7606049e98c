"""Edge cases of the sync step against the oracle (oracle/hsadmm_oracle.py, pinned
to the reference), on identical inputs, in one process (LocalCluster):

* a prunable layer whose state is all zeros: every group norm ties at 0, the kept
  groups (lower indices) are all zero, so the union mask, K_out and K_in are empty
  and the layer sends no payload (reference consensus.py:478-481, decompress of an
  empty keep set -> zeros :498-504);
* keep rate 1.0 (nothing dropped: payload = dense);
* no prunable layer at all (every layer dense: no selection, projection or union);
* a layer with a single output row and one with a single input channel (ragged
  c_in * kh * kw, rows not a multiple of the tile height).
Masks, payload sizes and z_sync ledger entries exact, state within 1e-5.
"""

import numpy as np
import pytest
import torch

from oracle import hsadmm_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-5


def rel_err(got, ref, *ops):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    scale = max([np.abs(ref).max()] + [np.abs(np.asarray(o, np.float64)).max() for o in ops] + [1e-30])
    return float(np.abs(got - ref).max() / scale)


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.set_device(0)


SPEC = [("c0", (16, 8, 3, 3)), ("b0", (1, 16)), ("c1", (32, 16, 3, 3)), ("c2", (1, 32, 1, 1)),
        ("c3", (24, 1, 3, 3)), ("c4", (8, 24, 1, 1)), ("fc", (10, 8)), ("fcb", (1, 10))]


def run_case(M, P, transport, keep, prunable, zero_layers=(), iters=3, t_freeze=2, seed=0):
    import paper_2512_14628_b200 as H

    rng = np.random.default_rng([seed, M, P])
    names = [n for n, _ in SPEC]
    layers = [H.LayerSpec(n, H.LayerKind.CONV if len(s) == 4 else H.LayerKind.FULLY_CONNECTED, s,
                          prunable=n in prunable) for n, s in SPEC]
    cons = {n: [H.SparsityConstraint(H.ConstraintKind.CHANNEL_KEEP, keep_rate=keep)] for n in prunable}
    sched = H.PenaltySchedule.uniform(names, 1.5e-3, 1.5e-4, adapt=False)
    settings = H.ConsensusSettings(t_freeze=t_freeze, weight_decay=1e-4)
    cluster = H.LocalCluster(H.Topology(M, P))
    engines = [H.HSADMMSync(r, cluster, layers, cons, sched, settings, transport=transport, residuals=False)
               for r in range(M * P)]
    p0 = {}
    for n, s in SPEC:
        t = rng.normal(0, 0.5, size=s)
        if len(s) == 4:
            t = t * rng.uniform(0.2, 1.0, size=(1, s[1], 1, 1))
        p0[n] = (np.zeros(s) if n in zero_layers else t).astype(np.float32)
    for e in engines:
        e.init_from(p0)
    olayers = O.make_layers(SPEC, {n: [(O.CHANNEL, None, keep)] for n in prunable})
    zeros = {n: np.zeros_like(a) for n, a in p0.items()}
    ost = [O.init_rank_state(olayers, p0, zeros, p0, zeros, p0) for _ in range(M * P)]
    rho = {n: 1.5e-3 for n in names}, {n: 1.5e-4 for n in names}
    for k in range(1, iters + 1):
        thetas = [{n: (np.zeros(s) if n in zero_layers else p0[n] + rng.normal(0, 0.05, size=s)).astype(np.float32)
                   for n, s in SPEC} for _ in range(M * P)]
        for e in engines:
            e.load(theta=thetas[e.rank])
        ledger = []
        H.run_local(engines, k)
        O.cluster_sync(olayers, ost, thetas, k, M, P, rho[0], rho[1], 1e-4, t_freeze=t_freeze, ledger=ledger)
        want_z = [d for d in ledger if d["label"].startswith("z_sync")]
        got_z = [d.to_dict() for d in cluster.ledger.entries if d.iteration == k and d.label.startswith("z_sync")]
        assert got_z == want_z, (k, got_z, want_z)
        for e in engines:
            o = ost[e.rank]
            assert e.frozen == o.frozen, (k, e.rank)
            for n, m in e.mask_dict().items():
                assert np.array_equal(m.cpu().numpy(), o.masks[n]), (k, e.rank, n)
            for key in ("z_node", "u", "v", "z"):
                for n, t in e.views(key).items():
                    err = rel_err(t.cpu().numpy(), getattr(o, key)[n], thetas[e.rank][n])
                    assert err <= TOL, (k, e.rank, key, n, err)
            assert e.payload_elements == sum(d["elements"] for d in want_z), (k, e.rank)
    return engines, ost


@pytest.mark.parametrize("M,P,transport", [(1, 1, "nccl"), (2, 2, "nccl"), (2, 2, "peer"), (1, 2, "peer")])
def test_layer_with_empty_union(M, P, transport):
    engines, ost = run_case(M, P, transport, 0.5, ("c0", "c1", "c2", "c3", "c4"), zero_layers=("c1",))
    assert not ost[0].masks["c1"].any()
    assert "c1" not in [n for n, _ in engines[0].payload]


@pytest.mark.parametrize("M,P,transport", [(1, 1, "nccl"), (2, 1, "peer"), (2, 2, "nccl")])
def test_keep_everything(M, P, transport):
    engines, _ = run_case(M, P, transport, 1.0, ("c0", "c1", "c3"))
    assert engines[0].payload_elements == sum(int(np.prod(s)) for _, s in SPEC)


@pytest.mark.parametrize("M,P,transport", [(1, 1, "nccl"), (2, 2, "peer")])
def test_no_prunable_layer(M, P, transport):
    engines, _ = run_case(M, P, transport, 0.5, ())
    assert engines[0].mask_dict() == {}


@pytest.mark.parametrize("M,P,transport", [(1, 1, "nccl"), (2, 2, "nccl"), (2, 2, "peer")])
def test_single_row_and_single_channel_layers(M, P, transport):
    run_case(M, P, transport, 0.3, ("c2", "c3"), iters=2, t_freeze=1)
