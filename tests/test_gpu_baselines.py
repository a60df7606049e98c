"""GPU parity of the comparison baselines against goldens from the
reference's run_flat_consensus / run_dense_sync (baselines.py:77-98, 151-293) and the
oracle restatement (oracle/hsadmm_oracle.py: flat_consensus_step, dense_sync_step).

Bars as for the sync step (tests/test_gpu_parity.py): masks exact, penalty decisions
exact, fp32 state within 1e-5 (H6 measure), report entries within 1e-5 relative,
the reference ledger entry for entry.
"""

import json

import numpy as np
import pytest
import torch

from tests import golden_io as G
from tests.test_gpu_parity import TOL, cpu, rel_err

pytestmark = pytest.mark.gpu

RTOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2512_14628_b200 import _lib

    _lib.load()
    torch.cuda.set_device(0)


def _flat_engines(world, adapt, transport):
    import paper_2512_14628_b200 as H

    kinds = {"filter": H.ConstraintKind.FILTER_KEEP, "channel": H.ConstraintKind.CHANNEL_KEEP,
             "shape": H.ConstraintKind.SHAPE_KEEP}
    layers = [H.LayerSpec(n, H.LayerKind.CONV if k == "conv" else H.LayerKind.FULLY_CONNECTED, shape,
                          prunable=bool(c)) for n, k, shape, c in G.E2E_LAYERS]
    cons = {n: [H.SparsityConstraint(kinds[g], keep_rate=r) for g, r in c] for n, _, _, c in G.E2E_LAYERS if c}
    names = [n for n, *_ in G.E2E_LAYERS]
    sched = H.PenaltySchedule.uniform(names, G.E2E_RHO1, G.E2E_RHO2, adapt=adapt)
    settings = H.ConsensusSettings(iterations=5, t_freeze=4, weight_decay=G.E2E_WD)
    # any topology of W ranks: the flat program talks to the global group only
    cluster = H.LocalCluster(H.Topology(world, 1) if world > 1 else H.Topology(1, 1))
    return cluster, [H.FlatConsensusSync(r, cluster, layers, cons, sched, settings, transport=transport)
                     for r in range(world)]


def _report_vec(rep, names):
    v = [x for n in names for x in (lambda r: (r.r_intra, r.s_intra, r.r_inter, r.s_inter, r.eps_pri_intra,
                                               r.eps_dual_intra, r.eps_pri_inter, r.eps_dual_inter))(rep.layers[n])]
    return np.array(v + [rep.r_pri, rep.r_dual, rep.eps_pri, rep.eps_dual, float(rep.converged)])


@pytest.mark.parametrize("transport", ["nccl", "peer"])
@pytest.mark.parametrize("world,adapt", G.FLAT_CASES)
def test_flat_consensus_against_reference_goldens(world, adapt, transport):
    import paper_2512_14628_b200 as H

    if transport == "peer" and world == 1:
        pytest.skip("one rank has no peers")
    ref = G.Flat(world, adapt)
    cluster, engines = _flat_engines(world, adapt, transport)
    for e in engines:
        e.init_from(ref.p0())
    saw_frozen = False
    for k in range(1, ref.iters + 1):
        for e in engines:
            s = e.current_schedule()
            assert [s.rho1[n] for n in ref.names] == list(ref.rho1(k)), (k, e.rank)
            e.load(theta=ref.theta(k, e.rank))
        H.run_flat_local(engines, k)
        for e in engines:
            got, want = _report_vec(e.last_report(), ref.names), ref.report(k)
            assert got[-1] == want[-1], k
            err = np.abs(got - want) / np.maximum(np.abs(want), 1e-30)
            assert float(err.max()) <= RTOL, (k, float(err.max()), int(err.argmax()))
            assert e.frozen == ref.frozen(k), k
            th = ref.theta(k, e.rank)
            for n in ref.names:
                for key, want in (("z", ref.state("z", k, e.rank)[n]), ("u", ref.state("u", k, e.rank)[n])):
                    err = rel_err(cpu(e.views(key)[n]), want, th[n])
                    assert err <= TOL, (k, e.rank, key, n, err)
                assert not cpu(e.views("v")[n]).any()
            for n, m in ref.masks(k, e.rank).items():
                assert np.array_equal(cpu(e.mask_dict()[n]), m), (k, e.rank, n)
        assert [engines[0].current_schedule().rho1[n] for n in ref.names] == list(ref.rho1_after(k))
        got = sorted(json.dumps(x.to_dict(), sort_keys=True) for x in cluster.ref_ledger.entries if x.iteration == k)
        want = sorted(json.dumps(x, sort_keys=True) for x in ref.ledger(k))
        assert got == want, (k, set(got) ^ set(want))
        saw_frozen |= ref.frozen(k)
    assert saw_frozen


@pytest.mark.parametrize("transport", ["nccl", "peer"])
@pytest.mark.parametrize("world", G.DENSE_WORLDS)
def test_dense_sync_against_reference_golden(world, transport):
    import paper_2512_14628_b200 as H

    if transport == "peer" and world == 1:
        pytest.skip("one rank has no peers")
    ref = G.Dense(world)
    layers = [H.LayerSpec(n, H.LayerKind.CONV if k == "conv" else H.LayerKind.FULLY_CONNECTED, shape)
              for n, k, shape, _ in G.E2E_LAYERS]

    class Solver:
        lr, momentum, weight_decay = ref.lr, ref.momentum, ref.weight_decay

    cluster = H.LocalCluster(H.Topology(1, world))
    engines = [H.DenseSync(r, cluster, layers, Solver, transport=transport) for r in range(world)]
    for e in engines:
        e.init_from(ref.p0())
    for s in range(1, ref.steps + 1):
        for e in engines:
            e.load_grads(ref.grads(s, e.rank))
        H.run_dense_local(engines, s)
    out = ref.out()
    for e in engines:
        for n in ref.names:
            err = rel_err(cpu(e.views("params")[n]), out[n], ref.p0()[n])
            assert err <= TOL, (e.rank, n, err)
    # bit-identical parameters on every rank (baselines.py:317-329, _check_divergence)
    for e in engines[1:]:
        assert torch.equal(e.params, engines[0].params)
    got = sorted(json.dumps(x.to_dict(), sort_keys=True) for x in cluster.ref_ledger.entries)
    want = sorted(json.dumps(x, sort_keys=True) for x in ref.ledger())
    assert got == want


def test_dense_apply_rejects_bad_arguments():
    from paper_2512_14628_b200 import _lib
    from paper_2512_14628_b200.errors import ConfigError, ShapeError
    from paper_2512_14628_b200.plan import current_stream

    p = torch.zeros(64, device="cuda")
    arr, keep = _lib.ptr_array([p.data_ptr()])
    with pytest.raises(ConfigError):
        _lib.call("hsx_dense_apply", arr, 1, 1.0, p.data_ptr(), p.data_ptr(), 0.0, 0.9, 0, 64, current_stream())
    with pytest.raises(Exception):
        _lib.call("hsx_dense_apply", arr, 5, 1.0, p.data_ptr(), p.data_ptr(), 0.1, 0.9, 0, 64, current_stream())
    del keep, ShapeError


def _topk_engines(ref, world):
    import paper_2512_14628_b200 as H

    layers = [H.LayerSpec(n, H.LayerKind.CONV if k == "conv" else H.LayerKind.FULLY_CONNECTED, shape)
              for n, k, shape, _ in G.E2E_LAYERS]

    class Solver:
        lr, momentum, weight_decay = ref.lr, ref.momentum, ref.weight_decay

    cluster = H.LocalCluster(H.Topology(1, world))
    return cluster, [H.TopKSync(r, cluster, layers, Solver, ref.rate) for r in range(world)]


@pytest.mark.parametrize("world", G.DENSE_WORLDS)
def test_topk_against_reference_golden(world):
    """topk_program (baselines.py:101-148): every rank's selections per step and layer
    exact (ties -> lower index; fc.b is built of exact ties), parameters within 1e-5,
    bit-identical on every rank, the ledger entry for entry."""
    import paper_2512_14628_b200 as H

    ref = G.TopK(world)
    cluster, engines = _topk_engines(ref, world)
    for e in engines:
        e.init_from(ref.p0())
    for s in range(1, ref.steps + 1):
        for e in engines:
            e.load_grads(ref.grads(s, e.rank))
        H.run_topk_local(engines, s)
        for e in engines:
            sel = e.selections()
            for n in ref.names:
                assert np.array_equal(cpu(sel[n]), ref.sel(s, e.rank, n)), (s, e.rank, n)
    out = ref.out()
    for e in engines:
        for n in ref.names:
            err = rel_err(cpu(e.views("params")[n]), out[n], ref.p0()[n])
            assert err <= TOL, (e.rank, n, err)
    for e in engines[1:]:
        assert torch.equal(e.params, engines[0].params)
    got = sorted(json.dumps(x.to_dict(), sort_keys=True) for x in cluster.ref_ledger.entries)
    want = sorted(json.dumps(x, sort_keys=True) for x in ref.ledger())
    assert got == want


def test_topk_full_size_selection_against_oracle():
    """RN18-224 at rate 0.01, two steps (error feedback on): the GPU selection of every
    layer equals the oracle's stable-argsort selection on the same fp64 accumulator,
    and the residual keeps exactly the unselected entries."""
    import paper_2512_14628_b200 as H
    from oracle import hsadmm_oracle as O
    from paper_2512_14628_b200.synthetic import model_layers, synthetic_base

    layers = model_layers("rn18_224")

    class Solver:
        lr, momentum, weight_decay = 0.05, 0.9, 1e-4

    cluster = H.LocalCluster(H.Topology(1, 1))
    e = H.TopKSync(0, cluster, layers, Solver, 0.01)
    base = synthetic_base(layers, seed=7)
    e.init_from(base)
    gen = torch.Generator(device="cuda").manual_seed(11)
    for s in (1, 2):
        g = torch.randn(e.plan.arena, device="cuda", generator=gen) * 0.1
        g[:4096] = torch.round(g[:4096] * 8) / 8          # coarse values: many exact ties
        e.load_grads(g)
        acc = {n: (e.views("residual")[n].double() + (e.views("grad")[n].double()
                   + Solver.weight_decay * e.views("params")[n].double())).cpu().numpy()
               for n in e.names}      # residual + (grad + wd * params), baselines.py:128-129
        H.run_topk_local([e], s)
        sel = e.selections()
        res = e.views("residual")
        for n, (k, _) in zip(e.names, e.keep):
            flat = acc[n].ravel()
            want = O.topk_select(flat, O.topk_keep_count(0.01, flat.size))
            assert len(want) == k
            assert np.array_equal(cpu(sel[n]), want), (s, n)
            kept = np.zeros_like(flat)
            kept[want] = flat[want]
            np.testing.assert_array_equal(cpu(res[n]).ravel(), flat - kept)
