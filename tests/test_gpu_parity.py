"""GPU parity of the libhsx path against the reference's golden vectors and the
CPU oracle (oracle/hsadmm_oracle.py) on identical inputs.

Bars (north_star): masks, keep sets and compaction indices bit-exact; fp32
tensors within 1e-5 relative, measured per tensor as
    max|gpu - ref| / max(max|ref|, max|operands|)
(duals are differences, elementwise relative error is
meaningless where they cancel). Where the GPU and the reference evaluate the
same fp64 expression on the same fp32 inputs, the fp32 output must equal the
fp32 rounding of the reference value exactly.
"""

import numpy as np
import pytest
import torch

from oracle import hsadmm_oracle as O
from tests import golden_io as G

pytestmark = pytest.mark.gpu

TOL = 1e-5


def rel_err(got, ref, *operands):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = max([np.max(np.abs(ref)) if ref.size else 0.0] +
                [np.max(np.abs(np.asarray(o, dtype=np.float64))) for o in operands if np.size(o)] + [1e-30])
    return float(np.max(np.abs(got - ref)) / scale) if ref.size else 0.0


def cpu(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module", autouse=True)
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2512_14628_b200 import _lib

    _lib.load()
    torch.cuda.set_device(0)


# -- per-tensor API vs the reference's golden vectors --------------------------------


def test_projection_golden_single():
    import paper_2512_14628_b200 as H

    kinds = {"filter": H.ConstraintKind.FILTER_KEEP, "channel": H.ConstraintKind.CHANNEL_KEEP,
             "shape": H.ConstraintKind.SHAPE_KEEP}
    groups = {"filter": H.GroupBy.FILTER, "channel": H.GroupBy.CHANNEL, "shape": H.GroupBy.SHAPE_POSITION}
    singles, _ = G.projection_cases()
    for c in singles:
        t = torch.tensor(c["t"], dtype=torch.float32, device="cuda")
        out = H.project(t, H.SparsityConstraint(kinds[c["kind"]], keep_count=c["keep"]))
        assert np.array_equal(cpu(out).astype(np.float64), c["out"]), c["kind"]
        assert np.array_equal(cpu(H.extract_mask(out)), c["mask"])
        norms = cpu(H.group_norms(t, groups[c["kind"]]))
        np.testing.assert_allclose(norms, c["norms"], rtol=1e-13, atol=0)


def test_projection_golden_composite():
    import paper_2512_14628_b200 as H

    kinds = {"filter": H.ConstraintKind.FILTER_KEEP, "channel": H.ConstraintKind.CHANNEL_KEEP,
             "shape": H.ConstraintKind.SHAPE_KEEP}
    _, comps = G.projection_cases()
    for c in comps:
        t = torch.tensor(c["t"], dtype=torch.float32, device="cuda")
        cons = [H.SparsityConstraint(kinds[k], keep_count=kp) for k, kp in c["plan"]]
        out = H.project_composite(t, cons)
        assert np.array_equal(cpu(out).astype(np.float64), c["out"])


def test_projection_errors():
    import paper_2512_14628_b200 as H

    with pytest.raises(H.ShapeError):
        H.project(torch.ones((2, 3, 1, 1), device="cuda"),
                  H.SparsityConstraint(H.ConstraintKind.CHANNEL_KEEP, keep_count=4))
    with pytest.raises(H.ShapeError):
        H.project(torch.ones((2, 3), device="cuda"),
                  H.SparsityConstraint(H.ConstraintKind.CHANNEL_KEEP, keep_count=1))


def test_shrinkage_golden():
    import paper_2512_14628_b200 as H

    for c in G.shrinkage_cases():
        shape = c["t"].shape
        layer = H.LayerSpec("c", H.LayerKind.CONV, shape, prunable=True)
        keep = H.derive_keep_sets(torch.tensor(c["mask"], device="cuda"), layer)
        assert keep.k_out == tuple(c["k_out"]) and keep.k_in == tuple(c["k_in"])
        t = torch.tensor(c["t"], dtype=torch.float32, device="cuda")
        cb = H.compress(t, keep)
        assert np.array_equal(cpu(cb.data).astype(np.float64), c["compact"])
        restored = H.decompress(cb, keep, shape)
        assert np.array_equal(cpu(restored).astype(np.float64), c["restored"])
        rect = cpu(H.rectangle_mask(keep, shape))
        assert np.array_equal(cpu(restored) != 0, (c["t"] != 0) & rect)


def test_keep_set_cache_counts_and_seal():
    import paper_2512_14628_b200 as H

    conv = H.LayerSpec("conv", H.LayerKind.CONV, (3, 2, 3, 3), prunable=True)
    rng = np.random.default_rng(6)
    a = np.zeros(conv.shape, bool)
    a[np.ix_([0, 2], [1])] = True
    b = ~a
    cache = H.KeepSetCache()
    cache.get(conv, torch.tensor(a))
    assert (cache.derive_calls, cache.hits) == (1, 0)
    cache.get(conv, torch.tensor(a))
    assert (cache.derive_calls, cache.hits) == (1, 1)
    cache.get(conv, torch.tensor(b))
    assert (cache.derive_calls, cache.hits) == (2, 1)
    cache.seal()
    keep = cache.get(conv, torch.tensor(a))
    assert (cache.derive_calls, cache.hits) == (2, 2)
    assert keep == H.derive_keep_sets(torch.tensor(b), conv)
    empty = H.KeepSetCache()
    empty.seal()
    with pytest.raises(H.ProtocolError):
        empty.get(conv, torch.tensor(a))
    del rng


def test_node_candidate_is_fp32_rounding_of_reference():
    import paper_2512_14628_b200 as H

    for c in G.candidate_cases():
        s, z, v = (torch.tensor(x, dtype=torch.float32, device="cuda") for x in c["svz"])
        r1, r2, wd, m, p = c["par"]
        out = H.node_candidate(s, z, v, r1, r2, wd, int(m), int(p))
        assert np.array_equal(cpu(out), c["out"].astype(np.float32))
    with pytest.raises(H.ConfigError):
        H.node_candidate(torch.ones(2), torch.ones(2), torch.ones(2), 0.0, 0.0, 0.0, 1, 1)


def test_update_rules_per_tensor():
    import paper_2512_14628_b200 as H

    rng = np.random.default_rng(2)
    cand = rng.normal(size=(2, 2, 1, 1)).astype(np.float32)
    cons = [H.SparsityConstraint(H.ConstraintKind.FILTER_KEEP, keep_count=1)]
    z, m = H.update_node_consensus(torch.tensor(cand), cons, True, np.ones(cand.shape, bool))
    assert np.array_equal(cpu(z), cand) and m is None
    gm = rng.random(cand.shape) < 0.5
    z, _ = H.update_node_consensus(torch.tensor(cand), cons, True, gm)
    assert np.array_equal(cpu(z), cand * gm)
    with pytest.raises(H.ProtocolError):
        H.update_node_consensus(torch.tensor(cand), cons, True, None)
    z, m = H.update_node_consensus(torch.tensor(cand[:, :, 0, 0]), [], False, None)
    assert np.array_equal(cpu(z), cand[:, :, 0, 0]) and bool(cpu(m).all())
    th, zn, u = (rng.normal(size=(5, 7)).astype(np.float32) for _ in range(3))
    got = cpu(H.dual_update_intra(torch.tensor(th), torch.tensor(zn), torch.tensor(u)))
    assert np.array_equal(got, (u.astype(np.float64) + (th.astype(np.float64) - zn)).astype(np.float32))
    a = np.array([True, False, True, True])
    b = a.copy()
    b[0] = False
    assert H.mask_drift(torch.tensor(a), torch.tensor(b)) == 0.25


# -- end-to-end: the fused step against run_hierarchical goldens -------------------


def _e2e_engines(M, P, transport="nccl"):
    import paper_2512_14628_b200 as H

    ref = G.E2E(M, P)
    kinds = {"filter": H.ConstraintKind.FILTER_KEEP, "channel": H.ConstraintKind.CHANNEL_KEEP,
             "shape": H.ConstraintKind.SHAPE_KEEP}
    layers = [H.LayerSpec(n, H.LayerKind.CONV if k == "conv" else H.LayerKind.FULLY_CONNECTED, shape,
                          prunable=bool(c)) for n, k, shape, c in G.E2E_LAYERS]
    cons = {n: [H.SparsityConstraint(kinds[g], keep_rate=r) for g, r in c] for n, _, _, c in G.E2E_LAYERS if c}
    sched = H.PenaltySchedule.uniform(ref.names, G.E2E_RHO1, G.E2E_RHO2, adapt=False)
    settings = H.ConsensusSettings(iterations=ref.iters, t_freeze=ref.t_freeze, weight_decay=G.E2E_WD)
    cluster = H.LocalCluster(H.Topology(M, P))
    engines = [H.HSADMMSync(r, cluster, layers, cons, sched, settings, transport=transport)
               for r in range(ref.world)]
    for e in engines:
        e.init_from(ref.p0())
    return ref, cluster, engines


@pytest.mark.parametrize("transport", ["nccl", "peer"])
@pytest.mark.parametrize("M,P", G.E2E_TOPOLOGIES)
def test_end_to_end_against_reference_goldens(M, P, transport):
    """Both transports: collectives as requests (NCCL semantics) and the fused
    peer-memory kernels (K1 reads the node's theta+u, K7 averages the leaders'
    compact buffers) — emulated in one process on one GPU."""
    import paper_2512_14628_b200 as H

    ref, cluster, engines = _e2e_engines(M, P, transport)
    for k in range(1, ref.iters + 1):
        for e in engines:
            e.load(theta=ref.theta(k, e.rank))
        n_before = len(cluster.ledger.entries)
        H.run_local(engines, k)
        for e in engines:
            node = e.rank // P
            assert e.frozen == ref.frozen(k, node)
            for n, m in ref.masks(k, node).items():
                assert np.array_equal(cpu(e.mask_dict()[n]), m), (k, e.rank, n)
            th = ref.theta(k, e.rank)
            for n in ref.names:
                for key, want in (("z_node", ref.node_state("z_node", k, node)[n]),
                                  ("v", ref.node_state("v", k, node)[n]),
                                  ("z", ref.node_state("z", k, node)[n]),
                                  ("u", ref.u(k, e.rank)[n])):
                    got = cpu(e.views(key)[n])
                    err = rel_err(got, want, th[n])
                    assert err <= TOL, (k, e.rank, key, n, err)
            if e.is_leader:
                assert (e.cache_derive, e.cache_hits) == ref.cache(k, e.rank)
        zs = [x.to_dict() for x in cluster.ledger.entries[n_before:] if x.label.startswith("z_sync")]
        assert zs == ref.zsync(k)
    # followers hold the leader's z / v / z_node bit-for-bit
    for e in engines:
        lead = engines[e.leader_rank]
        for key in ("z_node", "v", "z"):
            assert torch.equal(getattr(e, key), getattr(lead, key))


@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_step_host_pipeline_against_reference_goldens(transport):
    """HSADMMSync.step_host: theta in from / z out to pinned host memory on copy
    streams, host bookkeeping deferred to the next call — every step's z_host and
    the settled freeze / cache / ledger state match run_hierarchical."""
    import paper_2512_14628_b200 as H

    ref, cluster, (e,) = _e2e_engines(1, 1, transport)
    dev = e.device
    thetas, outs, done = [], [], None
    for k in range(1, ref.iters + 1):
        t = e.plan.empty_arena(dev)
        e.plan.load_arena(t, ref.theta(k, 0))
        thetas.append(t.cpu().pin_memory())
        outs.append(torch.empty(e.plan.arena, dtype=torch.float32).pin_memory())
    for k in range(1, ref.iters + 1):
        done = e.step_host(k, thetas[k - 1], outs[k - 1])
    done.synchronize()
    e.settle()
    for k in range(1, ref.iters + 1):
        zk = e.plan.views(outs[k - 1])
        th = ref.theta(k, 0)
        for n in ref.names:
            err = rel_err(zk[n].numpy(), ref.node_state("z", k, 0)[n], th[n])
            assert err <= TOL, (k, n, err)
    k = ref.iters
    assert e.frozen == ref.frozen(k, 0)
    assert (e.cache_derive, e.cache_hits) == ref.cache(k, 0)
    for n, m in ref.masks(k, 0).items():
        assert np.array_equal(cpu(e.mask_dict()[n]), m), n
    zs = [x.to_dict() for x in cluster.ledger.entries if x.label.startswith("z_sync")]
    assert zs == [d for kk in range(1, k + 1) for d in ref.zsync(kk)]


@pytest.mark.parametrize("transport", ["nccl", "peer"])
def test_graph_step_against_reference_goldens(transport):
    """HSADMMSync.graph_step (captured CUDA graphs of the step, replayed with the
    host bookkeeping deferred) reproduces run_hierarchical across the freeze."""
    import paper_2512_14628_b200 as H

    ref, cluster, (e,) = _e2e_engines(1, 1, transport)
    for k in range(1, ref.iters + 1):
        e.load(theta=ref.theta(k, 0))
        e.graph_step(k)
        e.settle()
        assert e.frozen == ref.frozen(k, 0)
        for n, m in ref.masks(k, 0).items():
            assert np.array_equal(cpu(e.mask_dict()[n]), m), (k, n)
        th = ref.theta(k, 0)
        for n in ref.names:
            for key, want in (("z_node", ref.node_state("z_node", k, 0)[n]), ("v", ref.node_state("v", k, 0)[n]),
                              ("z", ref.node_state("z", k, 0)[n]), ("u", ref.u(k, 0)[n])):
                err = rel_err(cpu(e.views(key)[n]), want, th[n])
                assert err <= TOL, (k, key, n, err)
        assert (e.cache_derive, e.cache_hits) == ref.cache(k, 0)
    zs = [x.to_dict() for x in cluster.ledger.entries if x.label.startswith("z_sync")]
    assert zs == [d for kk in range(1, ref.iters + 1) for d in ref.zsync(kk)]
    assert len(e._graphs) >= 2   # dynamic (both mask buffers) and frozen graphs were replayed


# -- full-size stage-wise parity vs the oracle on identical inputs -------------------


@pytest.mark.parametrize("model,keep", [("rn18_224", 0.4), ("rn50_224", 0.4)])
def test_full_size_step_against_oracle(model, keep):
    """One dynamic then one frozen iteration of RN18/RN50 at 1x1 on the GPU and
    in the fp64 oracle from the same fp32 state: masks / keep sets bit-exact,
    z_node / u / v / z within 1e-5."""
    import paper_2512_14628_b200 as H
    from paper_2512_14628_b200.synthetic import channel_keep_constraints, model_layers, synthetic_rank_state

    layers = model_layers(model)
    cons = channel_keep_constraints(layers, keep)
    names = [ls.name for ls in layers]
    sched = H.PenaltySchedule.uniform(names, 1.5e-3, 1.5e-4, adapt=False)
    settings = H.ConsensusSettings(t_freeze=2, weight_decay=1e-4)
    cluster = H.LocalCluster(H.Topology(1, 1))
    eng = H.HSADMMSync(0, cluster, layers, cons, sched, settings)
    st = synthetic_rank_state(layers, 0, 1, seed=1)
    eng.load(**st)
    ocons = {n: [(O.CHANNEL, None, keep)] for n in cons}
    olayers = O.make_layers([(ls.name, ls.shape) for ls in layers], ocons)
    ost = O.init_rank_state(olayers, st["theta"], st["u"], st["z_node"], st["v"], st["z"])
    rho1 = {n: 1.5e-3 for n in names}
    rho2 = {n: 1.5e-4 for n in names}
    for k in (1, 2):
        # stage-wise: the oracle starts from the GPU's fp32 state of the previous iteration
        for key in ("u", "v", "z", "z_node"):
            setattr(ost, key, {n: cpu(t).astype(np.float64) for n, t in eng.views(key).items()})
        ost.masks = {n: cpu(m) for n, m in eng.mask_dict().items()}
        frozen_before = eng.frozen
        H.run_local([eng], k)
        O.cluster_sync(olayers, [ost], [st["theta"]], k, 1, 1, rho1, rho2, 1e-4, t_freeze=2)
        assert eng.frozen == ost.frozen
        gm = eng.mask_dict()
        for n in ost.masks:
            assert np.array_equal(cpu(gm[n]), ost.masks[n]), (k, n)
        for key in ("z_node", "u", "v", "z"):
            for n in names:
                err = rel_err(cpu(eng.views(key)[n]), getattr(ost, key)[n], st["theta"][n])
                assert err <= TOL, (k, key, n, err, frozen_before)
    ratio = eng.payload_elements / sum(ls.elements for ls in layers)
    assert 0.40 < ratio < 0.47     # leader bytes vs dense (0.428 / 0.450)


@pytest.mark.parametrize("zero_step", [1, 2])
def test_single_node_keep_sets_with_kept_zeros(zero_step):
    """One node derives the keep sets from the selection flags (the mask is the
    kept rectangle R x C) and K3 only checks for kept elements that are exactly
    zero. Here some kept elements (and a whole filter) are exactly zero, from
    iteration `zero_step` on, so the fixup re-derives those layers from their
    bits (and counts the drift of the next step from bits): masks, keep sets,
    payload sizes, state and drift against the oracle / numpy on the same inputs."""
    import paper_2512_14628_b200 as H
    from paper_2512_14628_b200.synthetic import channel_keep_constraints, model_layers, synthetic_rank_state

    layers = model_layers("rn18_cifar")
    keep = 0.5
    cons = channel_keep_constraints(layers, keep)
    names = [ls.name for ls in layers]
    sched = H.PenaltySchedule.uniform(names, 1.5e-3, 1.5e-4, adapt=False)
    settings = H.ConsensusSettings(t_freeze=100, drift_window=0, weight_decay=1e-4)
    eng = H.HSADMMSync(0, H.LocalCluster(H.Topology(1, 1)), layers, cons, sched, settings)
    st = synthetic_rank_state(layers, 0, 1, seed=4)
    convs = [ls for ls in layers if ls.kind is H.LayerKind.CONV and ls.shape[2] == 3]
    hit = [convs[1].name, convs[5].name]

    def zero_pattern(state):
        for n in hit:
            for key in ("theta", "u", "z_node", "v", "z"):
                t = state[key][n]
                t[3] = 0.0             # a whole filter: not in K_out
                t[:, :, 1, 1] = 0.0    # the centre tap of every channel: kept zeros

    if zero_step == 1:
        zero_pattern(st)
    eng.load(**st)
    ocons = {n: [(O.CHANNEL, None, keep)] for n in cons}
    olayers = O.make_layers([(ls.name, ls.shape) for ls in layers], ocons)
    ost = O.init_rank_state(olayers, st["theta"], st["u"], st["z_node"], st["v"], st["z"])
    rho = {n: 1.5e-3 for n in names}, {n: 1.5e-4 for n in names}
    prev = {n: np.ones(ls.shape, bool) for n, ls in zip(names, layers) if n in cons}
    for k in (1, 2, 3):
        if k == zero_step and k > 1:   # zeros appear later: the previous mask was a rectangle
            for n in hit:
                for key in ("theta", "u", "z_node", "v", "z"):
                    t = eng.views(key)[n]
                    t[3] = 0.0
                    t[:, :, 1, 1] = 0.0
            zs = {key: {n: cpu(t) for n, t in eng.views(key).items()} for key in ("theta",)}
            st["theta"] = {n: zs["theta"][n].copy() for n in names}
        for key in ("u", "v", "z", "z_node"):
            setattr(ost, key, {n: cpu(t).astype(np.float64) for n, t in eng.views(key).items()})
        ost.masks = {n: cpu(m) for n, m in eng.mask_dict().items()}
        H.run_local([eng], k)
        O.cluster_sync(olayers, [ost], [st["theta"]], k, 1, 1, rho[0], rho[1], 1e-4, t_freeze=100)
        gm = {n: cpu(m) for n, m in eng.mask_dict().items()}
        for n in ost.masks:
            assert np.array_equal(gm[n], ost.masks[n]), (k, n)
        if k >= zero_step:
            for n in hit:  # the pattern really made kept zeros / an empty filter
                assert not gm[n][3].any() and gm[n].any()
        for key in ("z_node", "u", "v", "z"):
            for n in names:
                err = rel_err(cpu(eng.views(key)[n]), getattr(ost, key)[n], st["theta"][n])
                assert err <= TOL, (k, key, n, err)
        # payload = sum over layers of |K_out| |K_in| kh kw from the union masks
        want = 0
        for ls in layers:
            if ls.name in gm:
                m = gm[ls.name]
                want += int(m.any(axis=(1, 2, 3)).sum()) * int(m.any(axis=(0, 2, 3)).sum()) * ls.shape[2] * ls.shape[3]
            else:
                want += ls.elements
        assert eng.payload_elements == want, k
        drift = max(float((gm[n] != prev[n]).mean()) for n in gm)
        assert abs(eng.drift_history[-1] - drift) < 1e-12, (k, eng.drift_history[-1], drift)
        prev = gm


def test_full_size_compaction_roundtrip_property():
    """decompress(compress(x)) == x * rectangle on every layer of RN50 (size-independent check)."""
    import paper_2512_14628_b200 as H
    from paper_2512_14628_b200.synthetic import channel_keep_constraints, model_layers, synthetic_base

    layers = model_layers("rn50_224")
    cons = channel_keep_constraints(layers, 0.3)
    names = [ls.name for ls in layers]
    sched = H.PenaltySchedule.uniform(names, 1.5e-3, 1.5e-4, adapt=False)
    eng = H.HSADMMSync(0, H.LocalCluster(H.Topology(1, 1)), layers, cons, sched, H.ConsensusSettings())
    base = synthetic_base(layers, seed=4)
    eng.load(theta=base, z=base, z_node=base)
    H.run_local([eng], 1)
    pl = eng.plan
    x = torch.randn(pl.arena, device="cuda")
    flat = torch.zeros(pl.arena, device="cuda")
    out = torch.zeros(pl.arena, device="cuda")
    pl.compact_dual(None, None, x, None, flat)
    pl.decompact_dual(flat, 1.0, None, None, out)
    pos_out, pos_in = pl.keep_positions(x.device)
    for i, ls in enumerate(layers):
        xv, ov = pl.view(x, i), pl.view(out, i)
        if i in pl.prunable:
            ko = pos_out[pl.keep_offset(i, 0):pl.keep_offset(i, 0) + ls.shape[0]] >= 0
            ki = pos_in[pl.keep_offset(i, 1):pl.keep_offset(i, 1) + ls.shape[1]] >= 0
            rect = ko.view(-1, 1, 1, 1) & ki.view(1, -1, 1, 1)
            assert torch.equal(ov, torch.where(rect, xv, torch.zeros_like(xv)))
        else:
            assert torch.equal(ov, xv)


def test_candidate_division_is_ieee():
    """K1 divides by gamma as q = RN(n*y), q' = fma(fma(-q, g, n), y, q) with y = RN(1/g)
    (Markstein). Check bit-equality with IEEE division for 4M numerators x 12 gammas,
    including the bench / golden gammas (wd/M + P*rho1 + rho2)."""
    from paper_2512_14628_b200 import _lib
    from paper_2512_14628_b200.plan import current_stream

    rng = np.random.default_rng(123)
    n = 1 << 22
    num = rng.normal(size=n) * np.exp2(rng.integers(-40, 40, size=n))
    num[:4096] = rng.integers(-(1 << 52), 1 << 52, size=4096) * 2.0 ** -30   # dense mantissas
    gammas = [1e-4 / M + P * 1.5e-3 + 1.5e-4 for M in (1, 2, 4) for P in (1, 2, 4)]
    gammas += [3.2e-3, float(np.nextafter(1.0, 2.0)), 0.3 / 7.0]
    d_num = torch.tensor(num, dtype=torch.float64, device="cuda")
    out = torch.empty_like(d_num)
    for g in gammas:
        _lib.call("hsx_selftest_division", d_num.data_ptr(), n, float(g), out.data_ptr(), current_stream())
        got = cpu(out)
        want = num / g
        bad = np.flatnonzero(got.view(np.int64) != want.view(np.int64))
        assert bad.size == 0, (g, num[bad[:5]], got[bad[:5]], want[bad[:5]])
