"""The reference's run entry point, end to end: ``run_hierarchical`` of this
package (paper_2512_14628_b200/hierarchical.py) reproduces the reference's own
``run_hierarchical`` fixtures (tests/golden/e2e_*.npz, made by
tests/golden/make_golden.py from /root/reference/pkg/src/admmprune/consensus.py:622-637).

Phase 1 is replaced exactly as the fixture generator replaced it in the
reference: ``hierarchical.batch_rng`` returns the (rank, k) key and
``hierarchical.proximal_sgd`` returns the recorded theta. Everything else is
the repo's drop-in path: ``Cluster(Topology(M, P))`` (a LocalCluster on one
GPU), the workload object, the constraint / schedule / settings objects, the
RankResult / ConsensusState / trace rows it returns and the cluster's
reference ledger.
"""

import numpy as np
import pytest
import torch

from tests import golden_io as G

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


class FixedWorkload:
    """make_golden._FixedWorkload: the golden's layers and initial parameters."""

    kind = "fixed"

    def __init__(self, layers, params0, world):
        self.layers = layers
        self.shards = [None] * world
        self._p0 = params0

    def init_params(self, rng):
        return {k: v.copy() for k, v in self._p0.items()}


def _setup(ref, adapt):
    import paper_2512_14628_b200 as H

    kinds = {"filter": H.ConstraintKind.FILTER_KEEP, "channel": H.ConstraintKind.CHANNEL_KEEP,
             "shape": H.ConstraintKind.SHAPE_KEEP}
    layers = [H.LayerSpec(n, H.LayerKind.CONV if k == "conv" else H.LayerKind.FULLY_CONNECTED, s,
                          prunable=bool(c)) for n, k, s, c in G.E2E_LAYERS]
    cons = {n: [H.SparsityConstraint(kinds[g], keep_rate=r) for g, r in c] for n, _, _, c in G.E2E_LAYERS if c}
    sched = H.PenaltySchedule.uniform(ref.names, G.E2E_RHO1, G.E2E_RHO2, adapt=adapt)
    return H, layers, cons, sched


def _run(H, ref, layers, cons, sched, iters, transport, monkeypatch):
    from paper_2512_14628_b200 import hierarchical as HI

    p0 = {n: a.astype(np.float32) for n, a in ref.p0().items()}
    monkeypatch.setattr(HI, "batch_rng", lambda seed, rank, k: (rank, k))
    monkeypatch.setattr(HI, "proximal_sgd",
                        lambda wl, shard, th, zn, u, rho1, solver, key: ref.theta(key[1], key[0]))
    settings = H.ConsensusSettings(iterations=iters, t_freeze=ref.t_freeze, stop_on_convergence=False,
                                   weight_decay=G.E2E_WD, seed=3)
    cluster = H.Cluster(H.Topology(ref.M, ref.P))
    assert isinstance(cluster, H.LocalCluster)
    res = H.run_hierarchical(cluster, FixedWorkload(layers, p0, ref.world), cons, sched, H.SolverConfig(),
                             settings, transport=transport)
    return cluster, res


@pytest.mark.parametrize("transport", ["nccl", "peer"])
@pytest.mark.parametrize("M,P", [(1, 1), (2, 2), (2, 4), (4, 2)])
def test_run_hierarchical_reproduces_reference(M, P, transport, monkeypatch):
    ref = G.E2E(M, P)
    H, layers, cons, sched = _setup(ref, adapt=False)
    for iters in (1, ref.t_freeze, ref.iters):     # dynamic, the freezing iteration, frozen
        cluster, res = _run(H, ref, layers, cons, sched, iters, transport, monkeypatch)
        assert sorted(res) == list(range(ref.world))
        for r, rr in res.items():
            node = r // P
            st = rr.state
            assert rr.rank == r and st.rank == r and st.iteration == iters and len(rr.trace) == iters
            assert st.frozen == ref.frozen(iters, node), (iters, r)
            for n, m in ref.masks(iters, node).items():
                assert st.masks[n].dtype == bool and np.array_equal(st.masks[n], m), (iters, r, n)
            th = ref.theta(iters, r)
            for key, want in (("z_node", ref.node_state("z_node", iters, node)),
                              ("v", ref.node_state("v", iters, node)),
                              ("z", ref.node_state("z", iters, node)), ("u", ref.u(iters, r))):
                for n in ref.names:
                    got = getattr(st, key)[n]
                    assert got.dtype == np.float64 and got.shape == want[n].shape
                    err = rel_err(got, want[n], th[n])
                    assert err <= TOL, (iters, r, key, n, err)
            assert (rr.cache_derive, rr.cache_hits) == ref.cache(iters, r), (iters, r)
            assert rr.converged_at is None
        zs = [e.to_dict() for e in cluster.ledger.entries if e.iteration == iters and e.label.startswith("z_sync")]
        assert zs == ref.zsync(iters)


@pytest.mark.parametrize("M,P", [(1, 1), (2, 2), (2, 4), (4, 2)])
def test_run_hierarchical_adaptive_trace_and_ledger(M, P, monkeypatch):
    """Phase 5 through the drop-in: rank 0's trace rows carry the reference's
    report and penalties per iteration, every rank its r_intra, the final schedule
    is the reference's, and the cluster's reference ledger equals
    run_hierarchical's ledger entry for entry."""
    ref = G.E2E(M, P, adapt=True)
    H, layers, cons, sched = _setup(ref, adapt=True)
    cluster, res = _run(H, ref, layers, cons, sched, ref.iters, "auto", monkeypatch)
    rows0 = res[0].trace
    for row in rows0:
        k = row["k"]
        r1, r2 = ref.rho(k)
        assert [row["rho1"][n] for n in ref.names] == list(r1), k
        assert [row["rho2"][n] for n in ref.names] == list(r2), k
        got = H.pack_report(row["report"], ref.names)
        want = ref.report(k)
        assert got[-1] == want[-1], k
        assert float((np.abs(got - want) / np.maximum(np.abs(want), 1e-30)).max()) <= TOL, k
    for r, rr in res.items():
        for row in rr.trace:
            got = np.array([row["r_intra"][n] for n in ref.names])
            want = ref.r_intra(row["k"], r)
            assert float((np.abs(got - want) / np.maximum(np.abs(want), 1e-30)).max()) <= TOL, (r, row["k"])
        s = rr.state.schedule
        assert [s.rho1[n] for n in ref.names] == list(ref.rho_final()[0])
        assert [s.rho2[n] for n in ref.names] == list(ref.rho_final()[1])
    for k in range(1, ref.iters + 1):
        got = [e.to_dict() for e in cluster.ref_ledger.entries if e.iteration == k]
        want = ref.ledger(k)
        key = lambda d: (d["group"], d["label"], d["op"])
        assert sorted(got, key=key) == sorted(want, key=key), k


def test_reference_helpers_on_device():
    """frobenius_norm against numpy fp64 on the same data (incl. a size that is not a multiple of a row)."""
    import paper_2512_14628_b200 as H

    rng = np.random.default_rng(3)
    t = rng.normal(size=(64, 32, 3, 3)).astype(np.float32)
    want = float(np.sqrt(np.sum(t.astype(np.float64) ** 2)))
    assert abs(H.frobenius_norm(torch.tensor(t, device="cuda")) - want) <= 1e-13 * want
    big = rng.normal(size=(3, 100_003)).astype(np.float32)
    want = float(np.sqrt(np.sum(big.astype(np.float64) ** 2)))
    assert abs(H.frobenius_norm(torch.tensor(big, device="cuda")) - want) <= 1e-12 * want
    assert H.frobenius_norm(torch.zeros(0, device="cuda")) == 0.0
