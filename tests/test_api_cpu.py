"""Host-side drop-in surface (no GPU): the reference-named objects and helpers
that do no device work — ``Cluster`` dispatch, ``Bucket.buffer`` /
``unbucketize`` copies, ``adapt_penalties`` / ``pack_report`` — against the
reference package itself when it is importable here (/root/reference, this
container only), else against fixed expectations."""

import os
import sys

import numpy as np
import pytest

REF_SRC = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import admmprune

    return admmprune


def test_cluster_dispatches_to_local_without_torch_distributed():
    import paper_2512_14628_b200 as H

    c = H.Cluster(H.Topology(2, 4))
    assert isinstance(c, H.LocalCluster) and isinstance(c, H.Cluster)
    assert c.intra_group(1).members == (4, 5, 6, 7)
    assert c.leader_group().members == (0, 4)
    assert c.global_group().members == tuple(range(8))
    c = H.Cluster(H.Topology(4, 2))
    assert c.leader_group().members == (0, 2, 4, 6)
    assert [c.intra_group(i).members for i in range(4)] == [(0, 1), (2, 3), (4, 5), (6, 7)]


def test_bucketize_buffer_and_unbucketize_copies(ref):
    from admmprune import transport as RT

    import paper_2512_14628_b200 as H

    rng = np.random.default_rng(0)
    payloads = [(f"p{i}", rng.normal(size=n)) for i, n in enumerate([5, 3, 9, 2, 7])]
    mine = H.bucketize(payloads, cap_bytes=40)
    theirs = RT.bucketize(payloads, cap_bytes=40)
    assert len(mine) == len(theirs)
    for a, b in zip(mine, theirs):
        assert a.layout == b.layout and a.detail == b.detail
        assert a.buffer.dtype == b.buffer.dtype and np.array_equal(a.buffer, b.buffer)
        got, want = H.unbucketize(a, a.buffer), RT.unbucketize(b, b.buffer)
        assert list(got) == list(want)
        for n in got:
            assert np.array_equal(got[n], want[n])
            assert not np.shares_memory(got[n], a.buffer)      # copies, like the reference
    with pytest.raises(H.ShapeError):
        H.unbucketize(mine[0], np.zeros(mine[0].elements + 1))


def _report(mod, names, rng):
    layers = {n: mod.LayerResiduals(*(float(x) for x in rng.choice([1e-6, 1e-3, 0.1, 1.0, 10.0], size=8)))
              for n in names}
    return mod.ResidualReport(layers, 0.1, 0.2, 0.3, 0.4, bool(rng.integers(2)))


def test_adapt_penalties_and_pack_report_match_reference(ref):
    from admmprune import consensus as RC

    import paper_2512_14628_b200 as H
    from paper_2512_14628_b200 import consensus as C

    names = [f"l{i}" for i in range(40)]
    rng = np.random.default_rng(5)
    for trial in range(20):
        state = rng.bit_generator.state
        rep_ref = _report(RC, names, rng)
        rng.bit_generator.state = state
        rep = _report(C, names, rng)
        r1 = {n: float(x) for n, x in zip(names, rng.choice([1.5e-3, 0.5, 6.0, 10.0], size=len(names)))}
        r2 = {n: float(x) for n, x in zip(names, rng.choice([0.0, 1.5e-4, 0.5, 8.0], size=len(names)))}
        s_ref = RC.PenaltySchedule(rho1=r1, rho2=r2)
        s = H.PenaltySchedule(rho1=r1, rho2=r2)
        a_ref = RC.adapt_penalties(rep_ref, s_ref)
        a = H.adapt_penalties(rep, s)
        assert a[0].rho1 == a_ref[0].rho1 and a[0].rho2 == a_ref[0].rho2
        assert a[1] == a_ref[1] and a[2] == a_ref[2]
        assert np.array_equal(H.pack_report(rep, names), RC.pack_report(rep_ref, names))
        back = C.unpack_report(H.pack_report(rep, names), names)
        assert back == rep


def test_run_hierarchical_signature_matches_reference(ref):
    import inspect

    from admmprune import consensus as RC

    import paper_2512_14628_b200 as H

    for fn in ("run_hierarchical", "hierarchical_program"):
        mine = list(inspect.signature(getattr(H, fn)).parameters)
        theirs = list(inspect.signature(getattr(RC, fn)).parameters)
        assert mine[:len(theirs)] == theirs, fn
    for cls in ("ConsensusState", "RankResult"):
        import dataclasses

        assert ([f.name for f in dataclasses.fields(getattr(H, cls))]
                == [f.name for f in dataclasses.fields(getattr(RC, cls))]), cls


def test_rooted_barrier_and_rank_concurrency_flags():
    """A one-sided (rooted) barrier is an ordinary rendezvous under the in-process
    scheduler; only a cluster whose ranks run concurrently (one process per GPU)
    may take the split two-rank K1, whose selection waits for the peer's kernel."""
    import paper_2512_14628_b200 as H
    from paper_2512_14628_b200.transport import Barrier, DistCluster

    c = H.LocalCluster(H.Topology(2, 2))
    order = []

    def prog(rank):
        g = c.intra_group(rank // 2)
        order.append(("before", rank))
        yield Barrier(g, "zhat_bcast", 1, root=g.members[0])
        order.append(("after", rank))
        return rank

    res = c.run({r: prog(r) for r in range(4)})
    assert res == {r: r for r in range(4)}
    # nobody passes the barrier before every member of its group reached it
    for r in range(4):
        mates = [m for m in range(4) if m // 2 == r // 2]
        assert all(order.index(("before", m)) < order.index(("after", r)) for m in mates)
    assert Barrier(c.intra_group(0), "m_bcast", 1).root is None
    assert H.LocalCluster.concurrent_ranks is False and DistCluster.concurrent_ranks is True
