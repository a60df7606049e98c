"""Multi-process host logic of the hierarchical transport on CPU (gloo).

DistCluster wires torch.distributed sub-groups for every intra group and the
leader group (reference Cluster.__init__, transport.py:305-318) and executes
the rank programs' collective requests. These tests run world sizes 2 and 4
(topologies 1x2, 2x1, 2x2) on the gloo backend with CPU tensors and compare
every collective with the reference semantics: SUM / AVG folds
(transport.py:453-462), broadcast copies and (g-1)x ledger bytes
(:418-435), all-gather in member order (:437-451).
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, M, P, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_14628_b200.transport import (AllGather, AllReduce, Broadcast, DistCluster,
                                                     ReduceOp, Topology)

        topo = Topology(M, P)
        cl = DistCluster(topo)
        node = topo.node_of(rank)
        intra = cl.intra_group(node)
        leaders = cl.leader_group()
        leader = topo.leader_of(node)

        def program():
            res = {}
            x = torch.arange(6, dtype=torch.float32) + 10.0 * rank
            res["sum"] = (yield AllReduce(intra, x, ReduceOp.SUM, "theta_u", 1)).clone()
            if rank == leader:
                bits = torch.tensor([1 << rank, rank], dtype=torch.int32)
                out = torch.zeros((M, 2), dtype=torch.int32)
                res["gather"] = (yield AllGather(leaders, bits, out, "mask_sync", 1)).clone()
                y = torch.full((5,), float(rank))
                res["avg"] = (yield AllReduce(leaders, y, ReduceOp.AVG, "z_sync/b0", 1,
                                              detail=(("a", 5),))).clone()
                buf = res["avg"].clone()
            else:
                buf = torch.zeros(5)
            res["bcast"] = (yield Broadcast(intra, leader, buf, "zhat_bcast", 1)).clone()
            return res

        res = cl.run_rank(program())
        ledger = [e.to_dict() for e in cl.ledger.entries]
        out_q.put((rank, {k: v.tolist() for k, v in res.items()}, ledger))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M,P", [(1, 2), (2, 1), (2, 2)])
def test_dist_cluster_collectives_gloo(M, P):
    world = M * P
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, P, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(world):
        rank, res, ledger = q.get(timeout=120)
        results[rank] = (res, ledger)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    leaders = [i * P for i in range(M)]
    for rank, (res, ledger) in results.items():
        node = rank // P
        members = range(node * P, (node + 1) * P)
        want_sum = [sum(i + 10.0 * r for r in members) for i in range(6)]
        assert res["sum"] == want_sum
        want_avg = [sum(float(r) for r in leaders) / M] * 5
        assert res["bcast"] == want_avg                      # leader's average reached followers
        if rank in leaders:
            assert res["avg"] == want_avg
            assert res["gather"] == [[1 << r, r] for r in leaders]
        labels = [e["label"] for e in ledger]
        assert labels[0] == "theta_u" and ledger[0]["bytes"] == 24 and ledger[0]["members"] == P
        if rank in leaders:
            zs = [e for e in ledger if e["label"] == "z_sync/b0"][0]
            assert zs == {"iter": 1, "group": "leaders", "scope": "inter", "op": "allreduce_avg",
                          "elements": 5, "bytes": 20, "members": M, "label": "z_sync/b0",
                          "detail": {"a": 5}}
        bc = [e for e in ledger if e["label"] == "zhat_bcast"]
        if P > 1:
            assert bc[0]["bytes"] == 20 * (P - 1)
        else:
            assert not bc                                  # single-member broadcasts are not logged


def test_local_cluster_matches_reference_protocol_errors():
    """LocalCluster enforces the reference's protocol checks (transport.py:378-411)."""
    from paper_2512_14628_b200.errors import ProtocolError
    from paper_2512_14628_b200.transport import AllReduce, LocalCluster, ReduceOp, Topology

    cl = LocalCluster(Topology(1, 2))
    g = cl.intra_group(0)

    def prog(tag, n):
        yield AllReduce(g, torch.ones(n), ReduceOp.SUM, tag, 1)

    with pytest.raises(ProtocolError, match="mismatched"):
        cl.run({0: prog("a", 2), 1: prog("b", 2)})
    with pytest.raises(ProtocolError, match="shapes disagree"):
        cl.run({0: prog("a", 2), 1: prog("a", 3)})

    def early():
        return
        yield  # pragma: no cover

    with pytest.raises(ProtocolError, match="deadlock"):
        cl.run({0: prog("a", 2), 1: early()})
    cl2 = LocalCluster(Topology(2, 2))

    def outsider():
        yield AllReduce(cl2.intra_group(0), torch.ones(1), ReduceOp.SUM, "s", 1)

    with pytest.raises(ProtocolError, match="not a member"):
        cl2.run({2: outsider()})
    out = cl.run({r: prog("a", 3) for r in (0, 1)})
    assert out == {0: None, 1: None}
    assert cl.ledger.entries[-1].bytes == 12
