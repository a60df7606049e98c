"""C-ABI boundary checks that need no GPU: the library loads, exports every
entry point include/hsx.h declares with the ctypes signatures, and host-side
layout logic (bucketize, topology, layer tables) matches the reference."""

import os
import re
import subprocess

import pytest

from tests import golden_io as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hsx.h")
LIB = os.path.join(ROOT, "paper_2512_14628_b200", "libhsx.so")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", ROOT], check=True, capture_output=True)
    from paper_2512_14628_b200 import _lib

    return _lib.load()


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hsx_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "hsx_candidate" in syms and "hsx_compact_dual" in syms and "hsx_decompact_dual" in syms
    assert len(syms) >= 30


def test_library_exports_every_declared_symbol(lib):
    from paper_2512_14628_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (hsx_[a-z0-9_]+)$", out, re.M))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert set(_lib.SIGNATURES) == set(declared_symbols())
    for s in declared_symbols():
        assert getattr(lib, s) is not None


def test_abi_version_and_no_cuda_work_on_load(lib):
    assert lib.hsx_abi_version() == 1
    assert lib.hsx_launch_count() == 0


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_bucketize_layout_matches_reference_goldens():
    from paper_2512_14628_b200.transport import bucketize

    for c in G.bucketize_cases():
        got = bucketize([(f"t{i}", s) for i, s in enumerate(c["sizes"])], cap_bytes=c["cap"])
        assert [[list(e) for e in b.layout] for b in got] == c["layout"]
        starts = [b.start for b in got]
        assert starts == [sum(b.elements for b in got[:i]) for i in range(len(got))]


def test_topology_and_groups():
    from paper_2512_14628_b200.errors import ShapeError
    from paper_2512_14628_b200.transport import GroupScope, LocalCluster, Topology

    topo = Topology(3, 4)  # reference tests/test_transport.py:26-43
    assert topo.world_size == 12 and topo.node_of(7) == 1 and topo.local_rank(7) == 3
    assert topo.leaders == (0, 4, 8) and topo.is_leader(4) and not topo.is_leader(5)
    with pytest.raises(ShapeError):
        Topology(0, 2)
    c = LocalCluster(Topology(2, 3))
    assert c.intra_group(1).members == (3, 4, 5)
    assert c.leader_group().members == (0, 3)
    assert c.global_group().members == tuple(range(6))
    assert c.intra_group(0).scope is GroupScope.INTRA and c.leader_group().scope is GroupScope.INTER
    assert Topology.parse("2x4") == Topology(2, 4)


def test_resnet_parameter_counts():
    from paper_2512_14628_b200.synthetic import model_layers

    counts = {m: sum(ls.elements for ls in model_layers(m)) for m in
              ("rn18_cifar", "rn18_224", "rn50_224", "rn152_224")}
    assert counts == {"rn18_cifar": 11_173_962, "rn18_224": 11_689_512,
                      "rn50_224": 25_557_032, "rn152_224": 60_192_808}


def test_constraint_resolution_matches_reference_rules():
    from paper_2512_14628_b200.errors import ShapeError
    from paper_2512_14628_b200.sparsity import ConstraintKind, SparsityConstraint, resolve_plan

    c = SparsityConstraint(ConstraintKind.CHANNEL_KEEP, keep_rate=0.5)
    assert c.resolve(3) == 2 and c.resolve(4) == 2
    assert SparsityConstraint(ConstraintKind.FILTER_KEEP, keep_rate=0.01).resolve(8) == 1
    assert SparsityConstraint(ConstraintKind.CHANNEL_KEEP, keep_rate=0.07).resolve(100) == 8
    for bad in (dict(), dict(keep_count=1, keep_rate=0.5), dict(keep_rate=1.5), dict(keep_count=0)):
        with pytest.raises(ShapeError):
            SparsityConstraint(ConstraintKind.FILTER_KEEP, **bad)
    with pytest.raises(ShapeError):
        resolve_plan((2, 2, 1, 1), [SparsityConstraint(ConstraintKind.FILTER_KEEP, keep_count=1),
                                    SparsityConstraint(ConstraintKind.FILTER_KEEP, keep_count=2)])
    with pytest.raises(ShapeError):
        resolve_plan((2, 3, 1, 1), [SparsityConstraint(ConstraintKind.CHANNEL_KEEP, keep_count=4)])


def test_freeze_check_and_schedule():
    from paper_2512_14628_b200.consensus import PenaltySchedule, freeze_check
    from paper_2512_14628_b200.errors import ConfigError

    assert freeze_check(10, 10, [], 3) and not freeze_check(3, 10, [0.0, 0.0], 3)
    assert freeze_check(4, 10, [0.5, 0.0, 0.0, 0.0], 3)
    with pytest.raises(ConfigError):
        PenaltySchedule({"x": 0.0}, {"x": 0.1})
    PenaltySchedule({"x": 1.0}, {"x": 0.0})
