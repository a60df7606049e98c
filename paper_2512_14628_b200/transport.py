"""Hierarchical process groups, collective requests and the two drivers.

Mirrors the reference's transport surface
(/root/reference/pkg/src/admmprune/transport.py): ``Topology`` (:36-69),
``GroupScope`` / ``ProcessGroup`` (:72-86), ``ReduceOp`` (:89-92), collective
request objects (:95-120), ``LedgerEntry`` / ``CommLedger`` (:126-188),
``bucketize`` / ``unbucketize`` (:227-290). A rank program is a generator that
yields collective requests and is resumed with the result, exactly like the
reference's ``Cluster.run`` protocol (:331-376) — but payloads are CUDA
tensors and there are two drivers:

* ``DistCluster``: one process per GPU under ``torchrun``; every request is
  executed with ``torch.distributed`` on NCCL sub-communicators built with
  ``new_group`` (intra groups, the leader group, global) — the B200 box
  emulates PruneX's hierarchy: intra = NVLink all-reduce among a node's
  ranks, inter = the leader-only all-reduce of compact buffers.
* ``LocalCluster``: all ranks of a topology inside one process (one GPU),
  collectives completed once every member has posted, folding in member order
  like the reference's deterministic scheduler. Used to check multi-rank
  parity on a single GPU and by the CPU (gloo-free) protocol tests.

Requests are in-place: an ``AllReduce`` / ``Broadcast`` writes its result
into ``payload`` on every member (NCCL semantics) and the program is resumed
with that same tensor.
"""

from __future__ import annotations

import enum
import logging
import numbers
from dataclasses import dataclass, field
from typing import Any, Generator, Mapping

from .errors import ProtocolError, ShapeError

log = logging.getLogger(__name__)

ELEMENT_BYTES = 4                      # fp32 wire accounting (reference transport.py:32)
BUCKET_CAP_BYTES = 32 * 1024 * 1024    # reference transport.py:33


@dataclass(frozen=True)
class Topology:
    """``num_nodes`` x ``accels_per_node`` ranks; local rank 0 leads its node."""

    num_nodes: int
    accels_per_node: int

    def __post_init__(self):
        if self.num_nodes < 1 or self.accels_per_node < 1:
            raise ShapeError("topology dimensions must be positive")

    @property
    def world_size(self) -> int:
        return self.num_nodes * self.accels_per_node

    def node_of(self, rank: int) -> int:
        return rank // self.accels_per_node

    def local_rank(self, rank: int) -> int:
        return rank % self.accels_per_node

    def leader_of(self, node: int) -> int:
        return node * self.accels_per_node

    def is_leader(self, rank: int) -> bool:
        return self.local_rank(rank) == 0

    @property
    def leaders(self) -> tuple[int, ...]:
        return tuple(self.leader_of(i) for i in range(self.num_nodes))

    @classmethod
    def parse(cls, text: str) -> "Topology":
        """'2x4' -> Topology(2, 4)."""
        m, p = text.lower().split("x")
        return cls(int(m), int(p))


class GroupScope(enum.Enum):
    INTRA = "intra"
    INTER = "inter"
    GLOBAL = "global"


@dataclass(frozen=True)
class ProcessGroup:
    id: str
    members: tuple[int, ...]
    scope: GroupScope

    def __post_init__(self):
        if not self.members or len(set(self.members)) != len(self.members):
            raise ShapeError(f"group {self.id}: members must be non-empty and unique")


class ReduceOp(enum.Enum):
    SUM = "sum"
    AVG = "avg"
    BITWISE_OR = "bor"


def hierarchy_groups(topology: Topology):
    """(intra groups by node, leader group, global group) — reference Cluster.__init__ :305-318."""
    P = topology.accels_per_node
    intra = {i: ProcessGroup(f"intra{i}", tuple(range(i * P, (i + 1) * P)), GroupScope.INTRA)
             for i in range(topology.num_nodes)}
    leaders = ProcessGroup("leaders", topology.leaders, GroupScope.INTER)
    world = ProcessGroup("global", tuple(range(topology.world_size)), GroupScope.GLOBAL)
    return intra, leaders, world


# -- collective requests -------------------------------------------------------


@dataclass
class AllReduce:
    group: ProcessGroup
    payload: Any            # tensor, reduced in place
    op: ReduceOp
    tag: str
    iteration: int
    detail: tuple | None = None
    # several logical collectives carried by this one call (the leader average's
    # buckets over the contiguous flat buffer): ledger entries (tag, elements, detail)
    parts: tuple | None = None


@dataclass
class Broadcast:
    group: ProcessGroup
    root: int
    payload: Any            # tensor: sent by root, received in place by the others
    tag: str
    iteration: int


@dataclass
class AllGather:
    group: ProcessGroup
    payload: Any            # local tensor
    out: Any                # (members, *payload.shape) output, member order
    tag: str
    iteration: int


@dataclass
class Barrier:
    """Every member reaches this point before any continues (device-side barrier over
    NVLink signal pads under DistCluster; scheduler rendezvous under LocalCluster).
    Orders the producers of shared (peer-mapped) buffers before their readers.

    ``root`` given: a one-sided hand-off — the root only publishes (it does not wait
    for the others), every other member waits for the root. For a buffer the root
    produces and the others read, when a later two-sided barrier already orders the
    root's next write after their reads."""

    group: ProcessGroup
    tag: str
    iteration: int
    root: int | None = None


class SharedBuffer:
    """A buffer every member of a group allocates; ``peer_ptrs()`` are the device
    pointers of all members' copies in member order (torch symmetric memory under
    DistCluster; the other in-process ranks' tensors under LocalCluster)."""

    def __init__(self, tensor, resolve):
        self.tensor = tensor
        self._resolve = resolve

    def peer_ptrs(self) -> list[int]:
        return self._resolve()


RankProgram = Generator[Any, Any, Any]


# -- ledger ---------------------------------------------------------------------


@dataclass(frozen=True)
class LedgerEntry:
    iteration: int
    group: str
    scope: str
    op: str
    elements: int
    bytes: int
    members: int
    label: str
    detail: tuple | None = None

    def to_dict(self) -> dict:
        d = dict(iter=self.iteration, group=self.group, scope=self.scope, op=self.op,
                 elements=self.elements, bytes=self.bytes, members=self.members, label=self.label)
        if self.detail is not None:
            d["detail"] = {name: n for name, n in self.detail}
        return d


class DeferredLedger:
    """A ledger whose per-iteration entries are produced on demand: the step
    records one closure (no per-entry host work while the GPU waits for the next
    launch); ``entries`` materializes them in order."""

    def __init__(self):
        self._items = []
        self._done: list[LedgerEntry] = []

    def append(self, entry: LedgerEntry) -> None:
        self._items.append(entry)

    def defer(self, thunk) -> None:
        self._items.append(thunk)

    @property
    def entries(self) -> list[LedgerEntry]:
        if self._items:
            for it in self._items:
                if callable(it):
                    self._done.extend(it())
                else:
                    self._done.append(it)
            self._items = []
        return self._done

    def to_jsonl(self, path) -> None:
        import json

        with open(path, "w", encoding="utf-8") as fh:
            for e in self.entries:
                fh.write(json.dumps(e.to_dict(), sort_keys=True) + "\n")


class CommLedger:
    """Append-only record of completed collectives (reference transport.py:154-188).

    ``bytes`` are the per-rank payload bytes actually moved: fp32 payloads at
    4 B/element like the reference; packed mask bits at their real size.
    """

    def __init__(self):
        self.entries: list[LedgerEntry] = []

    def append(self, entry: LedgerEntry) -> None:
        if entry.bytes <= 0:
            raise ShapeError("ledger entries must carry positive byte counts")
        self.entries.append(entry)

    def total_bytes(self, scope=None, iteration=None, label_prefix=None) -> int:
        sv = scope.value if isinstance(scope, GroupScope) else scope
        return sum(e.bytes for e in self.entries
                   if (sv is None or e.scope == sv) and (iteration is None or e.iteration == iteration)
                   and (label_prefix is None or e.label.startswith(label_prefix)))

    def to_jsonl(self, path) -> None:
        import json

        with open(path, "w", encoding="utf-8") as fh:
            for e in self.entries:
                fh.write(json.dumps(e.to_dict(), sort_keys=True) + "\n")


def _ledger(ledger, req, members: int, nbytes: int, op: str):
    if ledger is None or nbytes <= 0:
        return
    parts = getattr(req, "parts", None)
    if parts:   # one call carrying several logical collectives: one entry each
        esize = int(req.payload.element_size())
        for tag, n, detail in parts:
            ledger.append(LedgerEntry(req.iteration, req.group.id, req.group.scope.value, op, int(n),
                                      int(n) * esize, members, tag, detail))
        return
    n = int(req.payload.numel())
    ledger.append(LedgerEntry(req.iteration, req.group.id, req.group.scope.value, op, n, nbytes,
                              members, req.tag, getattr(req, "detail", None)))


def _payload_bytes(t) -> int:
    return int(t.numel()) * int(t.element_size())


# -- bucketing (layout only: the payload already lives in one flat buffer) --------


@dataclass
class Bucket:
    """A contiguous slice of the flat compact buffer (reference transport.py:227-236).

    ``start`` is the slice's first element in the flat buffer the compaction
    kernel wrote (the sync step's buckets carry only the layout, no copy);
    ``buffer`` holds the concatenated payloads when :func:`bucketize` was given
    arrays / tensors, like the reference's ``Bucket.buffer``.
    """

    start: int
    layout: tuple[tuple[str, int, int], ...]  # (name, offset inside bucket, elements)
    buffer: Any = None

    @property
    def elements(self) -> int:
        return sum(e for _, _, e in self.layout)

    @property
    def detail(self) -> tuple[tuple[str, int], ...]:
        return tuple((name, e) for name, _, e in self.layout)


def _concat(arrays):
    """The reference's bucket buffer: the payloads raveled and concatenated, in a
    new buffer (torch on the payloads' device, else float64 numpy)."""
    import numpy as np

    if any(_is_tensor(a) for a in arrays):
        import torch

        dev = next(a.device for a in arrays if _is_tensor(a))
        return torch.cat([torch.as_tensor(a, device=dev).reshape(-1) for a in arrays])
    return np.ascontiguousarray(np.concatenate([np.asarray(a).ravel() for a in arrays]), dtype=np.float64)


def _is_tensor(x) -> bool:
    return type(x).__module__.startswith("torch")


def bucketize(payloads, cap_bytes: int = BUCKET_CAP_BYTES) -> list[Bucket]:
    """Greedy <= ``cap_bytes`` buckets over (name, elements) in order, never split.

    Same grouping rule as the reference (transport.py:239-280): a payload
    larger than the cap gets its own bucket with a warning. ``payloads`` may
    hold element counts (layout only: the sync step's payload already lives in
    one flat buffer, so a bucket is a [start, start+n) slice of what the
    compaction kernel wrote) or arrays / tensors (the bucket's ``buffer`` is
    their concatenation, as in the reference).
    """
    sizes, arrays = [], {}
    for i, (name, x) in enumerate(payloads):
        if isinstance(x, numbers.Integral):
            sizes.append((name, int(x)))
        else:
            n = int(x.numel()) if _is_tensor(x) else int(x.size)
            sizes.append((name, n))
            arrays[i] = x
    buckets: list[Bucket] = []
    cur: list[tuple[int, str, int]] = []
    cur_bytes = 0
    start = 0

    def close():
        nonlocal cur, cur_bytes, start
        if cur:
            lay, off = [], 0
            for _, name, n in cur:
                lay.append((name, off, n))
                off += n
            buf = _concat([arrays[i] for i, _, _ in cur]) if arrays else None
            buckets.append(Bucket(start, tuple(lay), buf))
            start += off
        cur, cur_bytes = [], 0

    for i, (name, n) in enumerate(sizes):
        nbytes = n * ELEMENT_BYTES
        if nbytes > cap_bytes:
            close()
            log.warning("payload %s (%d bytes) exceeds bucket cap %d; using oversized bucket",
                        name, nbytes, cap_bytes)
            cur, cur_bytes = [(i, name, n)], nbytes
            close()
            continue
        if cur_bytes + nbytes > cap_bytes:
            close()
        cur.append((i, name, n))
        cur_bytes += nbytes
    close()
    return buckets


def unbucketize(bucket: Bucket, buffer) -> dict:
    """Copies of the bucket's named payloads out of a (reduced) flat ``buffer``
    (reference transport.py:283-290: fresh arrays, never views)."""
    n = int(buffer.numel()) if _is_tensor(buffer) else int(buffer.size)
    if n != bucket.elements:
        raise ShapeError(f"buffer size {n} does not match bucket {bucket.elements}")
    if _is_tensor(buffer):
        return {name: buffer[off:off + e].clone() for name, off, e in bucket.layout}
    return {name: buffer[off:off + e].copy() for name, off, e in bucket.layout}


# -- drivers --------------------------------------------------------------------


def _validate(rank: int, req) -> None:
    if not isinstance(req, (AllReduce, Broadcast, AllGather, Barrier)):
        raise ProtocolError(f"rank {rank} yielded a non-collective object: {req!r}")
    if rank not in req.group.members:
        raise ProtocolError(f"rank {rank} is not a member of group {req.group.id}")
    if isinstance(req, Broadcast) and req.root not in req.group.members:
        raise ProtocolError(f"broadcast root {req.root} is not in group {req.group.id}")
    if isinstance(req, AllReduce) and req.op is ReduceOp.BITWISE_OR:
        raise ProtocolError("BITWISE_OR is carried as an AllGather of packed bits + OR kernel")


def _dist_spans(topology) -> bool:
    try:
        import torch.distributed as dist
    except Exception:
        return False
    return (dist.is_available() and dist.is_initialized() and topology is not None
            and dist.get_world_size() == topology.world_size)


class Cluster:
    """The reference's ``Cluster(topology)`` (transport.py:302-376): topology, the
    intra / leader / global groups, ``run(programs)`` and the ledger.

    ``Cluster(topology)`` constructs a :class:`DistCluster` (this process is one
    rank, collectives on NCCL sub-communicators) when ``torch.distributed`` is
    initialized over exactly ``topology.world_size`` ranks, else a
    :class:`LocalCluster` (every rank in this process on one GPU, the
    reference's deterministic scheduler).
    """

    def __new__(cls, topology=None, *args, **kwargs):
        if cls is Cluster:
            cls = DistCluster if _dist_spans(topology) else LocalCluster
        return super().__new__(cls)


class LocalCluster(Cluster):
    """All ranks of a topology in one process; deterministic round-based scheduler."""

    # the ranks' kernels run one after another on one device: no kernel may wait for
    # another rank's concurrently running kernel
    concurrent_ranks = False

    def __init__(self, topology: Topology, latency=None):
        self.topology = topology
        self.ledger = CommLedger()
        self.ref_ledger = DeferredLedger()   # the reference's logical entries (HSADMMSync._log_reference)
        self._intra, self._leaders, self._global = hierarchy_groups(topology)
        self._shared = {}

    def intra_group(self, node: int) -> ProcessGroup:
        return self._intra[node]

    def leader_group(self) -> ProcessGroup:
        return self._leaders

    def global_group(self) -> ProcessGroup:
        return self._global

    supports_peer = True  # all ranks share one device: "peer" pointers are the other ranks' tensors
    shared_ledger = True

    def shared(self, rank: int, group: ProcessGroup, key: str, numel: int, dtype, device) -> SharedBuffer:
        import torch

        t = torch.zeros(max(int(numel), 1), dtype=dtype, device=device)
        self._shared[(group.id, key, rank)] = t

        def resolve():
            return [self._shared[(group.id, key, r)].data_ptr() for r in group.members]

        return SharedBuffer(t, resolve)

    def log(self, entry: LedgerEntry) -> None:
        self.ledger.append(entry)

    def run(self, programs: Mapping[int, RankProgram]) -> dict[int, Any]:
        gens = dict(programs)
        started, results = set(), {}
        inbox: dict[int, Any] = {}
        blocked: dict[int, Any] = {}
        pending: dict[str, dict[int, Any]] = {}
        while len(results) < len(gens):
            progressed = False
            for rank in sorted(gens):
                if rank in results or rank in blocked:
                    continue
                try:
                    req = next(gens[rank]) if rank not in started else gens[rank].send(inbox.pop(rank, None))
                    started.add(rank)
                except StopIteration as stop:
                    started.add(rank)
                    results[rank] = stop.value
                    progressed = True
                    continue
                _validate(rank, req)
                blocked[rank] = req
                pending.setdefault(req.group.id, {})[rank] = req
                progressed = True
            for gid in sorted(pending):
                posted = pending[gid]
                group = next(iter(posted.values())).group
                if set(posted) != set(group.members):
                    continue
                for r, value in self._complete(group, posted).items():
                    inbox[r] = value
                    del blocked[r]
                del pending[gid]
                progressed = True
            if not progressed:
                raise ProtocolError(f"collective deadlock; blocked ranks: "
                                    f"{ {r: q.tag for r, q in blocked.items()} }")
        return results

    def _complete(self, group: ProcessGroup, posted: dict[int, Any]) -> dict[int, Any]:
        reqs = [posted[r] for r in group.members]
        first = reqs[0]
        for q in reqs[1:]:
            if type(q) is not type(first) or q.tag != first.tag or q.iteration != first.iteration:
                raise ProtocolError(f"group {group.id}: mismatched collectives "
                                    f"({type(first).__name__}:{first.tag} vs {type(q).__name__}:{q.tag})")
        g = len(group.members)
        if isinstance(first, Barrier):
            return {r: None for r in group.members}
        if isinstance(first, Broadcast):
            if len({q.root for q in reqs}) != 1:
                raise ProtocolError(f"group {group.id}: broadcast roots disagree")
            src = posted[first.root].payload
            for q in reqs:
                if tuple(q.payload.shape) != tuple(src.shape):
                    raise ProtocolError(f"group {group.id}: broadcast shapes disagree on '{first.tag}'")
                if q.payload.data_ptr() != src.data_ptr():
                    q.payload.copy_(src)
            _ledger(self.ledger, first, g, _payload_bytes(src) * (g - 1), "broadcast")
            return {r: posted[r].payload for r in group.members}
        if len({tuple(q.payload.shape) for q in reqs}) != 1:
            raise ProtocolError(f"group {group.id}: payload shapes disagree on '{first.tag}'")
        if isinstance(first, AllGather):
            for q in reqs:
                for i, r in enumerate(group.members):
                    q.out[i].copy_(posted[r].payload)
            _ledger(self.ledger, first, g, _payload_bytes(first.payload), "allgather")
            return {r: posted[r].out for r in group.members}
        if g == 1:                               # identity: nothing moves
            _ledger(self.ledger, first, g, _payload_bytes(first.payload), f"allreduce_{first.op.value}")
            return {first.group.members[0]: first.payload}
        acc = reqs[0].payload.clone()            # serial fold in member order
        for q in reqs[1:]:
            acc += q.payload
        if first.op is ReduceOp.AVG:
            acc /= float(g)
        for q in reqs:
            q.payload.copy_(acc)
        _ledger(self.ledger, first, g, _payload_bytes(first.payload), f"allreduce_{first.op.value}")
        return {r: posted[r].payload for r in group.members}


class DistCluster(Cluster):
    """Executes one rank's program with torch.distributed (NCCL on B200, gloo on CPU).

    All ranks construct it collectively: ``dist.new_group`` is called for every
    intra group and the leader group in the same order on every rank.
    """

    concurrent_ranks = True   # one process (and device) per rank

    def __init__(self, topology: Topology, latency=None):
        import torch.distributed as dist

        if not dist.is_initialized():
            raise ProtocolError("torch.distributed is not initialized")
        if dist.get_world_size() != topology.world_size:
            raise ProtocolError(f"world size {dist.get_world_size()} != topology {topology.world_size}")
        self.topology = topology
        self.rank = dist.get_rank()
        self.ledger = CommLedger()
        self.ref_ledger = DeferredLedger()   # this rank's share of the reference's logical entries
        self._intra, self._leaders, self._global = hierarchy_groups(topology)
        self._handles = {}
        for i in range(topology.num_nodes):
            self._handles[self._intra[i].id] = dist.new_group(list(self._intra[i].members))
        self._handles["leaders"] = dist.new_group(list(self._leaders.members))
        self._handles["global"] = dist.group.WORLD
        self._avg = dist.get_backend() == "nccl"
        self.supports_peer = self._avg and self._symm_available()
        self._epoch: dict[str, int] = {}
        self._flags = None
        if self.supports_peer:
            # one world-symmetric int32 flag per (receiver, sender) for group barriers
            self._flags = self._world_buffer(topology.world_size, "int32")

    @staticmethod
    def _symm_available() -> bool:
        try:
            import torch.distributed._symmetric_memory  # noqa: F401
        except Exception:
            return False
        return True

    def _world_buffer(self, numel: int, dtype, device=None):
        """(tensor, world pointers): symmetric memory rendezvoused over the WORLD group.

        Every rank allocates every shared buffer in the same order — torch's
        symmetric-memory rendezvous must see the same sequence on all ranks — and
        sub-groups just read their members' entries."""
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        dt = getattr(torch, dtype) if isinstance(dtype, str) else dtype
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        t = symm.empty(max(int(numel), 1), dtype=dt, device=dev)
        t.zero_()
        h = symm.rendezvous(t, dist.group.WORLD)
        return t, [int(p) for p in h.buffer_ptrs], h

    def shared(self, rank: int, group: ProcessGroup, key: str, numel: int, dtype, device) -> SharedBuffer:
        """Collective over the WORLD (all ranks, same order): a buffer mapped on every rank;
        ``peer_ptrs()`` are ``group``'s members' copies in member order."""
        t, ptrs, _ = self._world_buffer(numel, dtype, device)
        members = [ptrs[m] for m in group.members]
        return SharedBuffer(t, lambda: members)

    def barrier(self, group: ProcessGroup, root: int | None = None) -> None:
        """Device-side barrier of ``group`` over NVLink flags (stream-ordered); with a
        root, one-sided: the root publishes, the others wait for the root."""
        from . import _lib
        from .plan import current_stream

        _, ptrs, _ = self._flags
        epoch = self._epoch.get(group.id, 0) + 1
        self._epoch[group.id] = epoch
        members = list(group.members)
        fl, keep1 = _lib.ptr_array([ptrs[m] for m in members])
        import ctypes as C

        slots = (C.c_int32 * len(members))(*members)
        mode = 0 if root is None else (1 if self.rank == root else 2)
        _lib.call("hsx_group_barrier_mode", fl, C.cast(slots, C.c_void_p), len(members), members.index(self.rank),
                  epoch, mode, members.index(root) if root is not None else 0, current_stream())
        del keep1

    def log(self, entry: LedgerEntry) -> None:
        self.ledger.append(entry)

    def intra_group(self, node: int) -> ProcessGroup:
        return self._intra[node]

    def leader_group(self) -> ProcessGroup:
        return self._leaders

    def global_group(self) -> ProcessGroup:
        return self._global

    def execute(self, req) -> Any:
        from .plan import note, timed

        _validate(self.rank, req)
        name = "C:" + req.tag.split("/")[0]
        g = len(req.group.members)
        if isinstance(req, Barrier):
            note(name, "barrier", 0, g)
        elif isinstance(req, Broadcast):
            note(name, "broadcast", _payload_bytes(req.payload), g)
        elif isinstance(req, AllGather):
            note(name, "all_gather", _payload_bytes(req.payload) * g, g)
        else:
            note(name, f"all_reduce_{req.op.value}", _payload_bytes(req.payload), g)
        with timed(name):
            return self._execute(req)

    def _execute(self, req) -> Any:
        import torch.distributed as dist

        h = self._handles[req.group.id]
        g = len(req.group.members)
        if isinstance(req, Barrier):
            if g > 1:
                self.barrier(req.group, req.root)
            return None
        if isinstance(req, Broadcast):
            if g > 1:
                dist.broadcast(req.payload, src=req.root, group=h)
            _ledger(self.ledger, req, g, _payload_bytes(req.payload) * (g - 1), "broadcast")
            return req.payload
        if isinstance(req, AllGather):
            if g > 1:
                dist.all_gather_into_tensor(req.out.view(-1), req.payload.view(-1), group=h)
            else:
                req.out[0].copy_(req.payload)
            _ledger(self.ledger, req, g, _payload_bytes(req.payload), "allgather")
            return req.out
        if g > 1:
            if req.op is ReduceOp.AVG and not self._avg:
                dist.all_reduce(req.payload, op=dist.ReduceOp.SUM, group=h)
                req.payload /= float(g)
            else:
                op = dist.ReduceOp.AVG if req.op is ReduceOp.AVG else dist.ReduceOp.SUM
                dist.all_reduce(req.payload, op=op, group=h)
        _ledger(self.ledger, req, g, _payload_bytes(req.payload), f"allreduce_{req.op.value}")
        return req.payload

    def run(self, programs: Mapping[int, RankProgram]) -> dict[int, Any]:
        """The reference's ``Cluster.run``: one process is one rank, so only this
        rank's program runs (the others' generators are never started)."""
        if self.rank not in programs:
            raise ProtocolError(f"no program for rank {self.rank}")
        return {self.rank: self.run_rank(programs[self.rank])}

    def run_rank(self, program: RankProgram) -> Any:
        """Drive this rank's generator to completion."""
        try:
            req = next(program)
            while True:
                req = program.send(self.execute(req))
        except StopIteration as stop:
            return stop.value
