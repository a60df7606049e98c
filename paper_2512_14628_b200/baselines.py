"""Comparison baselines on B200: the reference's flat consensus
and dense synchronous SGD (/root/reference/pkg/src/admmprune/baselines.py), for the
Fig. 6-style comparison against the hierarchical sync step.

* :class:`FlatConsensusSync` — ``flat_consensus_program`` (baselines.py:151-293)
  after phase 1: a dense all-rank SUM of theta + u, the candidate
  rho1 * total / (wd + W rho1) projected on the global tensor, the u-update, the
  3-slot residual SUM, the flat report and rho1 adaptation. It is the
  hierarchical engine on a one-node view of the cluster (1 x W) with rho2 = 0 and
  v = 0: the one-node leader average is the identity, so z = z_node (the fused
  K6 + K7 pass), v stays 0, and the candidate reduces to the flat one bit for
  bit (gamma = wd / 1 + W rho1 + 0; rho1 S + 0 (z - v) = rho1 S). The report
  kernel runs in its flat mode (inter entries 0, hsx_resid_params.flat).
* :class:`DenseSync` — ``dense_sync_program`` (baselines.py:77-98): per step
  g = grad + wd * params packed by ``hsx_dense_grad_pack``, the all-rank AVG, and
  the momentum update ``hsx_dense_apply``. Transport "peer": the AVG is fused into
  the update kernel, which folds the W ranks' send buffers over NVLink in rank
  order (no reduced buffer, one device barrier per step); "nccl": ncclAvg on the
  send buffer, then the update.
"""

from __future__ import annotations

import dataclasses

import torch

from . import _lib
from .errors import ProtocolError
from .plan import Plan, current_stream, ptr, timed
from .sync import HSADMMSync
from .transport import AllGather, AllReduce, Barrier, GroupScope, LedgerEntry, ProcessGroup, ReduceOp, Topology


class _FlatView:
    """A cluster seen as one node of W ranks: the intra group is the global group
    (baselines.py:164, ``cluster.global_group()``); everything else is the cluster's."""

    def __init__(self, cluster):
        self._cluster = cluster
        world = cluster.topology.world_size
        self.topology = Topology(1, world)
        self._leaders = ProcessGroup("flat_leader", (0,), GroupScope.INTER)

    def intra_group(self, node: int) -> ProcessGroup:
        return self._cluster.global_group()

    def leader_group(self) -> ProcessGroup:
        return self._leaders

    def __getattr__(self, name):
        return getattr(self._cluster, name)


class FlatConsensusSync(HSADMMSync):
    """One rank of ``flat_consensus_program`` (baselines.py:151-293) after phase 1.

    Same state arenas and API as :class:`~.sync.HSADMMSync` (``init_from``, ``load``,
    ``program`` / ``run_local`` / ``step``, ``views``, ``mask_dict``, ``last_report``,
    ``current_schedule``); ``z`` is the global variable (``z_node`` holds the same
    values), ``v`` stays 0. Every iteration syncs (the flat program has no sync period).
    """

    def __init__(self, rank: int, cluster, layers, constraints: dict, schedule, settings, device=None,
                 transport: str = "auto", residuals: bool = True):
        self._caller_schedule = schedule
        flat_sched = dataclasses.replace(schedule, rho2={n: 0.0 for n in schedule.rho2})
        flat_settings = dataclasses.replace(settings, sync_period=1)
        super().__init__(rank, _FlatView(cluster), layers, constraints, flat_sched, flat_settings, device=device,
                         transport=transport, residuals=residuals)
        self._resid_params.flat = 1

    def init_from(self, params0: dict) -> None:
        """theta = z = params0, u = 0 (baselines.py:169-172); z_node = z, v = 0."""
        super().init_from(params0)

    def current_schedule(self):
        """rho1 after device-side adaptation; rho2 as the caller gave it (unused by the
        flat program)."""
        s = super().current_schedule()
        return dataclasses.replace(s, rho2=dict(self._caller_schedule.rho2))

    def _reference_entries(self, k, sync, frozen, residuals, buckets, intra_first, inter_first):
        """flat_consensus_program's ledger for iteration k: z_sync/{layer} dense SUMs over
        the global group (baselines.py:190), then res_flat (3 slots per layer, :214)."""
        if not intra_first:
            return []
        g, W = self.intra, self.P
        out = [LedgerEntry(k, g.id, g.scope.value, "allreduce_sum", ls.elements, 4 * ls.elements, W,
                           f"z_sync/{ls.name}") for ls in self.layers]
        if residuals:
            L = len(self.layers)
            out.append(LedgerEntry(k, g.id, g.scope.value, "allreduce_sum", 3 * L, 12 * L, W, "res_flat"))
        return out


def run_flat_local(engines: list[FlatConsensusSync], k: int):
    """Iteration k of every rank of a LocalCluster (single process, one GPU)."""
    from .sync import run_local

    return run_local(engines, k)


class DenseSync:
    """One rank of ``dense_sync_program`` (baselines.py:77-98) after the gradient:
    params and velocity in fp32 arenas (the plan's layout), fp64 update math.

    ``load_grads(grads)`` (per-layer dict or a flat arena), then ``program(step)`` /
    ``step(step)`` applies g = grad + wd * params, the all-rank AVG, velocity =
    momentum * velocity + avg, params -= lr * velocity. The first step starts from
    zero velocity (:82).
    """

    def __init__(self, rank: int, cluster, layers, solver, device=None, transport: str = "auto"):
        if not solver.lr > 0:
            from .errors import ConfigError

            raise ConfigError(f"learning rate must be positive, got {solver.lr}")
        self.rank = rank
        self.cluster = cluster
        self.group = cluster.global_group()
        self.W = len(self.group.members)
        self.layers = list(layers)
        self.names = [ls.name for ls in layers]
        self.lr, self.momentum, self.weight_decay = float(solver.lr), float(solver.momentum), float(solver.weight_decay)
        zeros = {n: 0.0 for n in self.names}
        self.plan = Plan(self.layers, {}, zeros, zeros)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        pl, dev = self.plan, self.device
        self.n = pl.arena
        self.params, self.velocity, self.grad = (pl.empty_arena(dev) for _ in range(3))
        peer_ok = getattr(cluster, "supports_peer", False) and self.W <= 4
        if transport == "auto":
            transport = "peer" if (peer_ok and self.W > 1) else "nccl"
        if transport == "peer" and not peer_ok:
            raise ProtocolError("peer transport needs symmetric memory and at most 4 ranks")
        self.transport = transport
        if transport == "peer":   # double-buffered by step parity: one barrier per step
            self.p_send = [cluster.shared(rank, self.group, f"dense_send{b}", self.n, torch.float32, dev)
                           for b in (0, 1)]
        else:
            self.send = pl.empty_arena(dev)
        self.first = True
        self.steps_done = 0

    def init_from(self, params0: dict) -> None:
        self.plan.load_arena(self.params, params0)
        self.velocity.zero_()
        self.first = True

    def load_grads(self, grads) -> None:
        if isinstance(grads, torch.Tensor):
            self.grad.copy_(grads)
        else:
            self.plan.load_arena(self.grad, grads)

    def views(self, key: str) -> dict:
        return self.plan.views(getattr(self, key))

    def program(self, step: int):
        """Generator: the step's collective requests (a Barrier over NVLink for "peer",
        the AVG all-reduce for "nccl")."""
        send = self.p_send[step & 1].tensor if self.transport == "peer" else self.send
        with timed("D_grad_pack"):
            _lib.call("hsx_dense_grad_pack", ptr(self.grad), ptr(self.params), self.weight_decay, ptr(send),
                      self.n, current_stream())
        if self.transport == "peer":
            yield Barrier(self.group, "grad", step)
            ptrs = self.p_send[step & 1].peer_ptrs()
            arr, keep = _lib.ptr_array(ptrs)
            with timed("D_avg_apply_peers"):
                _lib.call("hsx_dense_apply", arr, len(ptrs), float(self.W), ptr(self.params), ptr(self.velocity),
                          self.lr, self.momentum, 1 if self.first else 0, self.n, current_stream())
            del keep
        else:
            yield AllReduce(self.group, send, ReduceOp.AVG, "grad", step)
            arr, keep = _lib.ptr_array([ptr(send)])
            with timed("D_apply"):
                _lib.call("hsx_dense_apply", arr, 1, 1.0, ptr(self.params), ptr(self.velocity), self.lr,
                          self.momentum, 1 if self.first else 0, self.n, current_stream())
            del keep
        self.first = False
        self.steps_done += 1
        self._log_reference(step)

    def _log_reference(self, step: int):
        """dense_sync_program's ledger: grad/{layer} AVG over the global group (:89)."""
        led = getattr(self.cluster, "ref_ledger", None)
        if led is None or (getattr(self.cluster, "shared_ledger", False) and self.rank != self.group.members[0]):
            return
        g, W = self.group, self.W
        entries = [LedgerEntry(step, g.id, g.scope.value, "allreduce_avg", ls.elements, 4 * ls.elements, W,
                               f"grad/{ls.name}") for ls in self.layers]
        led.defer(lambda: entries)

    def step(self, step: int):
        if not hasattr(self.cluster, "run_rank"):
            raise ProtocolError("step() needs a DistCluster; use run_dense_local for in-process ranks")
        return self.cluster.run_rank(self.program(step))


def run_dense_local(engines: list[DenseSync], step: int):
    """Step ``step`` of every rank of a LocalCluster (single process, one GPU)."""
    cluster = engines[0].cluster
    return cluster.run({e.rank: e.program(step) for e in engines})


class TopKSync:
    """One rank of ``topk_program`` (baselines.py:101-148) after the gradient: Top-K
    compression with error feedback. Per layer the ceil(rate * n) largest |acc| of
    acc = residual + grad + wd * params (fp64 residual arena, in place) travel as
    (fp32 value, int32 index) pairs — 8 B per pair, the reference ledger's 2 x 4 B —
    in ONE all-gather for all layers; the gathered pairs are scatter-added in rank
    order into an fp64 buffer, then / W and the momentum update.

    Device path: ``hsx_topk_select`` (fused acc + 8-pass radix select per layer +
    ordered write + residual clear), the all-gather, W x ``hsx_topk_scatter``,
    ``hsx_topk_apply``.
    """

    def __init__(self, rank: int, cluster, layers, solver, rate: float, device=None):
        import ctypes as C

        if not solver.lr > 0:
            from .errors import ConfigError

            raise ConfigError(f"learning rate must be positive, got {solver.lr}")
        self.rank = rank
        self.cluster = cluster
        self.group = cluster.global_group()
        self.W = len(self.group.members)
        self.layers = list(layers)
        self.names = [ls.name for ls in layers]
        self.rate = float(rate)
        self.lr, self.momentum, self.weight_decay = float(solver.lr), float(solver.momentum), float(solver.weight_decay)
        zeros = {n: 0.0 for n in self.names}
        self.plan = Plan(self.layers, {}, zeros, zeros)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        pl, dev = self.plan, self.device
        self.params, self.velocity, self.grad = (pl.empty_arena(dev) for _ in range(3))
        self.residual = torch.zeros(pl.arena, dtype=torch.float64, device=dev)
        self.dense = torch.zeros(pl.arena, dtype=torch.float64, device=dev)
        L = len(self.layers)
        offs = (C.c_int64 * max(L, 1))(*pl.offsets)
        elems = (C.c_int64 * max(L, 1))(*[ls.elements for ls in self.layers])
        h = C.c_void_p()
        lib = _lib.load()
        _lib.check(lib.hsx_topk_create(C.cast(offs, C.c_void_p), C.cast(elems, C.c_void_p), self.rate, L,
                                       C.byref(h)), "hsx_topk_create")
        self._h = h
        self.K = int(lib.hsx_topk_total(h))
        self.keep = []
        for i in range(L):
            k, o = C.c_int64(), C.c_int64()
            _lib.call("hsx_topk_layer_keep", h, i, C.byref(k), C.byref(o))
            self.keep.append((int(k.value), int(o.value)))
        self.payload = torch.zeros(2 * max(self.K, 1), dtype=torch.int32, device=dev)
        self.gathered = torch.zeros((self.W, 2 * max(self.K, 1)), dtype=torch.int32, device=dev)
        self.first = True

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.load().hsx_topk_destroy(h)
            except Exception:
                pass

    def init_from(self, params0: dict) -> None:
        self.plan.load_arena(self.params, params0)
        self.velocity.zero_()
        self.residual.zero_()
        self.dense.zero_()
        self.first = True

    def load_grads(self, grads) -> None:
        if isinstance(grads, torch.Tensor):
            self.grad.copy_(grads)
        else:
            self.plan.load_arena(self.grad, grads)

    def views(self, key: str) -> dict:
        t = getattr(self, key)
        return {n: t[o:o + ls.elements].view(ls.shape) for n, ls, o in zip(self.names, self.layers, self.plan.offsets)}

    def selections(self) -> dict:
        """This rank's last selected (layer-local, ascending) indices per layer."""
        idx = self.payload[self.K:2 * self.K]
        return {n: idx[o:o + k] for n, (k, o) in zip(self.names, self.keep)}

    def program(self, step: int):
        K = self.K
        vals = self.payload[:K].view(torch.float32)
        with timed("T_select"):
            _lib.call("hsx_topk_select", self._h, ptr(self.grad), ptr(self.params), self.weight_decay,
                      ptr(self.residual), ptr(vals), ptr(self.payload[K:]), current_stream())
        yield AllGather(self.group, self.payload, self.gathered, "topk", step)
        with timed("T_scatter_apply"):
            for j in range(self.W):   # rank order (:137-139)
                row = self.gathered[j]
                _lib.call("hsx_topk_scatter", self._h, ptr(row[:K].view(torch.float32)), ptr(row[K:2 * K]),
                          ptr(self.dense), current_stream())
            _lib.call("hsx_topk_apply", self._h, ptr(self.dense), float(self.W), ptr(self.params),
                      ptr(self.velocity), self.lr, self.momentum, 1 if self.first else 0, current_stream())
        self.first = False
        self._log_reference(step)

    def _log_reference(self, step: int):
        """topk_program's ledger: topk/{layer} all-gathers of 2k elements (:136)."""
        led = getattr(self.cluster, "ref_ledger", None)
        if led is None or (getattr(self.cluster, "shared_ledger", False) and self.rank != self.group.members[0]):
            return
        g, W = self.group, self.W
        entries = [LedgerEntry(step, g.id, g.scope.value, "allgather", 2 * k, 8 * k, W, f"topk/{n}")
                   for n, (k, _) in zip(self.names, self.keep)]
        led.defer(lambda: entries)

    def step(self, step: int):
        if not hasattr(self.cluster, "run_rank"):
            raise ProtocolError("step() needs a DistCluster; use run_topk_local for in-process ranks")
        return self.cluster.run_rank(self.program(step))


def run_topk_local(engines: list[TopKSync], step: int):
    cluster = engines[0].cluster
    return cluster.run({e.rank: e.program(step) for e in engines})
