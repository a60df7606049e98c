"""HSADMMSync — the B200-native H-SADMM synchronization step (one rank).

Replaces phases 2-4 and the u-update of phase 5 of the reference's
``hierarchical_program`` (/root/reference/pkg/src/admmprune/consensus.py:436-535)
plus the freeze / keep-set seal (:600-606), in SPMD form: one engine per rank
(one rank per GPU under ``torchrun``, or all ranks of a topology on one GPU
through :class:`~.transport.LocalCluster`).

Per iteration k (leader = local rank 0 of its node):

    K0  S = theta + u                        (skipped when P == 1: fused into K1)
    C1  intra all-reduce SUM of S            (NCCL over NVLink)
    K1  z_node = candidate; fp64 group-norm partials          [dynamic]
    K2  top-k keep flags per constraint pass                  [dynamic]
    K3  zero dropped groups, local mask bits                  [dynamic]
    C2  leaders all-gather packed mask bits; K4 OR -> union   [dynamic, M > 1]
    C4a intra broadcast of the union bits                     [dynamic, P > 1]
    K5  keep sets (K_out/K_in, positions, payload offsets), drift popcounts;
        one D2H of the per-layer counts sizes the collectives [dynamic]
    K6  leader: flat <- compress(z_node + v) fused with u += theta - z_node
        follower: K6f u += theta - z_node
    C3  leaders all-reduce AVG of the flat compact buffer, per <=32 MiB bucket
    C4  intra broadcast of the reduced compact buffer (not of z and v: every
        rank of a node holds bitwise-identical z_node and v, so followers
        decompact locally and get the leader's z, v bit-for-bit)
    K7  z = decompress(flat); v += z_node - z

Frozen iterations (after ``t_freeze`` or a zero-drift window) skip K2-K5,
C2 and C4a: K1 applies the frozen union mask and the sealed keep sets stay
on the device.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from .consensus import ConsensusSettings, PenaltySchedule, freeze_check
from .errors import ProtocolError, ShapeError
from .layers import LayerSpec
from .plan import Plan, mask_or, mask_or_ptrs
from .sparsity import resolve_plan
from .transport import AllGather, AllReduce, Barrier, Broadcast, LedgerEntry, ReduceOp, bucketize
from . import _lib


_F1 = os.environ.get("HSX_F1", "0") == "1"               # two leaders: average fused into K7
_REMOTE_K7 = os.environ.get("HSX_REMOTE_K7", "1") != "0"  # followers decompact from the leader's payload
# leaders, opt-in: the intra dual on a side stream beside the exchange; measured no
# faster (RN50 2x2: K6 95 -> 56 us, but K8 87 -> 121 us and K6f 87 us beside it, r2ze)
_SPLIT_K6 = os.environ.get("HSX_SPLIT_K6") == "1"
# leader -> follower hand-offs (union mask, node payload) as one-sided barriers: the
# leader publishes and runs on; the next step's two-sided theta_u barrier orders the
# followers' reads before the leader's next write. Parity green, measured no faster
# (the leader's path is the long one; 2x2 RN18/RN50 steady step unchanged), so
# opt-in (HSX_ONESIDED=1)
_ONESIDED = os.environ.get("HSX_ONESIDED") == "1"
# multi-node peer steps: the mask union (K4) formed inside K5 from the leaders' mask
# bits over NVLink, for leaders and followers alike (HSX_FUSED_UNION=0: K4, then the
# followers copy their leader's union, then K5)
_FUSED_UNION = os.environ.get("HSX_FUSED_UNION", "1") != "0"
# P > 2 peer steps: K1 reads the intra sum from the reduce-scatter slices over NVLink
# instead of all-gathering S first (HSX_DIST_SUM=0: all-gather, then K1 on S)
_DIST_SUM = os.environ.get("HSX_DIST_SUM", "1") != "0"


class HSADMMSync:
    """Device state + sync program of one rank.

    State arenas (fp32, shared layout from :class:`~.plan.Plan`): ``theta``,
    ``u``, ``z_node``, ``v``, ``z``; ``masks`` holds the global union mask bits
    of the prunable layers (initially all ones, consensus.py:418).
    """

    def __init__(self, rank: int, cluster, layers: list[LayerSpec], constraints: dict,
                 schedule: PenaltySchedule, settings: ConsensusSettings, device=None,
                 transport: str = "auto", residuals: bool = True):
        topo = cluster.topology
        self.rank = rank
        self.cluster = cluster
        self.topology = topo
        self.M, self.P = topo.num_nodes, topo.accels_per_node
        self._staged = False
        self._split = False
        self.node = topo.node_of(rank)
        self.leader_rank = topo.leader_of(self.node)
        self.is_leader = rank == self.leader_rank
        self.intra = cluster.intra_group(self.node)
        self.inter = cluster.leader_group()
        self.layers = list(layers)
        self.names = [ls.name for ls in layers]
        self.settings = settings
        self.schedule = schedule
        groups = {ls.name: resolve_plan(ls.shape, constraints[ls.name])
                  for ls in layers if constraints.get(ls.name)}
        self.plan = Plan(self.layers, groups, schedule.rho1, schedule.rho2)
        self.plan.set_penalties(schedule.rho1, schedule.rho2, settings.weight_decay, self.M, self.P)
        # one node: the union mask is every rank's local mask, so the selection derives
        # the keep sets of the kept rectangle and K3 only checks it (hsx_project_keep_sets)
        self.plan.set_single_node(self.M == 1 and os.environ.get("HSX_SINGLE_NODE", "1") != "0")
        # one node, opt-in (HSX_K67_CHAIN=1): every sync step's projection is followed
        # by K67, so the two may chain per layer; that needs the keep-set summary fetched
        # after K67 (the fetch's event would sit between them), which delays the host's
        # next step: measured +6% on RN18 1x1, -1..3% on RN50 / RN152 (r2p)
        self._k67_chain = (os.environ.get("HSX_K67_CHAIN") == "1" and self.M == 1
                           and os.environ.get("HSX_SINGLE_NODE", "1") != "0"
                           and os.environ.get("HSX_LOCAL_SYNC", "1") != "0")
        self.plan.set_k67_chain(self._k67_chain)
        self.prunable = self.plan.prunable
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        pl, dev = self.plan, self.device
        self.theta, self.u, self.z_node, self.v, self.z = (pl.empty_arena(dev) for _ in range(5))
        # phase 5 (consensus.py:537-598): residual sums fused into K6 / K7, the report
        # and the adaptive penalties on the device; z_node is double-buffered so K7
        # sees the previous iteration's z_node
        self.residuals = bool(residuals)
        self.z_node_prev = pl.empty_arena(dev) if self.residuals else None
        nl = len(self.layers)
        self.rvec = torch.zeros(max(nl * _lib.RESID_SLOTS, 1), dtype=torch.float64, device=dev)
        self.report = torch.zeros(nl * 8 + 5, dtype=torch.float64, device=dev)
        self.scales = torch.ones(max(2 * nl, 1), dtype=torch.float64, device=dev)
        self._resid_params = _lib.ResidParams(
            settings.weight_decay, settings.eps_abs, settings.eps_rel, schedule.mu, schedule.tau_inc,
            schedule.tau_dec, schedule.rho1_max, schedule.rho2_max, self.M, self.P, 1 if schedule.adapt else 0)
        self.reported = False
        self.sum = pl.empty_arena(dev) if self.P > 1 else None
        self.flat = torch.zeros(max(pl.arena, 1), dtype=torch.float32, device=dev)
        self.masks = pl.empty_mask(dev, ones=True)
        self.union = pl.empty_mask(dev)
        self.local_mask = pl.empty_mask(dev)
        self.gathered = (torch.zeros((self.M, max(pl.mask_words, 1)), dtype=torch.int32, device=dev)
                         if self.is_leader and self.M > 1 else None)
        self.frozen = False
        self.drift_history: list[float] = []
        self.drift_now: dict[str, float] = {}
        self.cache_derive = 0
        self.cache_hits = 0
        self.cache_seen = False
        self.payload_elements = sum(ls.elements for ls in self.layers)  # all kept initially
        self.buckets = None
        self._elems = None
        self._prunable_idx = np.array(self.prunable, dtype=np.int64)
        self._prunable_names = [self.names[i] for i in self.prunable]
        self._prunable_elems = np.array([self.layers[i].elements for i in self.prunable], dtype=np.float64)
        self._layout_from_summary(initial=True)
        # transport: "peer" = fused NVLink kernels on peer-mapped buffers (no NCCL on the
        # step, no mid-step host sync); "nccl" = torch.distributed collectives
        peer_ok = getattr(cluster, "supports_peer", False) and self.M <= 4 and self.P <= 4
        if transport == "auto":  # one rank has no collectives: the plain path has fewer launches
            transport = "peer" if (peer_ok and self.M * self.P > 1) else "nccl"
        if transport == "peer" and not peer_ok:
            raise ProtocolError("peer transport needs symmetric memory and at most 4 x 4 ranks")
        self.transport = transport
        if transport == "peer":
            self._init_peer_buffers()
            if self.P == 2 and "HSX_K1_ORDER" not in os.environ:
                self.plan.set_order(False)   # K1 reads the intra sum over NVLink: layer order (r2n)
            # two ranks, opt-in (HSX_PEER_STAGING=1): the peer's send staged into local
            # memory by a copy kernel on a side stream running ahead of K1; measured
            # much slower (RN18 1x2 0.21 -> 0.54 ms, r2zc: the copy kernel does not keep
            # pace next to K1), so by default K1 reads it over NVLink itself
            self._staged = self.P == 2 and os.environ.get("HSX_PEER_STAGING") == "1"
            if self._staged:
                self.plan.set_peer_staging(True)
            self._init_split()
        # deferred host bookkeeping (step_host): a step returns once its launches are
        # queued; the keep-set counts are read back when the next step starts
        self.defer_host = False
        self._pending = None
        self._pipe = None

    def _init_split(self):
        """Split two-rank K1 (HSX_K1_SPLIT=1; P == 2, one process per rank): each rank
        computes half of the prunable tiles reading half of the peer's send over NVLink
        and writes z_node, the group-norm partials and the chained selection's tile
        counts into both ranks' (peer-mapped) buffers. z_node (and its residual double
        buffer) move into peer-mapped memory; the allocations are collective over the
        world, so every rank takes the same decision (same env, topology and plan)."""
        self._split = False
        self._zn_peer = {}
        if not (self.P == 2 and os.environ.get("HSX_K1_SPLIT") == "1"
                and getattr(self.cluster, "concurrent_ranks", False) and self.prunable):
            return
        pl, dev, cl = self.plan, self.device, self.cluster
        me = self.intra.members.index(self.rank)
        zn = [cl.shared(self.rank, self.intra, f"zn{b}", pl.arena, torch.float32, dev) for b in (0, 1)]
        npart, ncnt = pl.split_sizes()
        part = cl.shared(self.rank, self.intra, "k1part", npart, torch.float64, dev)
        cnt = cl.shared(self.rank, self.intra, "k1cnt", ncnt, torch.int32, dev)
        try:
            pl.set_split(me, part.tensor, part.peer_ptrs()[1 - me], cnt.tensor, cnt.peer_ptrs()[1 - me])
        except Exception:   # e.g. a multi-pass plan: the same outcome on every rank
            return
        zn[0].tensor.copy_(self.z_node)
        self.z_node = zn[0].tensor
        if self.z_node_prev is not None:
            zn[1].tensor.copy_(self.z_node_prev)
            self.z_node_prev = zn[1].tensor
        self._zn_spare = zn[1].tensor
        self._zn_peer = {b.tensor.data_ptr(): b.peer_ptrs()[1 - me] for b in zn}
        self._split_bufs = (zn, part, cnt)
        self._split = True

    def _init_peer_buffers(self):
        """Shared (peer-mapped) buffers; allocation is collective over each group."""
        pl, dev, cl = self.plan, self.device, self.cluster
        words = max(pl.mask_words, 1)
        self.p_send = self.p_umask = self.p_zhat = self.p_lmask = None
        self.p_flat = None
        self._send_idx = 0      # p_send buffer of the next step
        self._nsync = 0         # leader syncs so far (p_flat buffer)
        # every rank allocates the same sequence (the allocation is collective over
        # all ranks); followers leave the leader-group buffers unused
        if self.P > 1:
            # double-buffered by step parity: a peer's K1 may still read this step's
            # send buffer when the next step packs theta + u (nothing else orders the
            # two when the node has no later intra barrier, e.g. M == 1); the next
            # step's theta_u barrier orders the rewrite two steps later
            self.p_send = [cl.shared(self.rank, self.intra, f"send{b}", pl.arena, torch.float32, dev)
                           for b in (0, 1)]
            self.p_umask = cl.shared(self.rank, self.intra, "umask", words, torch.int32, dev)
            self.p_zhat = cl.shared(self.rank, self.intra, "zhat", pl.arena, torch.float32, dev)
        self.p_ssum = self.p_favg = None
        if self.P > 2:   # reduce-scatter + all-gather of the intra sum
            self.p_ssum = cl.shared(self.rank, self.intra, "ssum", pl.arena, torch.float32, dev)
        self._lmask_all = None
        self._nmask = 0         # fused-union mask phases so far (leader mask buffer)
        if self.M > 1:
            # the leaders' local masks, double-buffered by step parity: with the union
            # formed inside K5 every rank (followers too) reads all leaders' masks, and
            # nothing orders another node's follower's read before this leader's next
            # K3; its rewrite two steps later is ordered by the next mask_sync
            lmask2 = [cl.shared(self.rank, self.inter, f"lmask{b}", words, torch.int32, dev) for b in (0, 1)]
            self._lmask_all = lmask2
            lmask = lmask2[0]
            # double-buffered by sync count: a leader may start the next compaction
            # while another still averages this one (the next z_sync barrier orders
            # the rewrite two syncs later)
            flat = [cl.shared(self.rank, self.inter, f"flat{b}", pl.arena, torch.float32, dev) for b in (0, 1)]
            favg = (cl.shared(self.rank, self.inter, "favg", pl.arena, torch.float32, dev)
                    if self.M > 2 else None)   # reduce-scatter + all-gather of the leader average
            if self.is_leader:
                self.p_lmask, self.p_flat, self.p_favg = lmask, flat, favg

    # -- state I/O ---------------------------------------------------------------
    def load(self, **arrays) -> None:
        """Copy per-layer dicts into arenas, e.g. ``load(theta=..., u=..., z=...)``."""
        for key, values in arrays.items():
            self.plan.load_arena(getattr(self, key), values)

    def init_from(self, params0: dict) -> None:
        """Reference initial state: theta = z_node = z = params0, u = v = 0 (consensus.py:412-418)."""
        self.load(theta=params0, z_node=params0, z=params0)
        self.u.zero_()
        self.v.zero_()

    def views(self, key: str) -> dict:
        return self.plan.views(getattr(self, key))

    def mask_dict(self) -> dict:
        return {self.names[i]: self.plan.unpack_mask(self.masks, i) for i in self.prunable}

    # -- layout of the flat compact buffer -------------------------------------------
    def _layout_from_summary(self, initial=False):
        if initial:
            elems = np.array([ls.elements for ls in self.layers], dtype=np.int64)
        else:
            rows, total = self.plan.summary_np()
            elems = rows[:, _lib.SUM_ELEMS]
            self.payload_elements = total
        if self._elems is not None and np.array_equal(elems, self._elems):
            return                                   # same sizes: reuse the bucket layout
        self._elems = elems.copy()
        # layers whose kept rectangle is empty are not sent (consensus.py:480)
        self.payload = [(n, int(e)) for n, e in zip(self.names, elems) if e > 0]
        self.buckets = bucketize(self.payload)

    def _after_keep_sets(self):
        """Host bookkeeping once the per-layer counts have landed (no device work)."""
        self._layout_from_summary()
        rows, _ = self.plan.summary_np()
        pr = self._prunable_idx
        drift_bits = rows[pr, _lib.SUM_DRIFT]
        drift = drift_bits / self._prunable_elems
        self.drift_now = dict(zip(self._prunable_names, drift.tolist()))
        self.drift_history.append(float(drift.max()))
        if self.is_leader:                              # KeepSetCache counters (shrinkage.py:115-130)
            derive = len(pr) if not self.cache_seen else int(np.count_nonzero(drift_bits))
            self.cache_derive += derive
            self.cache_hits += len(pr) - derive
            self.cache_seen = True

    @property
    def leader_bytes(self) -> int:
        """z_sync payload bytes per leader per sync (4 B / element, harness.py:447-449 convention)."""
        return 4 * self.payload_elements

    # -- the per-iteration program ------------------------------------------------------
    def _begin_step(self):
        """z_node_prev <- the last iteration's z_node (K1 writes the other buffer)."""
        if self.residuals:
            self.z_node, self.z_node_prev = self.z_node_prev, self.z_node

    def program(self, k: int):
        """Generator: yields collective requests, performs phases 2-5 of iteration k."""
        self.settle()
        self._begin_step()
        if self.transport == "peer":
            return (yield from self._program_peer(k))
        return (yield from self._program_nccl(k))

    def _log_zsync(self, k: int):
        """Ledger entries of the leader average, identical to the reference's z_sync/b{i}
        (one entry per group collective: a ledger shared by in-process ranks gets it once)."""
        if getattr(self.cluster, "shared_ledger", False) and self.rank != self.inter.members[0]:
            return
        for bi, b in enumerate(self.buckets):
            self.cluster.log(LedgerEntry(k, self.inter.id, self.inter.scope.value, "allreduce_avg",
                                         b.elements, 4 * b.elements, self.M, f"z_sync/b{bi}", b.detail))

    def _log_reference(self, k: int, sync: bool, frozen: bool):
        """The ledger the reference writes for iteration k (transport.py:413-476 entries of
        hierarchical_program's collectives, consensus.py:436-573), into
        ``cluster.ref_ledger``: per-layer theta_u / mask_sync / z_bcast / v_bcast / m_bcast,
        the z_sync buckets, res_intra / res_inter / report — 4 B per element, broadcasts
        only in groups of > 1, each group collective once (by its first member). The
        physical transfers (one arena all-reduce, packed mask bits, the compact
        broadcast) are in ``cluster.ledger``."""
        led = getattr(self.cluster, "ref_ledger", None)
        if led is None:
            return
        shared = getattr(self.cluster, "shared_ledger", False)
        intra_first = not shared or self.rank == self.intra.members[0]
        inter_first = self.is_leader and (not shared or self.rank == self.inter.members[0])
        if not (intra_first or inter_first):
            return
        # everything the entries depend on, captured now; the entries are built on read
        ctx = (k, sync, frozen, self.residuals, self.buckets, intra_first, inter_first)
        led.defer(lambda: self._reference_entries(*ctx))

    def _reference_entries(self, k, sync, frozen, residuals, buckets, intra_first, inter_first):
        out = []
        L = len(self.layers)
        sizes = [(ls.name, ls.elements) for ls in self.layers]
        pr = [(self.names[i], self.layers[i].elements) for i in self.prunable]
        P, M = self.P, self.M

        def add(group, op, elems, nbytes, members, label, detail=None):
            if nbytes > 0:
                out.append(LedgerEntry(k, group.id, group.scope.value, op, int(elems), int(nbytes), members,
                                       label, detail))

        if intra_first:
            for n, e in sizes:
                add(self.intra, "allreduce_sum", e, 4 * e, P, f"theta_u/{n}")
        if sync:
            if inter_first and not frozen:
                for n, e in pr:
                    add(self.inter, "allreduce_bor", e, 4 * e, M, f"mask_sync/{n}")
            if inter_first:
                for bi, b in enumerate(buckets):
                    add(self.inter, "allreduce_avg", b.elements, 4 * b.elements, M, f"z_sync/b{bi}", b.detail)
            if intra_first and P > 1:
                for tag in ("z_bcast", "v_bcast"):
                    for n, e in sizes:
                        add(self.intra, "broadcast", e, 4 * e * (P - 1), P, f"{tag}/{n}")
                if not frozen:
                    for n, e in pr:
                        add(self.intra, "broadcast", e, 4 * e * (P - 1), P, f"m_bcast/{n}")
        if residuals:
            if intra_first:
                add(self.intra, "allreduce_sum", 3 * L, 12 * L, P, "res_intra")
            if inter_first:
                add(self.inter, "allreduce_sum", 9 * L, 36 * L, M, "res_inter")
            if intra_first and P > 1:
                add(self.intra, "broadcast", 8 * L + 5, 4 * (8 * L + 5) * (P - 1), P, "report")
        return out

    def _program_peer(self, k: int):
        """Phases 2-5(u) with the collectives fused into the kernels over NVLink.

        intra sum -> K1 reads the P ranks' theta+u over NVLink (rank-order fp64 fold);
        mask union -> K4 reads the M leaders' mask bits; leader average -> K8 streams
        the M leaders' compact buffers (rank-order fold, / M) into the node's payload
        buffer; intra broadcast -> each follower streams its leader's payload; then
        every rank decompacts locally (K7). Barriers order producers before peer
        readers; payload sizes stay on the device, so the step has no host sync
        until its end. Inter-node traffic stays leader-to-leader (hierarchy kept).
        """
        pl = self.plan
        frozen = self.frozen
        dynamic = not frozen and bool(self.prunable)
        fmask = self.masks if (frozen and self.prunable) else None
        s_local, peers = None, None
        send = None
        if self.P > 1:
            send = self.p_send[self._send_idx]
            self._send_idx ^= 1
        if self.P > 2:
            # reduce-scatter (my slice of the rank-order sum) + all-gather, then K1 on S
            self._pack_send(send.tensor)
            yield Barrier(self.intra, "theta_u", k)
            me = self.intra.members.index(self.rank)
            pl.slices_peers(send.peer_ptrs(), me, 1.0, False, self.p_ssum.tensor, "K8_intra_rs")
            yield Barrier(self.intra, "theta_u_ag", k)
            if _DIST_SUM and pl.max_passes == 1:
                # K1 reads each quad of S from its slice owner over NVLink: no
                # all-gather of S (composite plans keep S for their renorm passes)
                pl.candidate_dist(self.p_ssum.peer_ptrs(), self.z, self.v, self.z_node, frozen_mask=fmask)
            else:
                pl.slices_peers(self.p_ssum.peer_ptrs(), -1, 1.0, False, self.sum, "K8_intra_ag")
                s_local = self.sum
                pl.candidate(s_local, None, None, self.z, self.v, self.z_node, frozen_mask=fmask)
        elif self.P == 2:
            # the intra sum fused into K1: theta+u of both ranks read over NVLink
            self._pack_send(send.tensor)
            yield Barrier(self.intra, "theta_u", k)
            peers = send.peer_ptrs()
            if self._split and fmask is None:
                pl.candidate_peers_split(peers, self.z, self.v, self.z_node, self._zn_peer[self.z_node.data_ptr()])
            elif self._staged and fmask is None:
                pl.candidate_peers_staged(peers, self.intra.members.index(self.rank), self.z, self.v, self.z_node)
            else:
                pl.candidate_peers(peers, self.z, self.v, self.z_node, frozen_mask=fmask)
        else:
            pl.candidate(None, self.theta, self.u, self.z, self.v, self.z_node, frozen_mask=fmask)
        # one node: every rank's local mask is the node's (identical z_node), so the
        # union needs no exchange and K3 derives the keep sets itself
        fused_keep = dynamic and self.M == 1 and k % self.settings.sync_period == 0
        if fused_keep:
            pl.project_all(s_local, self.theta, self.u, self.z, self.v, self.z_node, self.union, peers=peers,
                           keep_prev=True, prev_mask=self.masks)
        elif dynamic:
            if _FUSED_UNION and self._lmask_all is not None:
                # leaders of a syncing step: this sync's buffer (read by every rank's K5)
                sync_now = k % self.settings.sync_period == 0
                local = (self._lmask_all[self._nmask & 1].tensor if (self.is_leader and sync_now)
                         else self.local_mask)
            else:
                local = self.p_lmask.tensor if self.p_lmask is not None else self.local_mask
            pl.project_all(s_local, self.theta, self.u, self.z, self.v, self.z_node, local, peers=peers)
        if k % self.settings.sync_period != 0:
            self._dual(None)
            yield from self._residual_phase(k, sync=False)
            self._log_reference(k, False, self.frozen)
            self.plan.join_stage()
            return None
        ev = None
        if fused_keep:
            if not self._k67_chain:   # chained: fetched after K67 (K3 -> K67 consecutive launches)
                ev = pl.keep_sets_fetch_async()
        elif dynamic and _FUSED_UNION and self._lmask_all is not None:
            # K4 fused into K5: after the leaders' masks are final (mask_sync among the
            # leaders, then m_bcast inside each node) every rank ORs the M leaders'
            # mask bits over NVLink while marking its keep sets
            if self.is_leader:
                yield Barrier(self.inter, "mask_sync", k)
            if self.P > 1:
                yield Barrier(self.intra, "m_bcast", k, root=self.leader_rank if _ONESIDED else None)
            pl.keep_sets_ptrs(self._lmask_all[self._nmask & 1].peer_ptrs(), self.union, self.masks)
            self._nmask += 1
            ev = pl.keep_sets_fetch_async()
        elif dynamic:
            words = pl.mask_words
            if self.is_leader:
                target = self.p_umask.tensor if self.P > 1 else self.union
                srcs = self.p_lmask.peer_ptrs() if self.M > 1 else [local.data_ptr()]
                if self.M > 1:
                    yield Barrier(self.inter, "mask_sync", k)
                mask_or_ptrs(srcs, words, target)
            if self.P > 1:
                yield Barrier(self.intra, "m_bcast", k, root=self.leader_rank if _ONESIDED else None)
                mask_or_ptrs([self.p_umask.peer_ptrs()[0]], words, self.union)  # copy of the leader's union
            pl.keep_sets(self.union, self.masks)
            ev = pl.keep_sets_fetch_async()
        elif self.is_leader and self.prunable:
            self.cache_hits += len(self.prunable)
        zhat = self.p_zhat.tensor if self.P > 1 else None
        if self.M == 1:
            # one node: the leader "average" is the identity and every rank holds the
            # same z_node and v, so each rank runs K6+K7 locally in one pass (bitwise
            # what the compact round trip and the intra broadcast would deliver)
            self._local_sync()
            if fused_keep and self._k67_chain:
                ev = pl.keep_sets_fetch_async()
            return (yield from self._end_step(k, dynamic, ev, log_zsync=True))
        decompacted = False
        if self.is_leader:
            if self.M > 1:
                flat = self.p_flat[self._nsync & 1]
                self._nsync += 1
                if not self.residuals and _SPLIT_K6:
                    # the leader's critical path needs only the compaction before the
                    # exchange: the intra dual u += theta - z_node (12N bytes, read by
                    # nothing until the next step) on a side stream under the leader
                    # average (HSX_SPLIT_K6=1)
                    pl.compact_dual(None, None, self.z_node, self.v, flat.tensor)
                    self._side_dual()
                else:
                    self._dual(flat.tensor)
                yield Barrier(self.inter, "z_sync", k)
                # leader average over NVLink into the node's payload buffer
                dst = zhat if zhat is not None else self.flat
                if self.M > 2:
                    me = self.inter.members.index(self.rank)
                    pl.slices_peers(flat.peer_ptrs(), me, float(self.M), True, self.p_favg.tensor, "K8_leader_rs")
                    yield Barrier(self.inter, "z_sync_ag", k)
                    pl.slices_peers(self.p_favg.peer_ptrs(), -1, 1.0, True, dst, "K8_leader_ag")
                elif _F1:
                    # F1: the average fused into the decompaction (the other leader's
                    # payload read over NVLink), the averaged payload left in zhat
                    pl.decompact_average(flat.peer_ptrs(), float(self.M), zhat, self.z_node, self.z_node_prev,
                                         self.v, self.z, self.residuals)
                    decompacted = True
                else:
                    pl.average_peers(flat.peer_ptrs(), float(self.M), dst, tag="K8_leader_avg")
            else:
                dst = zhat if zhat is not None else self.flat
                self._dual(dst)
        else:
            self._dual(None)
        if self.P > 1:
            yield Barrier(self.intra, "zhat_bcast", k, root=self.leader_rank if _ONESIDED else None)
            if not self.is_leader:
                # the intra broadcast: decompact straight from the leader's payload over
                # NVLink (HSX_REMOTE_K7=0: copy it first)
                if _REMOTE_K7:
                    dst = self.p_zhat.peer_ptrs()[0]
                else:
                    pl.average_peers([self.p_zhat.peer_ptrs()[0]], 1.0, self.flat, tag="K8_zhat_read")
                    dst = self.flat
        if not decompacted:
            self._decompact(dst)
        return (yield from self._end_step(k, dynamic, ev, log_zsync=True))

    # -- phase-1 boundary ------------------------------------------------------------
    def send_buffer(self):
        """The intra-sum send buffer (theta + u) of this rank, or None when P == 1."""
        if self.P == 1:
            return None
        return self.p_send[self._send_idx].tensor if self.transport == "peer" else self.sum

    def prox_sgd_step(self, grad, lr: float, momentum: float, first: bool, last: bool = False):
        """One step of the reference's proximal SGD on this rank's theta (workloads.py:
        316-320): combined = grad + rho1 * (theta - z_node + u), velocity = momentum *
        velocity + combined, theta -= lr * velocity, fused over every layer with rho1
        from the (possibly adapted) device penalties. ``grad`` is a flat fp32 arena
        tensor. ``first`` starts the velocity at 0 (per outer iteration, :312); ``last``
        also writes theta + u into the intra-sum send buffer, so the next program
        skips K0."""
        if grad.dtype != torch.float32 or grad.numel() != self.plan.arena or not grad.is_cuda:
            raise ShapeError("grad must be a CUDA fp32 tensor of arena size")
        if getattr(self, "velocity", None) is None:
            self.velocity = self.plan.empty_arena(self.device)
        send = self.send_buffer() if last else None
        self.plan.prox_sgd_step(grad, self.theta, self.z_node, self.u, self.velocity, lr, momentum, first, send)
        self._send_packed = send is not None

    def _pack_send(self, buf):
        """K0 (theta + u into the send buffer) unless the last SGD step already wrote it."""
        if getattr(self, "_send_packed", False):
            self._send_packed = False
            return
        self.plan.pack_theta_u(self.theta, self.u, buf)

    # -- K6 / K7 with or without the fused residual sums -------------------------------
    def _dual(self, flat):
        """K6 (flat given: compaction + intra dual) or K6f (intra dual alone)."""
        pl = self.plan
        if self.residuals:
            pl.compact_dual_resid(self.theta, self.u, self.z_node, self.v, flat)
        elif flat is not None:
            pl.compact_dual(self.theta, self.u, self.z_node, self.v, flat)
        else:
            pl.dual_intra(self.theta, self.u, self.z_node)

    def _side_dual(self):
        """K6f on a side stream forked from the current one (joined at the end of the
        step by :meth:`_join_side`)."""
        cur = torch.cuda.current_stream(self.device)
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(self.device)
        fork = torch.cuda.Event()
        fork.record(cur)
        self._side.wait_event(fork)
        with torch.cuda.stream(self._side):
            self.plan.dual_intra(self.theta, self.u, self.z_node)
            done = torch.cuda.Event()
            done.record(self._side)
        self._side_done = done

    def _join_side(self):
        if getattr(self, "_side_done", None) is not None:
            torch.cuda.current_stream(self.device).wait_event(self._side_done)
            self._side_done = None

    def _local_sync(self):
        """K6 + K7 of a one-node cluster in one pass (HSX_LOCAL_SYNC=0: the two kernels)."""
        if os.environ.get("HSX_LOCAL_SYNC", "1") == "0":
            self._dual(self.flat)
            self._decompact(self.flat)
            return
        self.plan.local_sync(self.theta, self.u, self.z_node, self.v, self.z, self.z_node_prev, self.residuals)

    def _decompact(self, flat):
        if self.residuals:
            self.plan.decompact_dual_resid(flat, 1.0, self.z_node, self.z_node_prev, self.v, self.z)
        else:
            self.plan.decompact_dual(flat, 1.0, self.z_node, self.v, self.z)

    def _residual_phase(self, k: int, sync: bool):
        """Phase 5 after the u-update (consensus.py:537-598): per-layer squared norms
        (accumulated in K6 / K7), intra SUM, leaders' inter SUM, the report on the
        leader, broadcast to the followers, adaptive penalties + dual rescale."""
        if not self.residuals:
            return None
        pl = self.plan
        if not sync and self.is_leader:   # z, v unchanged: the leader's slots 3-8 (dz = 0)
            pl.decompact_dual_resid(None, 1.0, self.z_node, self.z_node_prev, self.v, self.z)
        pl.residual_fold(self.is_leader, self.rvec)
        if self.P > 1:
            yield AllReduce(self.intra, self.rvec, ReduceOp.SUM, "res_intra", k)
        if self.is_leader:
            if self.M > 1:
                yield AllReduce(self.inter, self.rvec, ReduceOp.SUM, "res_inter", k)
            pl.residual_report(self.rvec, self.report, self.scales, self._resid_params)
        if self.P > 1:
            yield Broadcast(self.intra, self.leader_rank, self.report, "report", k)
            if not self.is_leader:
                pl.residual_report(None, self.report, self.scales, self._resid_params)
        if self._resid_params.adapt:
            pl.scale_duals(self.scales, self.u, self.v)
        self.reported = True
        return None

    def set_residuals(self, on: bool, adapt: bool | None = None) -> None:
        """Turn phase 5 on / off between steps (adapt: override the schedule's flag)."""
        self.settle()
        self.residuals = bool(on)
        if self.residuals and self.z_node_prev is None:
            # split K1: the peer-mapped spare (K1 writes the peer's z_node buffer too)
            self.z_node_prev = self._zn_spare if getattr(self, "_split", False) else self.plan.empty_arena(self.device)
        if adapt is not None:
            self._resid_params.adapt = 1 if adapt else 0

    def check_barriers(self) -> None:
        """Raise ProtocolError if a device-side group barrier of this device gave up
        waiting for a peer (peer transport; synchronous device read)."""
        if self.transport != "peer":
            return
        n = _lib.barrier_timeouts(reset=True)
        if n:
            raise ProtocolError(f"{n} group barrier(s) timed out waiting for a peer rank "
                                "(HSX_BARRIER_TIMEOUT_S); the step's shared buffers are not valid")

    def last_report(self):
        """The last iteration's ResidualReport (consensus.py:84-91); synchronizes."""
        from .consensus import unpack_report

        if not self.reported:
            raise ProtocolError("no residual report yet (residuals off or no step run)")
        torch.cuda.current_stream(self.device).synchronize()
        return unpack_report(self.report.cpu().numpy(), self.names)

    def current_schedule(self) -> PenaltySchedule:
        """The penalty schedule after device-side adaptation (synchronizes)."""
        import dataclasses

        torch.cuda.current_stream(self.device).synchronize()
        r1, r2 = self.plan.read_penalties()
        return dataclasses.replace(self.schedule, rho1=dict(zip(self.names, r1)), rho2=dict(zip(self.names, r2)))

    def _end_step(self, k: int, dynamic: bool, ev, log_zsync: bool):
        """Phase 5; masks <- union; host bookkeeping now, or at the next step (defer_host)."""
        yield from self._residual_phase(k, sync=True)
        self.plan.join_fetch()
        self.plan.join_stage()
        self._join_side()
        if dynamic:
            self.masks, self.union = self.union, self.masks
        if ev is not None and self.defer_host:
            self._pending = (k, ev, log_zsync)
        else:
            if ev is not None:
                ev.synchronize()
                self._after_keep_sets()
            self._host_tail(k, dynamic, log_zsync)
        return None

    def _host_tail(self, k: int, dynamic: bool, log_zsync: bool):
        """Ledgers of the sync iteration; freeze + seal (consensus.py:600-606)."""
        if log_zsync and self.is_leader:
            self._log_zsync(k)
        self._log_reference(k, True, self.frozen)   # sync iterations only reach here
        if dynamic and freeze_check(k, self.settings.t_freeze, self.drift_history,
                                    self.settings.drift_window):
            self.frozen = True
            if self.is_leader:
                self.cache_hits += len(self.prunable)

    def settle(self) -> None:
        """Finish the deferred host bookkeeping of the last step (waits for its counts)."""
        if self._pending is None:
            return
        k, ev, log_zsync = self._pending
        self._pending = None
        ev.synchronize()
        self._after_keep_sets()
        self._host_tail(k, True, log_zsync)

    def _program_nccl(self, k: int):
        pl = self.plan
        frozen = self.frozen
        dynamic = not frozen and bool(self.prunable)
        # phase 2: intra-node sum of theta + u
        s = None
        if self.P > 1:
            self._pack_send(self.sum)
            s = yield AllReduce(self.intra, self.sum, ReduceOp.SUM, "theta_u", k)
        # phase 3: node candidate, projection or frozen mask
        pl.candidate(s, self.theta, self.u, self.z, self.v, self.z_node,
                     frozen_mask=self.masks if (frozen and self.prunable) else None)
        # one node: every rank's local mask is the union (identical z_node), so K3
        # derives the keep sets from the bits it writes (no exchange, no K5)
        fused_keep = dynamic and self.M == 1 and k % self.settings.sync_period == 0
        if fused_keep:
            pl.project_all(s, self.theta, self.u, self.z, self.v, self.z_node, self.union,
                           keep_prev=True, prev_mask=self.masks)
        elif dynamic:
            pl.project_all(s, self.theta, self.u, self.z, self.v, self.z_node, self.local_mask)
        if k % self.settings.sync_period != 0:
            self._dual(None)
            yield from self._residual_phase(k, sync=False)
            self._log_reference(k, False, self.frozen)
            return None
        # phase 4: mask union (leaders), broadcast to followers, keep sets
        ev = None
        if fused_keep:
            if not self._k67_chain:   # chained: fetched after K67 (K3 -> K67 consecutive launches)
                ev = pl.keep_sets_fetch_async()
        elif dynamic:
            if self.is_leader:
                yield AllGather(self.inter, self.local_mask, self.gathered, "mask_sync", k)
                mask_or(self.gathered, self.M, pl.mask_words, self.union)
            if self.P > 1:
                yield Broadcast(self.intra, self.leader_rank, self.union, "m_bcast", k)
            pl.keep_sets(self.union, self.masks)
            ev = pl.keep_sets_fetch_async()             # the one D2H of the dynamic step
        elif self.is_leader and self.prunable:
            self.cache_hits += len(self.prunable)
        if self.M == 1:
            # one node: no leader exchange; every rank runs K6+K7 locally (bitwise the
            # leader's compact round trip + broadcast), no mid-step host wait
            self._local_sync()
            if fused_keep and self._k67_chain:
                ev = pl.keep_sets_fetch_async()
            return (yield from self._end_step(k, dynamic, ev, log_zsync=True))
        # compaction fused with the intra dual update (K6 reads sizes on device, so
        # it runs while the host waits for the D2H and sizes the collectives); a leader
        # without phase 5 runs the intra dual on a side stream beside the collectives
        if self.is_leader and not self.residuals and _SPLIT_K6:
            pl.compact_dual(None, None, self.z_node, self.v, self.flat)
            self._side_dual()
        else:
            self._dual(self.flat if self.is_leader else None)
        collectives = self.M > 1 or self.P > 1
        if ev is not None and collectives:      # the leader all-reduce / broadcast need the sizes
            ev.synchronize()
            self._after_keep_sets()
            ev = None
        total = self.payload_elements
        if self.is_leader and collectives:
            yield from self._leader_average(k)
        if self.P > 1 and total > 0:
            yield Broadcast(self.intra, self.leader_rank, self.flat[:total], "zhat_bcast", k)
        self._decompact(self.flat)
        # one rank (no collectives): K6 / K7 are queued, the counts land meanwhile; the
        # leader average is the identity (ledger entries only)
        return (yield from self._end_step(k, dynamic, ev, log_zsync=not collectives))

    # -- host-buffer steps ---------------------------------------------------------------
    def step_host(self, k: int, theta_host: torch.Tensor, z_host: torch.Tensor | None = None):
        """Iteration k fed from, and returned to, pinned host memory (flat fp32 arenas).

        theta_host is copied in on a copy stream into one of two device theta
        buffers, the step runs on the current stream once it has landed, and z is
        copied out to z_host on a second copy stream (from one of two staging
        buffers). Host bookkeeping is deferred to the next call, so consecutive
        calls overlap: step k+1's input copy and step k's output copy run while
        the GPU computes. Returns the CUDA event after which z_host holds z(k);
        call :meth:`settle` before reading host-side state (drift, freeze, ledger).
        """
        if theta_host.is_cuda or theta_host.dtype != torch.float32 or theta_host.numel() != self.plan.arena:
            raise ShapeError("theta_host must be a host fp32 tensor of arena size")
        if z_host is not None and (z_host.is_cuda or z_host.dtype != torch.float32
                                   or z_host.numel() != self.plan.arena):
            raise ShapeError("z_host must be a host fp32 tensor of arena size")
        local = not hasattr(self.cluster, "run_rank")
        if local and self.topology.world_size != 1:
            raise ProtocolError("step_host runs one rank per engine: DistCluster, or a one-rank LocalCluster")
        if self._pipe is None:
            dev = self.device
            self._pipe = {
                "theta": [self.theta, self.plan.empty_arena(dev, fill_zero=False)],
                "zout": [self.plan.empty_arena(dev, fill_zero=False) for _ in range(2)],
                "h2d": torch.cuda.Stream(dev), "d2h": torch.cuda.Stream(dev),
                "free": [None, None],      # compute done with theta[b]
                "drained": [None, None],   # z_host copy out of zout[b] done
            }
        pp = self._pipe
        b = k & 1
        compute = torch.cuda.current_stream(self.device)
        # input copy: into the theta buffer the previous-but-one step used
        h2d = pp["h2d"]
        if pp["free"][b] is not None:
            h2d.wait_event(pp["free"][b])
        with torch.cuda.stream(h2d):
            pp["theta"][b].copy_(theta_host, non_blocking=True)
            landed = torch.cuda.Event()
            landed.record(h2d)
        self.theta = pp["theta"][b]
        compute.wait_event(landed)
        self.defer_host = True
        try:
            if local:
                self.cluster.run({self.rank: self.program(k)})
            else:
                self.cluster.run_rank(self.program(k))
        finally:
            self.defer_host = False
        free = torch.cuda.Event()
        free.record(compute)
        pp["free"][b] = free
        if z_host is None:
            return free
        # output copy from a staging buffer (the next step rewrites z)
        if pp["drained"][b] is not None:
            compute.wait_event(pp["drained"][b])
        pp["zout"][b].copy_(self.z)
        staged = torch.cuda.Event()
        staged.record(compute)
        d2h = pp["d2h"]
        d2h.wait_event(staged)
        with torch.cuda.stream(d2h):
            z_host.copy_(pp["zout"][b], non_blocking=True)
            drained = torch.cuda.Event()
            drained.record(d2h)
        pp["drained"][b] = drained
        return drained

    def _leader_average(self, k: int):
        """C3: leader all-reduce AVG of the flat buffer. The buckets (<= 32 MiB, the
        reference's z_sync/b{i} collectives, transport.py:239-280) are contiguous slices
        of the one flat buffer the compaction wrote, so they travel as one NCCL call
        over the whole payload (one launch and one ring pipeline instead of one per
        bucket; elementwise the same average) and are logged one ledger entry per
        bucket. HSX_NCCL_BUCKETS=1: one call per bucket."""
        if os.environ.get("HSX_NCCL_BUCKETS") == "1" or len(self.buckets) <= 1:
            for bi, b in enumerate(self.buckets):
                yield AllReduce(self.inter, self.flat[b.start:b.start + b.elements], ReduceOp.AVG,
                                f"z_sync/b{bi}", k, detail=b.detail)
            return
        total = sum(b.elements for b in self.buckets)
        parts = tuple((f"z_sync/b{bi}", b.elements, b.detail) for bi, b in enumerate(self.buckets))
        yield AllReduce(self.inter, self.flat[:total], ReduceOp.AVG, "z_sync", k, parts=parts)

    # -- CUDA-graph steps (one rank) -------------------------------------------------
    def graph_step(self, k: int):
        """Iteration k of a one-rank engine as a replay of a captured CUDA graph.

        The launches of a step depend only on (frozen, which mask buffer holds the
        current union, which theta buffer is live, sync or not); each combination is
        captured once from :meth:`program` under stream capture and replayed after,
        so a step costs one graph launch on the host. Host bookkeeping is deferred
        exactly as with ``defer_host`` (settled when the next step starts).
        """
        if self.topology.world_size != 1:
            raise ProtocolError("graph_step drives a one-rank engine (collectives are not captured)")
        self.settle()
        sync = k % self.settings.sync_period == 0
        dynamic = not self.frozen and bool(self.prunable)
        key = (dynamic, sync, self.masks.data_ptr(), self.theta.data_ptr(), self.z_node.data_ptr(),
               self.residuals, self._resid_params.adapt)
        graphs = self.__dict__.setdefault("_graphs", {})
        g = graphs.get(key)
        if g is None:
            g = torch.cuda.CUDAGraph()
            self.defer_host = True
            n0 = _lib.launch_count()
            try:
                with torch.cuda.graph(g, capture_error_mode="relaxed"):
                    self._run_program(k)   # host effects of step k applied once here
            finally:
                self.defer_host = False
            # captured launches went through the ABI counter once; replays add them again
            g = (g, _lib.launch_count() - n0)
            graphs[key] = g
            g[0].replay()
        else:
            self._graph_effects(k, dynamic, sync)
            g[0].replay()
            _lib.note_graph_replay(g[1])
        if self._pending is not None:
            # the summary copy is part of the graph and signals an external event
            # node right after it: the host resumes mid-replay
            from .plan import FetchDone

            self._pending = (self._pending[0], FetchDone(self.plan), self._pending[2])

    def _run_program(self, k: int):
        if hasattr(self.cluster, "run_rank"):
            return self.cluster.run_rank(self.program(k))
        return self.cluster.run({self.rank: self.program(k)})

    def _graph_effects(self, k: int, dynamic: bool, sync: bool):
        """Host side of program(k) for a replayed graph (one rank, deferred mode)."""
        self._begin_step()
        if self.residuals:
            self.reported = True
        if not sync:
            self._log_reference(k, False, self.frozen)
        if not sync:
            return
        if not dynamic:
            if self.is_leader and self.prunable:
                self.cache_hits += len(self.prunable)
            self._host_tail(k, False, log_zsync=True)
            return
        self.masks, self.union = self.union, self.masks
        self._pending = (k, None, True)

    def step(self, k: int):
        """Run iteration k through a DistCluster (one rank per process)."""
        if not hasattr(self.cluster, "run_rank"):
            raise ProtocolError("step() needs a DistCluster; use LocalCluster.run for in-process ranks")
        return self.cluster.run_rank(self.program(k))


def run_local(engines: list[HSADMMSync], k: int):
    """Run iteration k for every rank of a LocalCluster (single process, one GPU)."""
    cluster = engines[0].cluster
    if len(engines) != cluster.topology.world_size:
        raise ShapeError("need one engine per rank")
    return cluster.run({e.rank: e.program(k) for e in engines})
