"""Python handle of an ``hsx_plan`` (layer table + work lists + scratch on device).

A plan fixes the arena layout of a model: every fp32 state arena (theta, u,
z_node, v, z, the intra-sum buffer, the flat compact buffer) has the same
per-layer offsets (multiples of 32 elements), and every mask arena holds one
bit per element of each prunable layer.
"""

from __future__ import annotations

import contextlib
import os
import ctypes as C

import torch

from . import _lib
from .errors import ShapeError
from .layers import GROUP_CODE, GroupBy, LayerKind, LayerSpec


def current_stream() -> int:
    return torch.cuda.current_stream().cuda_stream


class KernelTimer:
    """CUDA-event timing of libhsx calls and collectives on the launching stream."""

    def __init__(self):
        self.events: dict[str, list] = {}

    @contextlib.contextmanager
    def __call__(self, name: str):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        try:
            yield
        finally:
            e.record()
            self.events.setdefault(name, []).append((s, e))

    def durations_ms(self) -> dict[str, list[float]]:
        torch.cuda.synchronize()
        return {k: [s.elapsed_time(e) for s, e in v] for k, v in self.events.items()}

    def reset(self):
        self.events.clear()


TIMER: KernelTimer | None = None
# what each timed collective call moved (bench's collectives block):
# name -> [(op, bytes, ranks)] in call order, parallel to TIMER.events[name]
NOTES: dict = {}


def timed(name: str):
    return TIMER(name) if TIMER is not None else contextlib.nullcontext()


def note(name: str, op: str, nbytes: int, ranks: int) -> None:
    """Record the payload of a timed collective (only while a KernelTimer is active)."""
    if TIMER is not None:
        NOTES.setdefault(name, []).append((op, int(nbytes), int(ranks)))


def ptr(t) -> int | None:
    """Device pointer of a tensor (an int is already one: a peer's mapped buffer)."""
    if t is None or isinstance(t, int):
        return t
    return t.data_ptr()


class Plan:
    """Owns one ``hsx_plan``; layer order is the caller's (reference) layer order."""

    def __init__(self, layers: list[LayerSpec], groups: dict[str, list[tuple[GroupBy, int]]],
                 rho1: dict[str, float] | None = None, rho2: dict[str, float] | None = None):
        lib = _lib.load()
        self.layers = list(layers)
        self.names = [ls.name for ls in layers]
        self.index = {n: i for i, n in enumerate(self.names)}
        self.groups = {n: list(groups.get(n, [])) for n in self.names}
        n = len(layers)
        descs = (_lib.LayerDesc * max(n, 1))()
        for i, ls in enumerate(layers):
            d = descs[i]
            shape = ls.shape
            d.rank = len(shape)
            for j in range(4):
                d.shape[j] = shape[j] if j < len(shape) else 1
            g = self.groups[ls.name]
            if g and ls.kind is not LayerKind.CONV:
                raise ShapeError(f"layer {ls.name}: only conv layers are prunable")
            d.n_constraints = len(g)
            for j, (grp, keep) in enumerate(g):
                d.group[j] = GROUP_CODE[grp]
                d.keep[j] = int(keep)
            d.rho1 = float((rho1 or {}).get(ls.name, 1.0))
            d.rho2 = float((rho2 or {}).get(ls.name, 0.0))
        h = C.c_void_p()
        _lib.check(lib.hsx_plan_create(descs, n, C.byref(h)), "hsx_plan_create")
        self._h = h
        self._lib = lib
        self.arena = int(lib.hsx_plan_arena_elements(h))
        self.offsets = [int(lib.hsx_plan_layer_offset(h, i)) for i in range(n)]
        self.mask_words = int(lib.hsx_plan_mask_words(h))
        self.mask_offsets = [int(lib.hsx_plan_mask_word_offset(h, i)) for i in range(n)]
        self.max_passes = int(lib.hsx_plan_max_passes(h))
        self.prunable = [i for i, ls in enumerate(layers) if self.groups[ls.name]]
        self._fetch_stream = None
        self._fetch_done = None
        self.summary_host = torch.zeros(n * _lib.SUM_COLS + 1, dtype=torch.int64).pin_memory() \
            if torch.cuda.is_available() else torch.zeros(n * _lib.SUM_COLS + 1, dtype=torch.int64)

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.hsx_plan_destroy(h)
            self._h = C.c_void_p()

    # -- configuration ---------------------------------------------------------
    def set_single_node(self, on: bool):
        """Structured keep sets in the selection tail (one node: the union is the local mask)."""
        _lib.call("hsx_plan_set_single_node", self._h, 1 if on else 0)

    def set_k67_chain(self, on: bool):
        """One node: the projection chains into K67 (hsx_plan_set_k67_chain); every
        project_keep_sets must then be followed by local_sync. The keep-set summary
        then lives in the plan's mapped host buffer, published by the device."""
        _lib.call("hsx_plan_set_k67_chain", self._h, 1 if on else 0)
        if on:
            import numpy as np

            buf = self._lib.hsx_plan_summary_host(self._h)
            if buf:
                n = len(self.names) * _lib.SUM_COLS + 1
                self.summary_host = torch.from_numpy(np.ctypeslib.as_array(buf, shape=(n,)))

    def set_order(self, big_first: bool):
        """Work-list order (hsx_plan_set_order): costliest selections first, or layer order."""
        _lib.call("hsx_plan_set_order", self._h, 1 if big_first else 0)

    def set_penalties(self, rho1: dict | None, rho2: dict | None, weight_decay: float,
                      num_nodes: int, accels_per_node: int, identity: bool = False):
        def arr(d):
            if d is None:
                return None
            a = (C.c_double * len(self.names))(*[float(d[n]) for n in self.names])
            return C.cast(a, C.c_void_p), a

        r1, r2 = arr(rho1), arr(rho2)
        _lib.check(self._lib.hsx_plan_set_penalties(
            self._h, r1[0] if r1 else None, r2[0] if r2 else None, float(weight_decay),
            int(num_nodes), int(accels_per_node), int(identity)), "set_penalties")

    # -- arena helpers -----------------------------------------------------------
    def empty_arena(self, device, fill_zero=True):
        t = torch.zeros(self.arena, dtype=torch.float32, device=device)
        return t

    def empty_mask(self, device, ones=False, count: int = 1):
        shape = (count, self.mask_words) if count > 1 else (self.mask_words,)
        t = torch.zeros(shape, dtype=torch.int32, device=device)
        if ones:
            self.fill_ones(t.view(-1, self.mask_words)[0] if count > 1 else t)
        return t

    def fill_ones(self, mask):
        """All-ones global masks (reference consensus.py:418), padding bits clear."""
        for i in self.prunable:
            n = self.layers[i].elements
            w0 = self.mask_offsets[i]
            full, rem = divmod(n, 32)
            mask[w0:w0 + full].fill_(-1)
            if rem:
                mask[w0 + full].fill_((1 << rem) - 1)
        return mask

    def view(self, arena, i: int):
        ls = self.layers[i]
        o = self.offsets[i]
        return arena[o:o + ls.elements].view(ls.shape)

    def views(self, arena) -> dict:
        return {n: self.view(arena, i) for i, n in enumerate(self.names)}

    def load_arena(self, arena, values: dict):
        for i, n in enumerate(self.names):
            self.view(arena, i).copy_(torch.as_tensor(values[n]).to(arena.device, torch.float32)
                                      .view(self.layers[i].shape))

    def mask_view_words(self, mask, i: int):
        n = self.layers[i].elements
        w0 = self.mask_offsets[i]
        return mask[w0:w0 + (n + 31) // 32]

    def unpack_mask(self, mask, i: int):
        """Bool tensor of layer i's mask bits (hsx_unpack_bits)."""
        ls = self.layers[i]
        out = torch.empty(ls.shape, dtype=torch.bool, device=mask.device)
        words = self.mask_view_words(mask, i)
        _lib.call("hsx_unpack_bits", words.data_ptr(), ls.elements, out.data_ptr(), current_stream())
        return out

    # -- kernels (thin wrappers; all on the current stream) ---------------------
    def pack_theta_u(self, theta, u, send):
        with timed("K0_pack_theta_u"):
            _lib.call("hsx_pack_theta_u", self._h, ptr(theta), ptr(u), ptr(send), current_stream())

    def candidate(self, s, theta, u, z, v, z_node, frozen_mask=None):
        with timed("K1_candidate"):
            _lib.call("hsx_candidate", self._h, ptr(s), ptr(theta), ptr(u), ptr(z), ptr(v), ptr(z_node),
                      ptr(frozen_mask), current_stream())

    def candidate_peers(self, sends: list[int], z, v, z_node, frozen_mask=None):
        arr, keep = _lib.ptr_array(sends)
        with timed("K1_candidate"):
            _lib.call("hsx_candidate_peers", self._h, arr, len(sends), ptr(z), ptr(v), ptr(z_node),
                      ptr(frozen_mask), current_stream())
        del keep

    def candidate_dist(self, slices: list[int], z, v, z_node, frozen_mask=None):
        """K1 reading the intra sum from the P ranks' reduce-scatter slices over NVLink
        (hsx_candidate_dist; replaces the all-gather of S and the local K1 on it)."""
        arr, keep = _lib.ptr_array(slices)
        with timed("K1_candidate"):
            _lib.call("hsx_candidate_dist", self._h, arr, len(slices), ptr(z), ptr(v), ptr(z_node),
                      ptr(frozen_mask), current_stream())
        del keep

    def split_sizes(self) -> tuple[int, int]:
        """(partials doubles, tile counters) of a split two-rank K1 (hsx_plan_split_sizes)."""
        import ctypes as C

        n, c = C.c_int64(0), C.c_int32(0)
        _lib.call("hsx_plan_split_sizes", self._h, C.byref(n), C.byref(c))
        return int(n.value), int(c.value)

    def set_split(self, me: int, partials: int, partials_peer: int, counts: int, counts_peer: int):
        """Install the peer-mapped partials / tile counts of a split K1 (hsx_plan_set_split)."""
        _lib.call("hsx_plan_set_split", self._h, int(me), ptr(partials), ptr(partials_peer), ptr(counts),
                  ptr(counts_peer))

    def candidate_peers_split(self, sends: list[int], z, v, z_node, z_node_peer: int):
        """K1 of half the prunable tiles (and every dense item) of a two-rank node,
        writing z_node / partials / tile counts to both ranks (hsx_candidate_peers_split)."""
        arr, keep = _lib.ptr_array(sends)
        with timed("K1_candidate"):
            _lib.call("hsx_candidate_peers_split", self._h, arr, len(sends), ptr(z), ptr(v), ptr(z_node),
                      ptr(z_node_peer), current_stream())
        del keep

    def set_peer_staging(self, on: bool):
        """Allocate the staged-peer-operand buffers (hsx_plan_set_peer_staging)."""
        _lib.call("hsx_plan_set_peer_staging", self._h, 1 if on else 0)

    def candidate_peers_staged(self, sends: list[int], me: int, z, v, z_node):
        """K1 for two ranks with the peer's send staged into local memory by a copy
        kernel on a side stream (forked here, joined by :meth:`join_stage`)."""
        cur = torch.cuda.current_stream()
        if getattr(self, "_stage_stream", None) is None:
            self._stage_stream = torch.cuda.Stream(cur.device)
            self._stage_done = None
        side = self._stage_stream
        fork = torch.cuda.Event()
        fork.record(cur)
        side.wait_event(fork)
        arr, keep = _lib.ptr_array(sends)
        with timed("K1_candidate"):
            _lib.call("hsx_candidate_peers_staged", self._h, arr, len(sends), int(me), ptr(z), ptr(v), ptr(z_node),
                      current_stream(), side.cuda_stream)
        del keep
        done = torch.cuda.Event()
        done.record(side)
        self._stage_done = done

    def join_stage(self):
        """The current stream waits for the last staging copy (end of a step; also
        closes the side branch under CUDA-graph capture)."""
        if getattr(self, "_stage_done", None) is not None:
            torch.cuda.current_stream().wait_event(self._stage_done)
            self._stage_done = None

    def average_peers(self, srcs: list[int], divisor, out, tag="C_avg"):
        """out[:payload] = rank-order average of the buffers at srcs (payload size on device)."""
        arr, keep = _lib.ptr_array(srcs)
        with timed(tag):
            _lib.call("hsx_average_peers", self._h, arr, len(srcs), float(divisor), ptr(out),
                      current_stream())
        del keep

    def slices_peers(self, srcs: list[int], part: int, divisor, payload: bool, out, tag):
        """part >= 0: slice ``part`` of the rank-order average; part < 0: gather all slices."""
        arr, keep = _lib.ptr_array(srcs)
        with timed(tag):
            _lib.call("hsx_slices_peers", self._h, arr, len(srcs), int(part), float(divisor), int(payload),
                      ptr(out), current_stream())
        del keep

    def renorm(self, p, s, theta, u, z, v):
        with timed("K1r_renorm"):
            _lib.call("hsx_candidate_renorm", self._h, p, ptr(s), ptr(theta), ptr(u), ptr(z), ptr(v),
                      current_stream())

    def select(self, p):
        with timed("K2_select"):
            _lib.call("hsx_select", self._h, p, current_stream())

    def project(self, z_node, local_mask):
        with timed("K3_project"):
            _lib.call("hsx_project", self._h, ptr(z_node), ptr(local_mask), current_stream())

    def project_keep_sets(self, z_node, mask, prev_mask=None):
        """K3 + K5 in one launch (one node: the union is the local mask)."""
        with timed("K3_project_keep"):
            _lib.call("hsx_project_keep_sets", self._h, ptr(z_node), ptr(mask), ptr(prev_mask),
                      current_stream())

    def project_all(self, s, theta, u, z, v, z_node, local_mask, peers=None, keep_prev=False,
                    prev_mask=None):
        """K2 (+ composite passes) + K3 after hsx_candidate (peers: the sends of
        hsx_candidate_peers, re-read by composite passes). keep_prev: K3 also derives
        the keep sets from the mask it writes (hsx_project_keep_sets, prev_mask for
        the drift count)."""
        if keep_prev and self.max_passes == 1 and os.environ.get("HSX_MERGE_SELECT_PROJECT") == "1":
            # one node, single-constraint plan: selection, projection and fixup in one launch
            with timed("K2K3_select_project_keep"):
                _lib.call("hsx_select_project_keep_sets", self._h, ptr(z_node), ptr(local_mask), ptr(prev_mask),
                          current_stream())
            return
        for p in range(self.max_passes):
            if p > 0:
                if peers:
                    arr, keep = _lib.ptr_array(peers)
                    with timed("K1r_renorm"):
                        _lib.call("hsx_candidate_renorm_peers", self._h, p, arr, len(peers), ptr(z), ptr(v),
                                  current_stream())
                    del keep
                else:
                    self.renorm(p, s, theta, u, z, v)
            self.select(p)
        if keep_prev:
            self.project_keep_sets(z_node, local_mask, prev_mask)
        else:
            self.project(z_node, local_mask)

    def group_norms(self, p: int, device):
        total = int(self._lib.hsx_plan_group_total(self._h, p))
        norms = torch.empty(total, dtype=torch.float64, device=device)
        flags = torch.empty(total, dtype=torch.uint8, device=device)
        _lib.call("hsx_read_groups", self._h, p, ptr(norms), ptr(flags), current_stream())
        return norms, flags

    def group_offset(self, i: int, p: int) -> int:
        return int(self._lib.hsx_plan_group_offset(self._h, i, p))

    def keep_sets(self, union_mask, prev_mask=None):
        with timed("K5_keep_sets"):
            _lib.call("hsx_keep_sets", self._h, ptr(union_mask), ptr(prev_mask), current_stream())

    def keep_sets_ptrs(self, srcs: list[int], union_out, prev_mask=None):
        """K5 with the union formed on the fly: OR of the leaders' mask bits ``srcs``
        (peer pointers), stored to ``union_out`` (hsx_keep_sets_ptrs)."""
        arr, keep = _lib.ptr_array(srcs)
        with timed("K5_keep_sets"):
            _lib.call("hsx_keep_sets_ptrs", self._h, arr, len(srcs), ptr(union_out), ptr(prev_mask),
                      current_stream())
        del keep

    def keep_sets_fetch(self):
        """D2H of the per-layer summary; synchronizes the current stream."""
        _lib.call("hsx_keep_sets_fetch", self._h, self.summary_host.data_ptr(), current_stream())
        return self.summary_host.view(-1)

    def keep_sets_fetch_async(self):
        """Enqueue the D2H of the summary on a side stream (forked from the current
        stream after the keep-set kernels), so the compaction launched next does not
        queue behind a copy-engine transfer; returns the CUDA event to wait on.
        :meth:`join_fetch` joins the side stream back before the summary is rewritten."""
        cur = torch.cuda.current_stream()
        if self._fetch_stream is None:
            self._fetch_stream = torch.cuda.Stream(cur.device)
        fs = self._fetch_stream
        ready = torch.cuda.Event()
        ready.record(cur)
        fs.wait_event(ready)
        _lib.call("hsx_keep_sets_fetch_async", self._h, self.summary_host.data_ptr(), fs.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(fs)
        self._fetch_done = ev
        return FetchDone(self)

    def join_fetch(self):
        """Current stream waits for the last summary copy (end of a step; also closes
        the fork under CUDA-graph capture)."""
        if self._fetch_done is not None:
            torch.cuda.current_stream().wait_event(self._fetch_done)
            self._fetch_done = None

    def summary_np(self):
        """(per-layer rows as a zero-copy numpy view, total payload elements)."""
        a = self.summary_host.numpy()
        n = len(self.names)
        return a[: n * _lib.SUM_COLS].reshape(n, _lib.SUM_COLS), int(a[n * _lib.SUM_COLS])

    def summary_rows(self):
        s = self.summary_host
        n = len(self.names)
        return s[: n * _lib.SUM_COLS].view(n, _lib.SUM_COLS), int(s[n * _lib.SUM_COLS])

    def keep_positions(self, device):
        out = []
        for which in (0, 1):
            n = int(self._lib.hsx_plan_keep_total(self._h, which))
            t = torch.empty(n, dtype=torch.int32, device=device)
            _lib.call("hsx_read_keep_positions", self._h, which, ptr(t), current_stream())
            out.append(t)
        return out

    def keep_offset(self, i: int, which: int) -> int:
        return int(self._lib.hsx_plan_keep_offset(self._h, i, which))

    def set_keep_sets(self, i: int, k_out, k_in):
        ko = (C.c_int32 * max(len(k_out), 1))(*k_out)
        ki = (C.c_int32 * max(len(k_in), 1))(*k_in)
        _lib.call("hsx_set_keep_sets", self._h, i, C.cast(ko, C.c_void_p), len(k_out),
                  C.cast(ki, C.c_void_p), len(k_in))

    def compact_dual(self, theta, u, z_node, v, flat):
        with timed("K6_compact_dual"):
            _lib.call("hsx_compact_dual", self._h, ptr(theta), ptr(u), ptr(z_node), ptr(v), ptr(flat),
                      current_stream())

    def dual_intra(self, theta, u, z_node):
        with timed("K6f_dual_intra"):
            _lib.call("hsx_dual_intra", self._h, ptr(theta), ptr(u), ptr(z_node), current_stream())

    def decompact_dual(self, flat, divisor, z_node, v, z):
        with timed("K7_decompact_dual"):
            _lib.call("hsx_decompact_dual", self._h, ptr(flat), float(divisor), ptr(z_node), ptr(v),
                      ptr(z), current_stream())


    # -- phase 5 (consensus.py:537-598) ----------------------------------------------
    def compact_dual_resid(self, theta, u, z_node, v, flat):
        """K6 (flat given) or K6f (flat None) + per-item residual slots 0-2."""
        with timed("K6_compact_dual_resid" if flat is not None else "K6f_dual_intra_resid"):
            _lib.call("hsx_compact_dual_resid", self._h, ptr(theta), ptr(u), ptr(z_node), ptr(v), ptr(flat),
                      current_stream())

    def decompact_dual_resid(self, flat, divisor, z_node, z_node_prev, v, z):
        """K7 (flat given) or the non-sync residual pass (flat None) + slots 3-8."""
        with timed("K7_decompact_dual_resid" if flat is not None else "K7r_residuals"):
            _lib.call("hsx_decompact_dual_resid", self._h, ptr(flat), float(divisor), ptr(z_node),
                      ptr(z_node_prev), ptr(v), ptr(z), current_stream())

    def decompact_average(self, srcs: list[int], divisor, zhat_out, z_node, z_node_prev, v, z, residuals):
        """F1: the two leaders' average fused into K7 (optionally writing the averaged
        payload to zhat_out for the followers)."""
        arr, keep = _lib.ptr_array(srcs)
        with timed("K78_average_decompact"):
            _lib.call("hsx_decompact_average", self._h, arr, len(srcs), float(divisor), ptr(zhat_out), ptr(z_node),
                      ptr(z_node_prev), ptr(v), ptr(z), 1 if residuals else 0, current_stream())
        del keep

    def local_sync(self, theta, u, z_node, v, z, z_node_prev=None, residuals=False):
        """K6 + K7 of one node in one pass (no compact buffer)."""
        with timed("K67_local_sync"):
            _lib.call("hsx_local_sync", self._h, ptr(theta), ptr(u), ptr(z_node), ptr(v), ptr(z), ptr(z_node_prev),
                      1 if residuals else 0, current_stream())

    def residual_fold(self, leader: bool, vec):
        with timed("K9_residual_fold"):
            _lib.call("hsx_residual_fold", self._h, 1 if leader else 0, ptr(vec), current_stream())

    def residual_report(self, global_sums, report, scales, params):
        with timed("K9_report"):
            _lib.call("hsx_residual_report", self._h, ptr(global_sums), ptr(report), ptr(scales),
                      C.byref(params), current_stream())

    def scale_duals(self, scales, u, v):
        with timed("K9_scale_duals"):
            _lib.call("hsx_scale_duals", self._h, ptr(scales), ptr(u), ptr(v), current_stream())

    def prox_sgd_step(self, grad, theta, z_node, u, velocity, lr, momentum, first, send=None):
        with timed("P1_prox_sgd"):
            _lib.call("hsx_prox_sgd_step", self._h, ptr(grad), ptr(theta), ptr(z_node), ptr(u), ptr(velocity),
                      float(lr), float(momentum), 1 if first else 0, ptr(send), current_stream())

    def read_penalties(self):
        """(rho1, rho2) per layer as currently in the device layer table (synchronous)."""
        n = len(self.names)
        r1, r2 = (C.c_double * n)(), (C.c_double * n)()
        _lib.call("hsx_plan_read_penalties", self._h, C.cast(r1, C.c_void_p), C.cast(r2, C.c_void_p))
        return list(r1), list(r2)


class FetchDone:
    """Host-side wait for the plan's last summary copy (works for graph replays too)."""

    def __init__(self, plan):
        self.plan = plan

    def synchronize(self):
        _lib.call("hsx_keep_sets_fetch_wait", self.plan._h)


def mask_or_ptrs(srcs: list[int], words: int, out):
    """out = OR of the masks at device pointers ``srcs`` (one source = a copy)."""
    arr, keep = _lib.ptr_array(srcs)
    with timed("K4_mask_or"):
        _lib.call("hsx_mask_or_ptrs", arr, len(srcs), int(words), ptr(out), current_stream())
    del keep


def mask_or(gathered, n_ranks: int, words: int, out):
    with timed("K4_mask_or"):
        _lib.call("hsx_mask_or", ptr(gathered), int(n_ranks), int(words), ptr(out), current_stream())
