"""CPU ORACLE for the H-SADMM synchronization step — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this module, and only as the checker or the
timed CPU baseline. The product (``paper_2512_14628_b200``) never imports it
and has no CPU fallback.

What it is: a float64 numpy restatement of the reference algorithm for the
sync step of ``admmprune`` 0.1.0 — phases 2-4 and the ``u``-update of phase 5
of ``hierarchical_program`` (/root/reference/pkg/src/admmprune/consensus.py:436-535)
plus the freeze/seal bookkeeping (:600-606) — and of the helpers it calls.
Each function cites the reference file:line it follows. The residual block,
residual report and penalty adaptation of phase 5 (:537-598, :189-219,
:239-288) are restated too (``cluster_sync(...,
residuals=True, sched=Schedule(...))``) and pinned by the adaptive end-to-end
goldens (``tests/golden/e2e_adapt_*.npz``).

Pinning: ``tests/test_oracle.py`` checks every function here against
(a) the reference's own known-answer tests restated (tie -> lower index,
ceil rounding, gamma = 3.2e-3, payload 36864/147456/73728, brute-force
projection, ...) and (b) golden vectors produced by running the real
reference (``tests/golden/make_golden.py`` imports ``admmprune`` from
/root/reference and writes ``tests/golden/*.npz``), including multi-iteration
end-to-end runs of ``run_hierarchical`` on 1x1, 2x1 and 2x2 topologies.
The oracle reproduces those vectors bit-for-bit (same fp64 operation order).

numpy is the only third-party arithmetic (pairwise summation inside
``np.sum``); it is what the reference itself uses (pkg/pyproject.toml:10).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

FILTER, CHANNEL, SHAPE = "filter", "channel", "shape"
ELEMENT_BYTES = 4                       # transport.py:32 (fp32 wire accounting)
BUCKET_CAP_BYTES = 32 * 1024 * 1024     # transport.py:33

# -- group norms / projection (tensors.py:75-93, sparsity.py:53-115) ---------

_REDUCE_AXES = {FILTER: (1, 2, 3), CHANNEL: (0, 2, 3), SHAPE: (0,)}


def group_norms(t: np.ndarray, group: str) -> np.ndarray:
    """sqrt of the sum of squares over the non-group axes (tensors.py:75-93)."""
    t = np.asarray(t, dtype=np.float64)
    assert t.ndim == 4
    return np.sqrt((t * t).sum(axis=_REDUCE_AXES[group])).ravel()


def resolve_keep(group_count: int, keep_count=None, keep_rate=None) -> int:
    """k = keep_count or ceil(keep_rate * G) as a Python float (sparsity.py:53-62)."""
    k = int(keep_count) if keep_count is not None else int(math.ceil(keep_rate * group_count))
    if k > group_count:
        raise ValueError(f"keep {k} exceeds group count {group_count}")
    return k


def keep_flags(norms: np.ndarray, keep: int) -> np.ndarray:
    """Boolean flags of the ``keep`` largest norms, lower index on ties.

    Same selection as a stable argsort of ``-norms`` truncated to ``keep``
    (sparsity.py:65-68).
    """
    order = np.argsort(-norms, kind="stable")
    flags = np.zeros(norms.size, dtype=bool)
    flags[order[:keep]] = True
    return flags


def group_broadcast(flags: np.ndarray, shape: tuple, group: str) -> np.ndarray:
    """Expand per-group flags to an elementwise indicator of ``shape``."""
    if group == FILTER:
        return np.broadcast_to(flags.reshape(-1, 1, 1, 1), shape)
    if group == CHANNEL:
        return np.broadcast_to(flags.reshape(1, -1, 1, 1), shape)
    return np.broadcast_to(flags.reshape(1, *shape[1:]), shape)


def project(t: np.ndarray, group: str, keep: int) -> np.ndarray:
    """Zero every group outside the top-``keep`` set; survivors untouched (sparsity.py:71-94)."""
    t = np.asarray(t, dtype=np.float64)
    flags = keep_flags(group_norms(t, group), keep)
    return np.where(group_broadcast(flags, t.shape, group), t, 0.0)


def project_composite(t: np.ndarray, plan: list[tuple[str, int]]) -> np.ndarray:
    """Sequential projections in listed order, norms recomputed each time (sparsity.py:97-110)."""
    out = np.array(t, dtype=np.float64, copy=True)
    for group, keep in plan:
        out = project(out, group, keep)
    return out


def extract_mask(t: np.ndarray) -> np.ndarray:
    return np.abs(t) > 0.0          # sparsity.py:113-115


def mask_drift(prev: np.ndarray, cur: np.ndarray) -> float:
    return float(np.mean(prev != cur))   # sparsity.py:118-122


# -- shrinkage (shrinkage.py:45-98) --------------------------------------------


def derive_keep_sets(mask: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(K_out, K_in): filters / channels with any set bit (shrinkage.py:45-58)."""
    return (np.flatnonzero(mask.any(axis=(1, 2, 3))), np.flatnonzero(mask.any(axis=(0, 2, 3))))


def compress(dense: np.ndarray, k_out: np.ndarray, k_in: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(dense[np.ix_(k_out, k_in)])       # shrinkage.py:61-68


def decompress(compact: np.ndarray, k_out, k_in, full_shape) -> np.ndarray:
    full = np.zeros(full_shape, dtype=np.float64)                  # shrinkage.py:71-82
    if len(k_out) and len(k_in):
        full[np.ix_(k_out, k_in)] = compact.reshape(len(k_out), len(k_in), *full_shape[2:])
    return full


def bucket_layout(sizes: list[tuple[str, int]], cap_bytes: int = BUCKET_CAP_BYTES):
    """Greedy <= cap buckets, never splitting a payload (transport.py:239-280).

    Returns a list of buckets, each a tuple of (name, offset, elements)."""
    buckets, cur, cur_bytes = [], [], 0

    def close():
        nonlocal cur, cur_bytes
        if cur:
            off, lay = 0, []
            for name, n in cur:
                lay.append((name, off, n))
                off += n
            buckets.append(tuple(lay))
        cur, cur_bytes = [], 0

    for name, n in sizes:
        nbytes = n * ELEMENT_BYTES
        if nbytes > cap_bytes:           # oversize payload gets its own bucket
            close()
            cur, cur_bytes = [(name, n)], nbytes
            close()
            continue
        if cur_bytes + nbytes > cap_bytes:
            close()
        cur.append((name, n))
        cur_bytes += nbytes
    close()
    return buckets


# -- update rules (consensus.py:142-186, 222-228) --------------------------------


def candidate_gamma(rho1, rho2, weight_decay, num_nodes, accels_per_node) -> float:
    return weight_decay / num_nodes + accels_per_node * rho1 + rho2      # consensus.py:157


def node_candidate(s, z, v, rho1, rho2, weight_decay, num_nodes, accels_per_node):
    gamma = candidate_gamma(rho1, rho2, weight_decay, num_nodes, accels_per_node)
    if gamma <= 0.0:
        raise ValueError(f"non-positive gamma {gamma}")
    return (rho1 * s + rho2 * (z - v)) / gamma                            # consensus.py:160


def dual_update_intra(theta, z_node, u):
    return u + (theta - z_node)                                           # consensus.py:186


def freeze_check(k, t_freeze, drift_history, window=3) -> bool:
    if k >= t_freeze:                                                     # consensus.py:222-228
        return True
    return window > 0 and len(drift_history) >= window and all(
        d == 0.0 for d in drift_history[-window:])


# -- residuals, report, penalty adaptation (consensus.py:189-219, 239-288, 537-598)

INTER_SLOTS = 9      # consensus.py:235
REPORT_SLOTS = 8     # consensus.py:236


def sq(a) -> float:
    return float(np.sum(a * a))                                           # consensus.py:382-383


@dataclass
class Schedule:
    """PenaltySchedule (consensus.py:42-69) as a mutable record; rho1 / rho2 are the
    dicts cluster_sync reads, so adaptation carries into the next iteration."""
    rho1: dict
    rho2: dict
    rho1_max: float = 10.0
    rho2_max: float = 10.0
    mu: float = 10.0
    tau_inc: float = 2.0
    tau_dec: float = 2.0
    adapt: bool = True


def build_residual_report(layers, g, sched: Schedule, num_nodes, per_node, eps_abs, eps_rel):
    """consensus.py:239-288: per-layer (r_intra, s_intra, r_inter, s_inter, eps_pri_intra,
    eps_dual_intra, eps_pri_inter, eps_dual_inter) and (r_pri, r_dual, eps_pri, eps_dual,
    converged) from the globally summed squared norms g[l * 9 + slot]."""
    world = num_nodes * per_node
    per_layer = {}
    r_pri_sq = r_dual_sq = eps_pri_sq = eps_dual_sq = 0.0
    for li, ly in enumerate(layers):
        gl = g[li * INTER_SLOTS:(li + 1) * INTER_SLOTS]
        rho1, rho2 = sched.rho1[ly.name], sched.rho2[ly.name]
        n = int(np.prod(ly.shape))
        r_intra = math.sqrt(gl[0])
        s_intra = rho1 * math.sqrt(per_node * gl[4])
        r_inter = math.sqrt(gl[3])
        s_inter = rho2 * math.sqrt(gl[7])
        eps_pri_intra = math.sqrt(n * world) * eps_abs + eps_rel * max(math.sqrt(gl[1]),
                                                                       math.sqrt(per_node * gl[5]))
        eps_dual_intra = math.sqrt(n * world) * eps_abs + eps_rel * rho1 * math.sqrt(gl[2])
        eps_pri_inter = math.sqrt(n * num_nodes) * eps_abs + eps_rel * max(math.sqrt(gl[5]), math.sqrt(gl[8]))
        eps_dual_inter = math.sqrt(n * num_nodes) * eps_abs + eps_rel * rho2 * math.sqrt(gl[6])
        per_layer[ly.name] = (r_intra, s_intra, r_inter, s_inter,
                              eps_pri_intra, eps_dual_intra, eps_pri_inter, eps_dual_inter)
        r_pri_sq += r_intra ** 2 + r_inter ** 2
        r_dual_sq += s_intra ** 2 + s_inter ** 2
        eps_pri_sq += eps_pri_intra ** 2 + eps_pri_inter ** 2
        eps_dual_sq += eps_dual_intra ** 2 + eps_dual_inter ** 2
    r_pri, r_dual = math.sqrt(r_pri_sq), math.sqrt(r_dual_sq)
    eps_pri, eps_dual = math.sqrt(eps_pri_sq), math.sqrt(eps_dual_sq)
    return {"layers": per_layer, "r_pri": r_pri, "r_dual": r_dual, "eps_pri": eps_pri,
            "eps_dual": eps_dual, "converged": r_pri <= eps_pri and r_dual <= eps_dual}


def adapt_penalties(report, sched: Schedule):
    """consensus.py:189-219, in place on sched; returns (u_scale, v_scale) per layer."""
    u_scale, v_scale = {}, {}
    for name in list(sched.rho1):
        r_intra, s_intra, r_inter, s_inter = report["layers"][name][:4]
        old = sched.rho1[name]
        if r_intra > sched.mu * s_intra:
            sched.rho1[name] = min(old * sched.tau_inc, sched.rho1_max)
        elif s_intra > sched.mu * r_intra:
            sched.rho1[name] = old / sched.tau_dec
        u_scale[name] = old / sched.rho1[name] if sched.rho1[name] != old else 1.0
        old2 = sched.rho2[name]
        if r_inter > sched.mu * s_inter:
            sched.rho2[name] = min(old2 * sched.tau_inc, sched.rho2_max)
        elif s_inter > sched.mu * r_inter:
            sched.rho2[name] = old2 / sched.tau_dec
        v_scale[name] = old2 / sched.rho2[name] if sched.rho2[name] != old2 else 1.0
    return u_scale, v_scale


def residual_phase(layers, states, zn_prev, z_prev, sync_iter, num_nodes, per_node, sched,
                   eps_abs, eps_rel):
    """consensus.py:537-598 for every rank (after the u-update): squared norms, intra
    SUM (rank order), leaders' 9-slot vectors, inter SUM (leader order), report,
    adaptation with the u / v rescaling. Returns (report, r_intra per rank)."""
    names = [ly.name for ly in layers]
    vec3 = {}
    r_intra_local = {}
    for r, st in enumerate(states):
        v3 = np.empty(len(names) * 3)
        for li, n in enumerate(names):
            d = st.theta[n] - st.z_node[n]
            v3[li * 3:li * 3 + 3] = (sq(d), sq(st.theta[n]), sq(st.u[n]))
        vec3[r] = v3
        r_intra_local[r] = {n: math.sqrt(v3[li * 3]) for li, n in enumerate(names)}
    leaders = [i * per_node for i in range(num_nodes)]
    vec9 = {}
    for i, lr in enumerate(leaders):
        node = vec3[lr].copy()
        for r in range(lr + 1, lr + per_node):
            node = node + vec3[r]
        st = states[lr]
        v9 = np.empty(len(names) * INTER_SLOTS)
        for li, n in enumerate(names):
            dz = st.z[n] - z_prev[lr][n] if sync_iter else np.zeros_like(st.z[n])
            v9[li * INTER_SLOTS:(li + 1) * INTER_SLOTS] = (
                node[li * 3], node[li * 3 + 1], node[li * 3 + 2],
                sq(st.z_node[n] - st.z[n]), sq(st.z_node[n] - zn_prev[lr][n]), sq(st.z_node[n]),
                sq(st.v[n]), sq(dz), sq(st.z[n]))
        vec9[lr] = v9
    g = vec9[leaders[0]].copy()
    for lr in leaders[1:]:
        g = g + vec9[lr]
    report = build_residual_report(layers, g, sched, num_nodes, per_node, eps_abs, eps_rel)
    report["global_sums"] = g
    if sched.adapt:
        u_scale, v_scale = adapt_penalties(report, sched)
        for st in states:
            for n in names:
                if u_scale[n] != 1.0:
                    st.u[n] = st.u[n] * u_scale[n]
                if v_scale[n] != 1.0:
                    st.v[n] = st.v[n] * v_scale[n]
    return report, r_intra_local


# -- phase-1 boundary: proximal SGD update (workloads.py:296-321) ---------------


def prox_sgd(w, z, u, rho1: dict, grads_seq, lr: float, momentum: float):
    """proximal_sgd's parameter updates for a given gradient sequence (one entry
    per mini-batch step): combined = grad + rho1 * (w - z + u), velocity =
    momentum * velocity + combined, w -= lr * velocity (workloads.py:316-320);
    velocity starts at zero (:312); inputs are not modified."""
    w = {n: np.asarray(a, dtype=np.float64).copy() for n, a in w.items()}
    vel = {n: np.zeros_like(a) for n, a in w.items()}
    for grads in grads_seq:
        for n in w:
            combined = grads[n] + rho1[n] * (w[n] - z[n] + u[n])
            vel[n] = momentum * vel[n] + combined
            w[n] -= lr * vel[n]
    return w


# -- the cluster-wide sync step ------------------------------------------------


@dataclass
class Layer:
    name: str
    shape: tuple
    plan: list = field(default_factory=list)   # [(group, keep)] in application order

    @property
    def prunable(self) -> bool:
        return bool(self.plan)


@dataclass
class RankState:
    theta: dict
    u: dict
    z_node: dict
    v: dict
    z: dict
    masks: dict                       # global (union) masks of prunable layers
    frozen: bool = False
    drift_history: list = field(default_factory=list)
    keep_cache: dict = field(default_factory=dict)   # leader: name -> (mask bytes, K_out, K_in)
    derive_calls: int = 0
    hits: int = 0
    sealed: bool = False


def make_layers(specs, constraints) -> list[Layer]:
    """specs: [(name, shape)]; constraints: name -> [(group, keep_count|None, keep_rate|None)]."""
    out = []
    for name, shape in specs:
        plan = []
        for group, kc, kr in constraints.get(name, []):
            g = {FILTER: shape[0], CHANNEL: shape[1]}.get(group, int(np.prod(shape[1:])))
            plan.append((group, resolve_keep(g, kc, kr)))
        out.append(Layer(name, tuple(shape), plan))
    return out


def init_rank_state(layers, theta, u, z_node, v, z) -> RankState:
    f64 = lambda d: {k: np.asarray(a, dtype=np.float64).copy() for k, a in d.items()}
    masks = {ly.name: np.ones(ly.shape, dtype=bool) for ly in layers if ly.prunable}
    return RankState(f64(theta), f64(u), f64(z_node), f64(v), f64(z), masks)


def _keep_sets(st: RankState, name: str, mask: np.ndarray):
    """KeepSetCache.get (shrinkage.py:115-130)."""
    if st.sealed:
        st.hits += 1
        return st.keep_cache[name][1:]
    fp = mask.tobytes()
    ent = st.keep_cache.get(name)
    if ent is not None and ent[0] == fp:
        st.hits += 1
        return ent[1:]
    ko, ki = derive_keep_sets(mask)
    st.derive_calls += 1
    st.keep_cache[name] = (fp, ko, ki)
    return ko, ki


def cluster_sync(layers, states: list[RankState], thetas: list[dict], k: int,
                 num_nodes: int, per_node: int, rho1: dict, rho2: dict,
                 weight_decay: float, t_freeze: int = 10, drift_window: int = 3,
                 sync_period: int = 1, ledger: list | None = None, residuals: bool = False,
                 sched: Schedule | None = None, eps_abs: float = 1e-4, eps_rel: float = 1e-3):
    """One outer iteration k of the sync path on every rank, in place.

    ``thetas[r]`` is rank r's phase-1 output (consensus.py:429). Follows
    consensus.py:436-535 (sums, candidate, projection, leader mask union,
    compaction with the fresh union, bucketed leader average, decompaction,
    inter dual, broadcast, intra dual) and the freeze/seal at :600-606.
    Ledger entries (dicts like transport.py:138-151) are appended to ``ledger``.
    With ``residuals`` (and ``sched`` holding ``rho1`` / ``rho2``) phase 5's residual
    block and penalty adaptation follow the u-update; returns (report, r_intra).
    """
    world = num_nodes * per_node
    names = [ly.name for ly in layers]
    prunable = [ly for ly in layers if ly.prunable]

    def log(group, scope, op, elems, nbytes, members, label, detail=None):
        if ledger is not None and nbytes > 0:
            e = dict(iter=k, group=group, scope=scope, op=op, elements=int(elems),
                     bytes=int(nbytes), members=members, label=label)
            if detail is not None:
                e["detail"] = dict(detail)
            ledger.append(e)

    for r in range(world):
        states[r].theta = {n: np.asarray(thetas[r][n], dtype=np.float64) for n in names}
    zn_prev = [st.z_node for st in states]
    z_prev = [st.z for st in states]

    # phase 2: intra-node SUM of theta+u, serial fold in rank order (transport.py:453-462)
    sums = {}
    for i in range(num_nodes):
        members = range(i * per_node, (i + 1) * per_node)
        acc = {}
        for n in names:
            parts = [states[r].theta[n] + states[r].u[n] for r in members]
            a = parts[0].copy()
            for p in parts[1:]:
                a = a + p
            acc[n] = a
            log(f"intra{i}", "intra", "allreduce_sum", a.size, a.size * ELEMENT_BYTES,
                per_node, f"theta_u/{n}")
        sums[i] = acc

    # phase 3: candidate + projection / frozen mask, every rank (consensus.py:442-454)
    local_masks = {}
    for r in range(world):
        st, node = states[r], r // per_node
        zn, lm = {}, {}
        for ly in layers:
            n = ly.name
            cand = node_candidate(sums[node][n], st.z[n], st.v[n], rho1[n], rho2[n],
                                  weight_decay, num_nodes, per_node)
            if not ly.prunable:
                zn[n] = cand.copy()
            elif st.frozen:
                zn[n] = cand * st.masks[n]
            else:
                zn[n] = project_composite(cand, ly.plan)
                lm[n] = extract_mask(zn[n])
        st.z_node = zn
        local_masks[r] = lm

    if k % sync_period != 0:
        for r in range(world):
            st = states[r]
            st.u = {n: dual_update_intra(st.theta[n], st.z_node[n], st.u[n]) for n in names}
        if residuals:
            return residual_phase(layers, states, zn_prev, z_prev, False, num_nodes, per_node, sched,
                                  eps_abs, eps_rel)
        return None

    # phase 4 (leaders): mask union, compaction, bucketed AVG (consensus.py:463-505)
    leaders = [i * per_node for i in range(num_nodes)]
    frozen = states[0].frozen
    new_masks = {}
    if not frozen:
        for ly in prunable:
            acc = local_masks[leaders[0]][ly.name].copy()
            for r in leaders[1:]:
                acc = np.logical_or(acc, local_masks[r][ly.name])
            new_masks[ly.name] = acc
            log("leaders", "inter", "allreduce_bor", acc.size, acc.size * ELEMENT_BYTES,
                num_nodes, f"mask_sync/{ly.name}")
    payloads = {r: [] for r in leaders}
    keeps = {}
    for ly in layers:
        n = ly.name
        for r in leaders:
            st = states[r]
            c = st.z_node[n] + st.v[n]
            if ly.prunable:
                eff = new_masks.get(n, st.masks[n])
                ko, ki = _keep_sets(st, n, eff)
                keeps[n] = (ko, ki)
                if len(ko) * len(ki):
                    payloads[r].append((n, compress(c, ko, ki).ravel()))
            else:
                payloads[r].append((n, c.ravel()))
    layout = bucket_layout([(n, a.size) for n, a in payloads[leaders[0]]])
    flat = {r: (np.concatenate([a for _, a in payloads[r]]) if payloads[r] else np.empty(0))
            for r in leaders}
    reduced = np.empty(flat[leaders[0]].size)
    start = 0
    for bi, bucket in enumerate(layout):
        size = sum(e for _, _, e in bucket)
        acc = flat[leaders[0]][start:start + size].copy()
        for r in leaders[1:]:
            acc = acc + flat[r][start:start + size]
        reduced[start:start + size] = acc / float(num_nodes)
        log("leaders", "inter", "allreduce_avg", size, size * ELEMENT_BYTES, num_nodes,
            f"z_sync/b{bi}", detail=[(nm, e) for nm, _, e in bucket])
        start += size
    offsets, off = {}, 0
    for n, a in payloads[leaders[0]]:
        offsets[n] = (off, a.size)
        off += a.size
    z_new = {}
    for ly in layers:
        n = ly.name
        if ly.prunable:
            ko, ki = keeps[n]
            if n in offsets:
                o, e = offsets[n]
                z_new[n] = decompress(reduced[o:o + e], ko, ki, ly.shape)
            else:
                z_new[n] = np.zeros(ly.shape)
        else:
            o, e = offsets[n]
            z_new[n] = reduced[o:o + e].reshape(ly.shape).copy()
    for i, lr in enumerate(leaders):
        st = states[lr]
        v_new = {n: st.v[n] + (st.z_node[n] - z_new[n]) for n in names}
        for r in range(lr, lr + per_node):      # intra broadcast of z, v, masks
            states[r].v = {n: a.copy() for n, a in v_new.items()}
            states[r].z = {n: a.copy() for n, a in z_new.items()}
        for n in names:
            log(f"intra{i}", "intra", "broadcast", z_new[n].size,
                z_new[n].size * ELEMENT_BYTES * (per_node - 1), per_node, f"z_bcast/{n}")
        for n in names:
            log(f"intra{i}", "intra", "broadcast", z_new[n].size,
                z_new[n].size * ELEMENT_BYTES * (per_node - 1), per_node, f"v_bcast/{n}")
        if not frozen:
            for ly in prunable:
                log(f"intra{i}", "intra", "broadcast", new_masks[ly.name].size,
                    new_masks[ly.name].size * ELEMENT_BYTES * (per_node - 1), per_node,
                    f"m_bcast/{ly.name}")
    for r in range(world):
        st = states[r]
        if not frozen and prunable:
            drift = {n: mask_drift(st.masks[n], m) for n, m in new_masks.items()}
            st.masks = {n: m.copy() for n, m in new_masks.items()}
            st.drift_history.append(max(drift.values()))
        # phase 5: intra dual update (consensus.py:535)
        st.u = {n: dual_update_intra(st.theta[n], st.z_node[n], st.u[n]) for n in names}
    out = None
    if residuals:   # residual block + adaptation (consensus.py:537-598), before the freeze check
        out = residual_phase(layers, states, zn_prev, z_prev, True, num_nodes, per_node, sched,
                             eps_abs, eps_rel)
    for r in range(world):
        st = states[r]
        # freeze + seal (consensus.py:600-606)
        if not st.frozen and prunable and freeze_check(k, t_freeze, st.drift_history, drift_window):
            st.frozen = True
            if r % per_node == 0:
                for ly in prunable:
                    _keep_sets(st, ly.name, st.masks[ly.name])
                st.sealed = True
    return out


# -- comparison baselines (baselines.py) ---------------------------


@dataclass
class FlatState:
    """flat_consensus_program's per-run state (baselines.py:169-181): the global z,
    every rank's u, the masks of the prunable layers, frozen, drift history."""
    z: dict
    u: list
    masks: dict
    frozen: bool = False
    drift_history: list = field(default_factory=list)


def init_flat_state(layers, params0, world) -> FlatState:
    p = {n: np.asarray(a, dtype=np.float64).copy() for n, a in params0.items()}
    return FlatState(z=p, u=[{n: np.zeros_like(a) for n, a in p.items()} for _ in range(world)],
                     masks={ly.name: np.ones(ly.shape, dtype=bool) for ly in layers if ly.prunable})


def flat_consensus_step(layers, st: FlatState, thetas: list[dict], k: int, sched: Schedule,
                        weight_decay: float, t_freeze: int = 10, drift_window: int = 3,
                        eps_abs: float = 1e-4, eps_rel: float = 1e-3, ledger: list | None = None):
    """One iteration k of flat_consensus_program (baselines.py:184-287) after phase 1,
    in place on ``st``: dense all-rank SUM of theta + u per layer (rank-order fold),
    cand = rho1 * total / (wd + W rho1), projection of the global tensor (frozen:
    cand * mask), u-update, the 3-slot residual SUM, the flat report, rho1 adaptation
    with the u rescale, freeze check. Returns (report, r_intra per rank, drift_now)."""
    world = len(thetas)
    z_prev, z, drift_now = st.z, {}, {}

    def log(op, elems, label):
        if ledger is not None:
            ledger.append({"iter": k, "group": "global", "scope": "global", "op": op,
                           "elements": int(elems), "bytes": ELEMENT_BYTES * int(elems), "members": world,
                           "label": label})

    for ly in layers:
        n = ly.name
        total = thetas[0][n] + st.u[0][n]                                 # transport.py:453-462
        for r in range(1, world):
            total = total + (thetas[r][n] + st.u[r][n])
        log("allreduce_sum", total.size, f"z_sync/{n}")
        gamma = weight_decay + world * sched.rho1[n]                      # baselines.py:195
        cand = (sched.rho1[n] * total) / gamma
        if ly.prunable and st.frozen:
            z[n] = cand * st.masks[n]
        elif ly.prunable:
            z[n] = project_composite(cand, ly.plan)
            new = extract_mask(z[n])
            drift_now[n] = mask_drift(st.masks[n], new)
            st.masks[n] = new
        else:
            z[n] = cand
    if drift_now:
        st.drift_history.append(max(drift_now.values()))
    st.u = [{n: st.u[r][n] + (thetas[r][n] - z[n]) for n in z} for r in range(world)]   # :210
    names = [ly.name for ly in layers]
    vecs, r_local = [], []
    for r in range(world):
        v3 = np.empty(len(names) * 3)
        rl = {}
        for li, n in enumerate(names):
            d = thetas[r][n] - z[n]
            rl[n] = math.sqrt(sq(d))
            v3[li * 3:li * 3 + 3] = (sq(d), float(np.sum(thetas[r][n] ** 2)), float(np.sum(st.u[r][n] ** 2)))
        vecs.append(v3)
        r_local.append(rl)
    sums = vecs[0].copy()
    for r in range(1, world):
        sums = sums + vecs[r]
    log("allreduce_sum", sums.size, "res_flat")
    per_layer = {}
    r_pri_sq = r_dual_sq = eps_pri_sq = eps_dual_sq = 0.0
    for li, ly in enumerate(layers):                                      # :230-254
        n = ly.name
        rho1 = sched.rho1[n]
        nel = int(np.prod(ly.shape))
        r = math.sqrt(sums[li * 3])
        s = rho1 * math.sqrt(world * float(np.sum((z[n] - z_prev[n]) ** 2)))
        eps_pri = math.sqrt(nel * world) * eps_abs + eps_rel * max(
            math.sqrt(sums[li * 3 + 1]), math.sqrt(world * float(np.sum(z[n] ** 2))))
        eps_dual = math.sqrt(nel * world) * eps_abs + eps_rel * rho1 * math.sqrt(sums[li * 3 + 2])
        per_layer[n] = (r, s, 0.0, 0.0, eps_pri, eps_dual, 0.0, 0.0)
        r_pri_sq += r * r
        r_dual_sq += s * s
        eps_pri_sq += eps_pri * eps_pri
        eps_dual_sq += eps_dual * eps_dual
    r_pri, r_dual = math.sqrt(r_pri_sq), math.sqrt(r_dual_sq)
    eps_pri, eps_dual = math.sqrt(eps_pri_sq), math.sqrt(eps_dual_sq)
    report = {"layers": per_layer, "r_pri": r_pri, "r_dual": r_dual, "eps_pri": eps_pri,
              "eps_dual": eps_dual, "converged": r_pri <= eps_pri and r_dual <= eps_dual}
    if sched.adapt:                                                       # :271-282 (rho1 only)
        for n in names:
            lr_ = per_layer[n]
            old = sched.rho1[n]
            if lr_[0] > sched.mu * lr_[1]:
                sched.rho1[n] = min(old * sched.tau_inc, sched.rho1_max)
            elif lr_[1] > sched.mu * lr_[0]:
                sched.rho1[n] = old / sched.tau_dec
            scale = old / sched.rho1[n] if sched.rho1[n] != old else 1.0
            if scale != 1.0:
                for r in range(world):
                    st.u[r][n] = st.u[r][n] * scale
    st.z = z
    if not st.frozen and any(ly.prunable for ly in layers):               # :284-286
        if freeze_check(k, t_freeze, st.drift_history, drift_window):
            st.frozen = True
    return report, r_local, drift_now


def dense_sync_step(params: dict, velocity: dict, grads: list[dict], lr: float, momentum: float,
                    weight_decay: float, ledger: list | None = None, step: int = 0):
    """One step of dense_sync_program (baselines.py:86-96), in place on params / velocity:
    per layer g_r = grad_r + wd * params, AVG over ranks (rank-order fold, / W),
    velocity = momentum * velocity + avg, params -= lr * velocity."""
    world = len(grads)
    avg = {}
    for n in params:
        acc = grads[0][n] + weight_decay * params[n]
        for r in range(1, world):
            acc = acc + (grads[r][n] + weight_decay * params[n])
        avg[n] = acc / float(world)
        if ledger is not None:
            ledger.append({"iter": step, "group": "global", "scope": "global", "op": "allreduce_avg",
                           "elements": int(acc.size), "bytes": ELEMENT_BYTES * int(acc.size),
                           "members": world, "label": f"grad/{n}"})
    for n in params:
        velocity[n] = momentum * velocity[n] + avg[n]
        params[n] -= lr * velocity[n]


def topk_keep_count(rate: float, size: int) -> int:
    return max(1, math.ceil(rate * size))                                 # baselines.py:132


def topk_select(flat: np.ndarray, k: int) -> np.ndarray:
    """Indices of the k largest |values|, ties toward lower indices, ascending
    (baselines.py:71-74: stable argsort of -|x|)."""
    order = np.argsort(-np.abs(flat), kind="stable")
    return np.sort(order[:k])


def topk_step(params: dict, velocity: dict, residual: list, grads: list[dict], rate: float, lr: float,
              momentum: float, weight_decay: float, ledger: list | None = None, step: int = 0):
    """One step of topk_program (baselines.py:124-146) for every rank, in place on
    params / velocity (shared: bit-identical on every rank) and residual[r]: acc =
    residual + grad + wd * params; rank r ships the top-k (value, index) pairs; the
    all-gathered pairs are scatter-added in rank order and / W; the untransmitted
    entries stay in the residual. Returns the selected indices per rank and layer."""
    world = len(grads)
    avg, sels = {}, [{} for _ in range(world)]
    for n in params:
        payloads = []
        for r in range(world):
            g = grads[r][n] + weight_decay * params[n]
            acc = residual[r][n] + g
            flat = acc.ravel()
            k = topk_keep_count(rate, flat.size)
            sel = topk_select(flat, k)
            sels[r][n] = sel
            payloads.append((flat[sel], sel, k))
            kept = np.zeros_like(flat)
            kept[sel] = flat[sel]
            residual[r][n] = (flat - kept).reshape(acc.shape)
        if ledger is not None:
            k = payloads[0][2]
            ledger.append({"iter": step, "group": "global", "scope": "global", "op": "allgather",
                           "elements": 2 * k, "bytes": ELEMENT_BYTES * 2 * k, "members": world,
                           "label": f"topk/{n}"})
        dense = np.zeros(params[n].size)
        for values, indices, _ in payloads:                               # :137-139
            dense[indices] += values
        avg[n] = (dense / float(world)).reshape(params[n].shape)
    for n in params:
        velocity[n] = momentum * velocity[n] + avg[n]
        params[n] -= lr * velocity[n]
    return sels
