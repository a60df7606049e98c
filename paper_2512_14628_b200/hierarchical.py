"""The reference's run entry points on the B200 engine.

``hierarchical_program`` / ``run_hierarchical`` keep the signatures of
/root/reference/pkg/src/admmprune/consensus.py:386-637, so a caller of the
reference switches by changing the import. Each rank program drives one
:class:`~.sync.HSADMMSync` (phases 2-5 of iteration k are its ``program(k)``:
the libhsx kernels + the collectives of the cluster it runs under):

* ``cluster``: :class:`~.transport.Cluster` — a ``LocalCluster`` (every rank in
  this process, one GPU, the reference's deterministic scheduler) or a
  ``DistCluster`` (one rank per process under torchrun, NCCL / NVLink peers);
* ``workload``: anything with ``layers`` (LayerSpecs, the reference's or
  ours), ``shards[rank]`` and ``init_params(rng)`` — the reference's workloads
  work unchanged;
* phase 1 (local proximal SGD, out of the sync path's scope) is the module
  attribute :data:`proximal_sgd`, called like the reference's
  (workloads.py:296-322). By default it runs the workload's
  ``loss_and_grad`` on the host for each mini-batch and applies the combined
  update ``grad + rho1 (theta - z_node + u)`` with momentum in the fused
  ``k_prox_sgd`` kernel (the last mini-batch also writes theta + u into the
  intra-sum send buffer). Replacing the attribute (as the reference's own
  fixtures replace ``consensus.proximal_sgd``) hands the hook numpy copies of
  theta / z_node / u and loads what it returns.

The returned :class:`RankResult` / :class:`ConsensusState` / trace rows carry
the reference's fields (consensus.py:114-139, :567-598), with the state as
float64 numpy copies of the engine's fp32 arenas. Digests (``state_sha``,
``mask_sha``) hash those arrays, so they identify this run's state but do not
equal the reference's fp64 digests.
"""

from __future__ import annotations

import dataclasses
import hashlib
import math
from dataclasses import dataclass

import numpy as np
import torch

from .consensus import ConsensusSettings, LayerResiduals, PenaltySchedule, REPORT_SLOTS, ResidualReport
from .errors import ConfigError
from .layers import LayerKind, LayerSpec
from .sparsity import ConstraintKind, SparsityConstraint
from .sync import HSADMMSync

_INIT_STREAM = 211    # reference workloads.py:21-22
_BATCH_STREAM = 307


@dataclass(frozen=True)
class SolverConfig:
    """Inner-solver settings (reference workloads.py:37-51)."""

    lr: float = 1e-3
    epochs: int = 5
    batch_size: int = 128
    momentum: float = 0.9
    weight_decay: float = 1e-4

    def __post_init__(self):
        if self.lr <= 0:
            raise ConfigError(f"learning rate must be positive, got {self.lr}")
        if self.epochs < 1:
            raise ConfigError(f"epochs must be at least 1, got {self.epochs}")
        if self.batch_size < 1:
            raise ConfigError(f"batch size must be at least 1, got {self.batch_size}")


@dataclass
class ConsensusState:
    """Per-rank fragment of the optimization state (consensus.py:114-127)."""

    rank: int
    iteration: int
    frozen: bool
    theta: dict
    u: dict
    z_node: dict
    v: dict
    z: dict
    masks: dict
    schedule: PenaltySchedule


@dataclass
class RankResult:
    """consensus.py:130-137."""

    rank: int
    state: ConsensusState
    trace: list
    converged_at: int | None
    cache_derive: int
    cache_hits: int


def batch_rng(seed: int, rank: int, outer_iteration: int) -> np.random.Generator:
    """Mini-batch order stream of a rank's phase 1 (workloads.py:281-282)."""
    return np.random.default_rng([seed, _BATCH_STREAM, rank, outer_iteration])


def init_rng(seed: int) -> np.random.Generator:
    """Initial-parameter stream (workloads.py:285-286)."""
    return np.random.default_rng([seed, _INIT_STREAM])


def _minibatches(rows: int, batch_size: int, rng: np.random.Generator):
    order = rng.permutation(rows)   # workloads.py:289-293
    return [order[s:s + batch_size] for s in range(0, rows, batch_size)]


def _fused_proximal_sgd(workload, shard, theta, z_node, u, rho1, solver, rng, *, engine=None):
    """Phase 1 on the engine (workloads.py:296-322): per mini-batch the workload's
    gradient on the host (float64, as the reference computes it), then the fused
    combined-gradient / momentum / lr update on the device arenas."""
    eng = engine
    batch = min(solver.batch_size, shard.rows)
    steps = [idx for _ in range(solver.epochs) for idx in _minibatches(shard.rows, batch, rng)]
    grad = eng.plan.empty_arena(eng.device)
    for s, idx in enumerate(steps):
        w = {n: t.detach().double().cpu().numpy() for n, t in eng.views("theta").items()}
        _, grads = workload.loss_and_grad(w, shard.features[idx], shard.targets[idx])
        eng.plan.load_arena(grad, grads)
        eng.prox_sgd_step(grad, solver.lr, solver.momentum, first=s == 0, last=s == len(steps) - 1)
    return None


#: Phase 1 hook, called as the reference calls its ``proximal_sgd``
#: (consensus.py:429). Replace it to supply theta some other way.
proximal_sgd = _fused_proximal_sgd


def adapt_penalties(report: ResidualReport, sched: PenaltySchedule):
    """Residual balancing per layer and level (consensus.py:189-219), host side.

    The engine applies the same rule on the device each iteration
    (``k_report``); this is the per-object API. Returns (new schedule, u scales,
    v scales)."""
    rho1, rho2 = dict(sched.rho1), dict(sched.rho2)
    u_scale, v_scale = {}, {}
    for name in rho1:
        lr = report.layers[name]
        old = rho1[name]
        if lr.r_intra > sched.mu * lr.s_intra:
            rho1[name] = min(old * sched.tau_inc, sched.rho1_max)
        elif lr.s_intra > sched.mu * lr.r_intra:
            rho1[name] = old / sched.tau_dec
        u_scale[name] = old / rho1[name] if rho1[name] != old else 1.0
        old2 = rho2[name]
        if lr.r_inter > sched.mu * lr.s_inter:
            rho2[name] = min(old2 * sched.tau_inc, sched.rho2_max)
        elif lr.s_inter > sched.mu * lr.r_inter:
            rho2[name] = old2 / sched.tau_dec
        v_scale[name] = old2 / rho2[name] if rho2[name] != old2 else 1.0
    return dataclasses.replace(sched, rho1=rho1, rho2=rho2), u_scale, v_scale


def pack_report(report: ResidualReport, layer_names) -> np.ndarray:
    """The report broadcast's vector layout (consensus.py:291-300): 8 slots per
    layer, then r_pri, r_dual, eps_pri, eps_dual, converged."""
    vec = np.empty(len(layer_names) * REPORT_SLOTS + 5, dtype=np.float64)
    for li, name in enumerate(layer_names):
        lr = report.layers[name]
        vec[li * REPORT_SLOTS:(li + 1) * REPORT_SLOTS] = (
            lr.r_intra, lr.s_intra, lr.r_inter, lr.s_inter,
            lr.eps_pri_intra, lr.eps_dual_intra, lr.eps_pri_inter, lr.eps_dual_inter)
    vec[-5:] = (report.r_pri, report.r_dual, report.eps_pri, report.eps_dual, float(report.converged))
    return vec


# -- adapters for the reference's own objects ------------------------------------------


def _as_layer(ls) -> LayerSpec:
    if isinstance(ls, LayerSpec):
        return ls
    return LayerSpec(ls.name, LayerKind(ls.kind.value), tuple(int(d) for d in ls.shape), bool(ls.prunable))


def _as_constraint(c) -> SparsityConstraint:
    if isinstance(c, SparsityConstraint):
        return c
    return SparsityConstraint(ConstraintKind(c.kind.value), keep_count=c.keep_count, keep_rate=c.keep_rate)


def _as(cls, obj):
    if isinstance(obj, cls):
        return obj
    return cls(**{f.name: getattr(obj, f.name) for f in dataclasses.fields(cls) if hasattr(obj, f.name)})


def _digest(arrays: dict, names) -> str:
    h = hashlib.sha256()
    for n in names:
        h.update(np.ascontiguousarray(arrays[n]).tobytes())
    return h.hexdigest()


def _host(eng: HSADMMSync, key: str) -> dict:
    return {n: t.detach().cpu().numpy().astype(np.float64) for n, t in eng.views(key).items()}


def _layer_sq_norms(a: torch.Tensor, b: torch.Tensor | None, eng: HSADMMSync) -> list[float]:
    """Per-layer sum of squares of (a - b) (or a), fp64 on the device."""
    d = a.double() if b is None else a.double() - b.double()
    d = d * d
    return [float(x) for x in torch.stack([d[o:o + ls.elements].sum()
                                           for o, ls in zip(eng.plan.offsets, eng.layers)]).cpu()]


def hierarchical_program(rank, cluster, workload, constraints, schedule, solver, settings,
                         capture_states: bool = False, transport: str = "auto"):
    """Generator program for one rank of the hierarchical consensus run
    (consensus.py:386-619) on the B200 sync engine."""
    layers = [_as_layer(ls) for ls in workload.layers]
    names = [ls.name for ls in layers]
    cons = {n: [_as_constraint(c) for c in cs] for n, cs in constraints.items() if cs}
    sched0 = _as(PenaltySchedule, schedule)
    sett = _as(ConsensusSettings, settings)
    eng = HSADMMSync(rank, cluster, layers, cons, sched0, sett, transport=transport, residuals=True)
    shard = workload.shards[rank]
    eng.init_from(workload.init_params(init_rng(sett.seed)))
    n_prunable = len(eng.prunable)
    trace: list[dict] = []
    converged_at = None
    for k in range(1, sett.iterations + 1):
        # phase 1 (consensus.py:428-434)
        sched_k = eng.current_schedule()
        rng = batch_rng(sett.seed, rank, k)
        hook = proximal_sgd
        if hook is _fused_proximal_sgd:
            hook(workload, shard, None, None, None, sched_k.rho1, solver, rng, engine=eng)
        else:
            out = hook(workload, shard, _host(eng, "theta"), _host(eng, "z_node"), _host(eng, "u"),
                       dict(sched_k.rho1), solver, rng)
            eng.load(theta=out)
        if not bool(torch.isfinite(eng.theta).all()):
            bad = next(n for n, t in eng.views("theta").items() if not bool(torch.isfinite(t).all()))
            raise FloatingPointError(f"rank {rank}, iteration {k}: non-finite values in theta[{bad}]")
        frozen = eng.frozen
        sync_iter = k % sett.sync_period == 0
        # phases 2-5 (consensus.py:436-606): the engine's step
        yield from eng.program(k)
        eng.settle()
        report = eng.last_report()
        froze_now = eng.frozen and not frozen
        masks = {n: m.cpu().numpy() for n, m in eng.mask_dict().items()}
        theta_h, z_h = _host(eng, "theta"), _host(eng, "z")
        hits = eng.cache_hits - (n_prunable if froze_now and eng.is_leader else 0)
        row = {
            "k": k,
            "frozen": frozen,
            "r_intra": dict(zip(names, map(math.sqrt, _layer_sq_norms(eng.theta, eng.z_node, eng)))),
            "state_sha": _digest(theta_h, names) + _digest(z_h, names)[:16],
            "cache_derive": eng.cache_derive,
            "cache_hits": hits,
            "mask_sha": {n: hashlib.sha256(m.tobytes()).hexdigest() for n, m in masks.items()},
        }
        if eng.is_leader:
            row["r_inter"] = dict(zip(names, map(math.sqrt, _layer_sq_norms(eng.z_node, eng.z, eng))))
        if rank == 0:
            row["report"] = report
            row["rho1"] = dict(sched_k.rho1)
            row["rho2"] = dict(sched_k.rho2)
            row["drift"] = dict(eng.drift_now) if (sync_iter and not frozen and n_prunable) else {}
            row["mask_popcount"] = {n: int(m.sum()) for n, m in masks.items()}
        if capture_states:
            row["theta_copy"] = theta_h
            row["z_node_copy"] = _host(eng, "z_node")
            sc = eng.scales.cpu().numpy()
            row["u_scale"] = ({n: float(sc[i]) for i, n in enumerate(names)} if sched0.adapt
                              else {n: 1.0 for n in names})
        trace.append(row)
        if sett.stop_on_convergence and report.converged:
            converged_at = k
            break
    eng.check_barriers()
    state = ConsensusState(
        rank=rank, iteration=trace[-1]["k"] if trace else 0, frozen=eng.frozen,
        theta=_host(eng, "theta"), u=_host(eng, "u"), z_node=_host(eng, "z_node"), v=_host(eng, "v"),
        z=_host(eng, "z"), masks={n: m.cpu().numpy() for n, m in eng.mask_dict().items()},
        schedule=eng.current_schedule())
    return RankResult(rank=rank, state=state, trace=trace, converged_at=converged_at,
                      cache_derive=eng.cache_derive, cache_hits=eng.cache_hits)


def run_hierarchical(cluster, workload, constraints, schedule, solver, settings,
                     capture_states: bool = False, transport: str = "auto") -> dict:
    """consensus.py:622-637: one program per rank, driven by ``cluster.run``. Under
    a DistCluster this process runs (and returns) its own rank only."""
    programs = {rank: hierarchical_program(rank, cluster, workload, constraints, schedule, solver, settings,
                                           capture_states, transport)
                for rank in range(cluster.topology.world_size)}
    return cluster.run(programs)
