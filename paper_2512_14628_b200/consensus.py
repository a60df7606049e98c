"""H-SADMM update rules, schedules and settings (per-tensor API).

Same public surface as the reference's ``admmprune.consensus`` for the sync
path (/root/reference/pkg/src/admmprune/consensus.py): ``PenaltySchedule``
(:42-69), ``ConsensusSettings`` (:94-110), ``node_candidate`` (:142-160),
``update_node_consensus`` (:163-182), ``dual_update_intra`` (:185-186),
``freeze_check`` (:222-228). The fused, arena-wide SPMD step that replaces
phases 2-5 of ``hierarchical_program`` is :class:`~.sync.HSADMMSync`.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import torch

from .errors import ConfigError, ProtocolError, ShapeError
from .layers import LayerKind, LayerSpec
from .plan import Plan
from .sparsity import as_cuda_f32, extract_mask, project_composite


@dataclass(frozen=True)
class PenaltySchedule:
    """Layer-wise penalties for the two consensus levels."""

    rho1: dict
    rho2: dict
    rho1_max: float = 10.0
    rho2_max: float = 10.0
    mu: float = 10.0
    tau_inc: float = 2.0
    tau_dec: float = 2.0
    adapt: bool = True

    def __post_init__(self):
        for name, value in self.rho1.items():
            if not (0.0 < value <= self.rho1_max):
                raise ConfigError(f"rho1[{name}]={value} outside (0, {self.rho1_max}]")
        for name, value in self.rho2.items():
            if not (0.0 <= value <= self.rho2_max):
                raise ConfigError(f"rho2[{name}]={value} outside [0, {self.rho2_max}]")

    @classmethod
    def uniform(cls, layer_names, rho1: float, rho2: float, **kwargs) -> "PenaltySchedule":
        return cls(rho1={n: float(rho1) for n in layer_names},
                   rho2={n: float(rho2) for n in layer_names}, **kwargs)


@dataclass(frozen=True)
class LayerResiduals:
    """Per-layer residuals and tolerances (consensus.py:72-81)."""

    r_intra: float
    s_intra: float
    r_inter: float
    s_inter: float
    eps_pri_intra: float
    eps_dual_intra: float
    eps_pri_inter: float
    eps_dual_inter: float


@dataclass(frozen=True)
class ResidualReport:
    """Phase-5 report (consensus.py:84-91): per-layer residuals + global totals."""

    layers: dict
    r_pri: float
    r_dual: float
    eps_pri: float
    eps_dual: float
    converged: bool


REPORT_SLOTS = 8  # consensus.py:236


def unpack_report(vec, layer_names) -> ResidualReport:
    """Inverse of the reference's pack_report layout (consensus.py:291-314)."""
    v = [float(x) for x in vec]
    layers = {n: LayerResiduals(*v[i * REPORT_SLOTS:(i + 1) * REPORT_SLOTS]) for i, n in enumerate(layer_names)}
    t = v[len(layer_names) * REPORT_SLOTS:]
    return ResidualReport(layers, t[0], t[1], t[2], t[3], bool(t[4]))


@dataclass(frozen=True)
class ConsensusSettings:
    iterations: int = 1
    t_freeze: int = 10
    drift_window: int = 3
    sync_period: int = 1
    eps_abs: float = 1e-4
    eps_rel: float = 1e-3
    stop_on_convergence: bool = True
    weight_decay: float = 1e-4
    seed: int = 0

    def __post_init__(self):
        if self.iterations < 1:
            raise ConfigError("iterations must be at least 1")
        if self.sync_period < 1:
            raise ConfigError("sync_period must be at least 1")


@lru_cache(maxsize=64)
def _dense_plan(n: int, rho1: float, rho2: float, wd: float, m: int, p: int) -> Plan:
    plan = Plan([LayerSpec("t", LayerKind.FULLY_CONNECTED, (1, n))], {}, {"t": rho1}, {"t": rho2})
    plan.set_penalties(None, None, wd, m, p)
    return plan


def node_candidate(sum_theta_u, z_global, v, rho1: float, rho2: float, weight_decay: float,
                   num_nodes: int, accels_per_node: int) -> torch.Tensor:
    """``(rho1*S + rho2*(z - v)) / gamma`` with ``gamma = wd/M + P*rho1 + rho2`` (fp64 math, fp32 out)."""
    gamma = weight_decay / num_nodes + accels_per_node * rho1 + rho2
    if gamma <= 0.0:
        raise ConfigError(f"non-positive candidate normalizer gamma={gamma}")
    s, z, v = (as_cuda_f32(x) for x in (sum_theta_u, z_global, v))
    if not (s.shape == z.shape == v.shape):
        raise ShapeError(f"shape mismatch: {tuple(s.shape)}, {tuple(z.shape)}, {tuple(v.shape)}")
    plan = _dense_plan(s.numel(), float(rho1), float(rho2), float(weight_decay), int(num_nodes),
                       int(accels_per_node))
    out = torch.empty_like(s)
    plan.candidate(s, None, None, z, v, out)
    return out


def update_node_consensus(candidate, constraints, frozen: bool, global_mask):
    """Dynamic: project + local mask; frozen: cand * global mask; unconstrained: copy."""
    cand = as_cuda_f32(candidate)
    if not constraints:
        return cand.clone(), (None if frozen else torch.ones(cand.shape, dtype=torch.bool, device=cand.device))
    if frozen:
        if global_mask is None:
            raise ProtocolError("frozen update requires a stored global mask")
        m = torch.as_tensor(global_mask).to(cand.device, torch.bool)
        if tuple(m.shape) != tuple(cand.shape):
            raise ShapeError("global mask shape does not match the candidate")
        plan = _masked_plan(tuple(cand.shape))
        bits = torch.zeros(max(plan.mask_words, 1), dtype=torch.int32, device=cand.device)
        from . import _lib
        from .plan import current_stream

        _lib.call("hsx_pack_bits", m.contiguous().data_ptr(), m.numel(), bits.data_ptr(), current_stream())
        out = torch.empty_like(cand)
        plan.candidate(cand, None, None, None, None, out, frozen_mask=bits)
        return out, None
    z = project_composite(cand, constraints)
    return z, extract_mask(z)


@lru_cache(maxsize=64)
def _masked_plan(shape: tuple[int, ...]) -> Plan:
    from .layers import GroupBy

    if len(shape) != 4:
        shape4 = (1, int(torch.tensor(shape).prod()), 1, 1)
    else:
        shape4 = shape
    plan = Plan([LayerSpec("t", LayerKind.CONV, shape4, prunable=True)], {"t": [(GroupBy.CHANNEL, shape4[1])]})
    plan.set_penalties(None, None, 0.0, 1, 1, identity=True)
    return plan


def dual_update_intra(theta, z_node, u) -> torch.Tensor:
    """``u + (theta - z_node)`` (fp64 math, fp32 out); inputs untouched."""
    th, zn, uu = (as_cuda_f32(x) for x in (theta, z_node, u))
    if not (th.shape == zn.shape == uu.shape):
        raise ShapeError("shape mismatch in dual_update_intra")
    out = uu.clone()
    plan = _dense_plan(out.numel(), 1.0, 0.0, 0.0, 1, 1)
    plan.dual_intra(th, out, zn)
    return out


def freeze_check(k: int, t_freeze: int, drift_history: list[float], window: int = 3) -> bool:
    """Freeze at the fixed iteration or after ``window`` zero-drift syncs."""
    if k >= t_freeze:
        return True
    if window > 0 and len(drift_history) >= window:
        return all(d == 0.0 for d in drift_history[-window:])
    return False
