"""Structured-sparsity constraints, projections and masks on the GPU.

Same public surface as the reference's ``admmprune.sparsity``
(/root/reference/pkg/src/admmprune/sparsity.py): ``ConstraintKind`` (:20-23),
``SparsityConstraint`` with ``resolve`` (:33-62), ``project`` (:71-94),
``project_composite`` (:97-110), ``extract_mask`` (:113-115) and
``mask_drift`` (:118-122). Tensors are CUDA ``torch`` tensors (float32 in,
float32 out; group norms are accumulated in float64 from the exact fp32
inputs); every computation runs in libhsx (K1 candidate in identity mode ->
K2 top-k -> K3 projection). Inputs are never mutated.
"""

from __future__ import annotations

import enum
import math
import warnings
from dataclasses import dataclass
from functools import lru_cache

import torch

from . import _lib
from .errors import ShapeError
from .layers import GroupBy, LayerKind, LayerSpec, group_count
from .plan import Plan, current_stream


class ConstraintKind(enum.Enum):
    FILTER_KEEP = "filter_keep"
    CHANNEL_KEEP = "channel_keep"
    SHAPE_KEEP = "shape_keep"


GROUP_FOR_KIND = {
    ConstraintKind.FILTER_KEEP: GroupBy.FILTER,
    ConstraintKind.CHANNEL_KEEP: GroupBy.CHANNEL,
    ConstraintKind.SHAPE_KEEP: GroupBy.SHAPE_POSITION,
}


@dataclass(frozen=True)
class SparsityConstraint:
    """Keep a bounded number of groups along one dimension (exactly one of count / rate)."""

    kind: ConstraintKind
    keep_count: int | None = None
    keep_rate: float | None = None

    def __post_init__(self):
        if (self.keep_count is None) == (self.keep_rate is None):
            raise ShapeError("specify exactly one of keep_count or keep_rate")
        if self.keep_count is not None and self.keep_count < 1:
            raise ShapeError(f"keep_count must be positive, got {self.keep_count}")
        if self.keep_rate is not None and not (0.0 < self.keep_rate <= 1.0):
            raise ShapeError(f"keep_rate must lie in (0, 1], got {self.keep_rate}")

    def resolve(self, group_count: int) -> int:
        """k = keep_count, or ceil(keep_rate * G) evaluated as a Python float (sparsity.py:53-62)."""
        k = int(self.keep_count) if self.keep_count is not None else int(math.ceil(self.keep_rate * group_count))
        if k > group_count:
            raise ShapeError(f"{self.kind.value}: keep_count {k} exceeds group count {group_count}")
        return k


def resolve_plan(shape: tuple[int, ...], constraints) -> list[tuple[GroupBy, int]]:
    """[(group, keep)] for a conv shape; ShapeError on duplicate kinds (sparsity.py:104-106)."""
    kinds = [c.kind for c in constraints]
    if len(set(kinds)) != len(kinds):
        raise ShapeError(f"duplicate constraint kinds: {[k.value for k in kinds]}")
    return [(GROUP_FOR_KIND[c.kind], c.resolve(group_count(shape, GROUP_FOR_KIND[c.kind])))
            for c in constraints]


def as_cuda_f32(t, name="tensor") -> torch.Tensor:
    """CUDA float32 contiguous tensor (copies numpy / float64 / CPU inputs)."""
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(t)
    if not torch.cuda.is_available():
        raise RuntimeError("libhsx needs a CUDA device (no CPU fallback)")
    if t.dtype == torch.float64:
        # the B200 path computes in fp32 (BASELINE north_star); the reference API is fp64
        warnings.warn(f"{name}: float64 input is rounded to float32 (libhsx computes the sync "
                      "step on fp32 state)", RuntimeWarning, stacklevel=3)
    if t.device.type != "cuda" or t.dtype != torch.float32 or not t.is_contiguous() or t.data_ptr() % 16:
        t = t.to(device="cuda", dtype=torch.float32).contiguous().clone()
    return t


def _tensor_plan(shape: tuple[int, ...], plan: tuple) -> Plan:
    """Plan of a one-tensor call; its device scratch is per (device, stream), so
    calls on another GPU or on concurrent streams never share in-flight scratch."""
    return _tensor_plan_on(shape, plan, torch.cuda.current_device(), current_stream())


@lru_cache(maxsize=64)
def _tensor_plan_on(shape: tuple[int, ...], plan: tuple, device: int, stream: int) -> Plan:
    ls = LayerSpec("t", LayerKind.CONV, shape, prunable=bool(plan))
    p = Plan([ls], {"t": list(plan)})
    p.set_penalties(None, None, 0.0, 1, 1, identity=True)
    return p


def _run_projection(t: torch.Tensor, plan_groups: list[tuple[GroupBy, int]]):
    """(projected tensor, packed mask words, Plan) — candidate(identity) -> select -> project."""
    p = _tensor_plan(tuple(t.shape), tuple(plan_groups))
    out = torch.empty_like(t)
    mask = torch.empty(max(p.mask_words, 1), dtype=torch.int32, device=t.device)
    p.candidate(t, None, None, None, None, out)
    p.project_all(t, None, None, None, None, out, mask)
    return out, mask, p


def group_norms_gpu(t, group: GroupBy) -> torch.Tensor:
    """fp64 group Frobenius norms of a rank-4 tensor (reference tensors.py:75-93)."""
    t = as_cuda_f32(t)
    if t.dim() != 4:
        raise ShapeError(f"group norms need a rank-4 tensor, got rank {t.dim()}")
    g = group_count(tuple(t.shape), group)
    _, _, p = _run_projection(t, [(group, g)])
    norms, _ = p.group_norms(0, t.device)
    return norms[:g].clone()


def frobenius_norm(t) -> float:
    """sqrt(sum t^2) in fp64 (reference tensors.py:71-72): the tensor (zero-padded
    to rows of 4096) as filters of a (rows, 4096, 1, 1) weight, fp64 filter norms
    accumulated in libhsx, then the fp64 root of their sum of squares."""
    t = as_cuda_f32(t)
    n = t.numel()
    if n == 0:
        return 0.0
    cols = 4096
    rows = (n + cols - 1) // cols
    padded = torch.zeros(rows * cols, dtype=torch.float32, device=t.device)
    padded[:n] = t.reshape(-1)
    norms = group_norms_gpu(padded.view(rows, cols, 1, 1), GroupBy.FILTER)
    return math.sqrt(float(torch.sum(norms * norms)))


def project(t, constraint: SparsityConstraint) -> torch.Tensor:
    """Keep the top-k groups by Frobenius norm (lower index wins ties); zero the rest."""
    t = as_cuda_f32(t)
    if t.dim() != 4:
        raise ShapeError(f"projection needs a rank-4 tensor, got rank {t.dim()}")
    out, _, _ = _run_projection(t, resolve_plan(tuple(t.shape), [constraint]))
    return out


def project_composite(t, constraints: list[SparsityConstraint]) -> torch.Tensor:
    """Sequential projections in the listed order, norms recomputed after each."""
    t = as_cuda_f32(t)
    plan = resolve_plan(tuple(t.shape), constraints) if constraints else []
    if not plan:
        return t.clone()
    if t.dim() != 4:
        raise ShapeError(f"projection needs a rank-4 tensor, got rank {t.dim()}")
    out, _, _ = _run_projection(t, plan)
    return out


def extract_mask(t) -> torch.Tensor:
    """Bool support mask, ``|t| > 0`` elementwise."""
    t = as_cuda_f32(t)
    out = torch.empty(t.shape, dtype=torch.bool, device=t.device)
    _lib.call("hsx_nonzero_u8", t.data_ptr(), t.numel(), out.data_ptr(), current_stream())
    return out


def mask_drift(prev, cur) -> float:
    """Fraction of differing bits between two equal-shape masks."""
    if tuple(prev.shape) != tuple(cur.shape):
        raise ShapeError(f"mask shape mismatch: {tuple(prev.shape)} vs {tuple(cur.shape)}")
    a = torch.as_tensor(prev).to("cuda", torch.bool).contiguous()
    b = torch.as_tensor(cur).to("cuda", torch.bool).contiguous()
    n = a.numel()
    if n == 0:
        return float("nan")
    cnt = torch.zeros(1, dtype=torch.int64, device=a.device)
    _lib.call("hsx_count_diff_u8", a.data_ptr(), b.data_ptr(), n, cnt.data_ptr(), current_stream())
    return int(cnt.item()) / n
