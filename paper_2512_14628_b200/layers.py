"""Layer metadata shared by the host API and the C-ABI layer table.

Mirrors the reference's ``LayerKind`` / ``GroupBy`` / ``LayerSpec``
(/root/reference/pkg/src/admmprune/tensors.py:19-56): conv weights are rank-4
``(c_out, c_in, kh, kw)`` row-major, fully connected weights rank-2, and only
conv layers may be pruned. BN scales/shifts and biases travel as rank-2
``(1, d)`` dense layers.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass

from .errors import ShapeError


class LayerKind(enum.Enum):
    CONV = "conv"
    FULLY_CONNECTED = "fc"


class GroupBy(enum.Enum):
    """Structured groups of a rank-4 weight (reference tensors.py:25-30)."""

    FILTER = "filter"          # one group per output filter (c_out groups)
    CHANNEL = "channel"        # one group per input channel (c_in groups)
    SHAPE_POSITION = "shape"   # one group per (c_in, kh, kw) column


# integer codes used by the C ABI (include/hsx.h HSX_GROUP_*)
GROUP_CODE = {GroupBy.FILTER: 0, GroupBy.CHANNEL: 1, GroupBy.SHAPE_POSITION: 2}


@dataclass(frozen=True)
class LayerSpec:
    """Static description of one weight tensor (reference tensors.py:33-56)."""

    name: str
    kind: LayerKind
    shape: tuple[int, ...]
    prunable: bool = False

    def __post_init__(self):
        dims = tuple(int(d) for d in self.shape)
        if any(d <= 0 for d in dims):
            raise ShapeError(f"layer {self.name}: non-positive dimension in {self.shape}")
        want = 4 if self.kind is LayerKind.CONV else 2
        if len(dims) != want:
            raise ShapeError(
                f"{self.kind.value} layer {self.name} must be rank-{want}, got {self.shape}")
        if self.prunable and self.kind is not LayerKind.CONV:
            raise ShapeError(f"layer {self.name}: only conv layers are prunable")
        object.__setattr__(self, "shape", dims)

    @property
    def elements(self) -> int:
        return int(math.prod(self.shape))


def group_count(shape: tuple[int, ...], group: GroupBy) -> int:
    if group is GroupBy.FILTER:
        return shape[0]
    if group is GroupBy.CHANNEL:
        return shape[1]
    return shape[1] * shape[2] * shape[3]
