"""Synthetic ResNet-shaped H-SADMM state (the BASELINE.json workloads).

Shapes are torchvision's parameter order (conv -> rank-4 prunable,
BN weight/bias and fc bias -> rank-2 ``(1, d)``, fc weight rank-2), hard-coded
so the package does not depend on torchvision. Parameter counts are pinned by
tests: RN18-CIFAR 11,173,962; RN18 11,689,512; RN50 25,557,032; RN152
60,192,808.

State recipe: a shared graded base ``N(0, 0.1)`` scaled per
input channel by ``U(0.2, 1.0)`` for conv layers (like the reference's
pretrained init, /root/reference/pkg/src/admmprune/workloads.py:254-258) from
stream ``[seed, 211]`` (the reference's ``_INIT_STREAM``, workloads.py:21);
``theta_r = base + N(0, 1e-3)`` from ``[seed, 307, r]``; ``u_r = 0.01 N(0, 0.1)``
from ``[seed, 401, r]``; ``v_i = 0.01 N(0, 0.1)`` from ``[seed, 503, i]`` shared by
the ranks of node ``i``; ``z = z_node = base``. Values are rounded to fp32 so
the fp64 oracle sees exactly the GPU's inputs.
"""

from __future__ import annotations

import numpy as np

from .layers import LayerKind, LayerSpec

_BLOCKS = {18: ("basic", (2, 2, 2, 2)), 34: ("basic", (3, 4, 6, 3)),
           50: ("bottleneck", (3, 4, 6, 3)), 101: ("bottleneck", (3, 4, 23, 3)),
           152: ("bottleneck", (3, 8, 36, 3))}

MODELS = {
    "rn18_cifar": dict(depth=18, cifar=True),
    "rn18_224": dict(depth=18, cifar=False),
    "rn50_224": dict(depth=50, cifar=False),
    "rn152_224": dict(depth=152, cifar=False),
}


def _conv(name, cout, cin, k):
    return LayerSpec(name, LayerKind.CONV, (cout, cin, k, k), prunable=True)


def _vec(name, d):
    return LayerSpec(name, LayerKind.FULLY_CONNECTED, (1, d))


def resnet_layers(depth: int, cifar: bool = False, classes: int | None = None) -> list[LayerSpec]:
    """Every trainable tensor of a torchvision ResNet, in parameter order."""
    style, counts = _BLOCKS[depth]
    classes = classes if classes is not None else (10 if cifar else 1000)
    out: list[LayerSpec] = []
    out.append(_conv("conv1.weight", 64, 3, 3 if cifar else 7))
    out += [_vec("bn1.weight", 64), _vec("bn1.bias", 64)]
    inplanes = 64
    expansion = 1 if style == "basic" else 4
    for stage, (planes, nblocks) in enumerate(zip((64, 128, 256, 512), counts), start=1):
        for b in range(nblocks):
            p = f"layer{stage}.{b}."
            stride = 2 if (stage > 1 and b == 0) else 1
            if style == "basic":
                out.append(_conv(p + "conv1.weight", planes, inplanes, 3))
                out += [_vec(p + "bn1.weight", planes), _vec(p + "bn1.bias", planes)]
                out.append(_conv(p + "conv2.weight", planes, planes, 3))
                out += [_vec(p + "bn2.weight", planes), _vec(p + "bn2.bias", planes)]
            else:
                width = planes
                out.append(_conv(p + "conv1.weight", width, inplanes, 1))
                out += [_vec(p + "bn1.weight", width), _vec(p + "bn1.bias", width)]
                out.append(_conv(p + "conv2.weight", width, width, 3))
                out += [_vec(p + "bn2.weight", width), _vec(p + "bn2.bias", width)]
                out.append(_conv(p + "conv3.weight", planes * 4, width, 1))
                out += [_vec(p + "bn3.weight", planes * 4), _vec(p + "bn3.bias", planes * 4)]
            if stride != 1 or inplanes != planes * expansion:
                out.append(_conv(p + "downsample.0.weight", planes * expansion, inplanes, 1))
                out += [_vec(p + "downsample.1.weight", planes * expansion),
                        _vec(p + "downsample.1.bias", planes * expansion)]
            inplanes = planes * expansion
    out.append(LayerSpec("fc.weight", LayerKind.FULLY_CONNECTED, (classes, 512 * expansion)))
    out.append(_vec("fc.bias", classes))
    return out


def model_layers(model: str) -> list[LayerSpec]:
    return resnet_layers(**MODELS[model])


def channel_keep_constraints(layers, keep_rate: float):
    """CHANNEL_KEEP(keep_rate) on every conv layer; everything else dense."""
    from .sparsity import ConstraintKind, SparsityConstraint

    c = SparsityConstraint(ConstraintKind.CHANNEL_KEEP, keep_rate=keep_rate)
    return {ls.name: [c] for ls in layers if ls.kind is LayerKind.CONV}


# -- synthetic state ----------------------------------------------------------


def _f32(a: np.ndarray) -> np.ndarray:
    return a.astype(np.float32)


def synthetic_base(layers, seed: int = 0) -> dict[str, np.ndarray]:
    rng = np.random.default_rng([seed, 211])
    base = {}
    for ls in layers:
        t = rng.normal(0.0, 0.1, size=ls.shape)
        if ls.kind is LayerKind.CONV:
            t *= rng.uniform(0.2, 1.0, size=(1, ls.shape[1], 1, 1))
        base[ls.name] = _f32(t)
    return base


def synthetic_rank_state(layers, rank: int, accels_per_node: int, seed: int = 0,
                         base: dict[str, np.ndarray] | None = None) -> dict[str, dict[str, np.ndarray]]:
    """fp32 numpy state of one rank: theta, u, z_node, v, z (per-layer dicts)."""
    base = synthetic_base(layers, seed) if base is None else base
    node = rank // accels_per_node
    r_t = np.random.default_rng([seed, 307, rank])
    r_u = np.random.default_rng([seed, 401, rank])
    r_v = np.random.default_rng([seed, 503, node])
    theta, u, v = {}, {}, {}
    for ls in layers:
        n = ls.name
        theta[n] = _f32(base[n] + r_t.normal(0.0, 1e-3, size=ls.shape))
        u[n] = _f32(0.01 * r_u.normal(0.0, 0.1, size=ls.shape))
        v[n] = _f32(0.01 * r_v.normal(0.0, 0.1, size=ls.shape))
    return {"theta": theta, "u": u, "z_node": {n: base[n].copy() for n in base},
            "v": v, "z": {n: base[n].copy() for n in base}}
