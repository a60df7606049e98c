"""Readers for the golden fixtures written by tests/golden/make_golden.py."""

from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
KIND_NAMES = ("filter", "channel", "shape")

# mirrors make_golden.E2E_LAYERS (the fixture generator needs the reference; this does not)
E2E_LAYERS = [
    ("stem", "conv", (8, 3, 3, 3), [("channel", 0.5)]),
    ("bn1.w", "fc", (1, 8), []),
    ("conv_a", "conv", (16, 8, 3, 3), [("channel", 0.5)]),
    ("conv_b", "conv", (32, 16, 1, 1), [("channel", 0.4)]),
    ("conv_c", "conv", (8, 32, 3, 3), [("filter", 0.75), ("channel", 0.5)]),
    ("conv_d", "conv", (12, 8, 1, 1), [("shape", 0.5)]),
    ("conv_e", "conv", (8, 12, 3, 3), []),
    ("fc.w", "fc", (10, 8), []),
    ("fc.b", "fc", (1, 10), []),
]
E2E_RHO1, E2E_RHO2, E2E_WD = 1.5e-3, 1.5e-4, 1e-4
E2E_TOPOLOGIES = [(1, 1), (2, 1), (1, 2), (2, 2), (2, 4), (4, 2), (1, 4), (4, 1)]
E2E_ADAPT_TOPOLOGIES = [(1, 1), (2, 1), (1, 2), (2, 2), (2, 4), (4, 2)]   # phase 5 with adaptive penalties


def load(name):
    return np.load(os.path.join(GOLDEN, name))


def projection_cases():
    d = load("projection.npz")
    singles = []
    for i in range(int(d["n_single"])):
        kind, keep = d[f"c{i}_meta"]
        singles.append(dict(t=d[f"c{i}_in"], kind=KIND_NAMES[kind], keep=int(keep),
                            norms=d[f"c{i}_norms"], out=d[f"c{i}_out"], mask=d[f"c{i}_mask"]))
    comps = []
    for i in range(int(d["n_composite"])):
        plan = [(KIND_NAMES[k], int(kp)) for k, kp in d[f"p{i}_plan"]]
        comps.append(dict(t=d[f"p{i}_in"], plan=plan, out=d[f"p{i}_out"]))
    return singles, comps


def shrinkage_cases():
    d = load("shrinkage.npz")
    return [dict(mask=d[f"s{i}_mask"], t=d[f"s{i}_t"], k_out=d[f"s{i}_kout"], k_in=d[f"s{i}_kin"],
                 compact=d[f"s{i}_compact"], restored=d[f"s{i}_restored"]) for i in range(int(d["n"]))]


def bucketize_cases():
    with open(os.path.join(GOLDEN, "bucketize.json")) as fh:
        return json.load(fh)


def candidate_cases():
    d = load("candidate.npz")
    return [dict(svz=d[f"k{i}_svz"], par=d[f"k{i}_par"], out=d[f"k{i}_out"]) for i in range(int(d["n"]))]


class E2E:
    """One end-to-end reference run (run_hierarchical, phase 1 replaced)."""

    def __init__(self, num_nodes, per_node, adapt=False):
        self.d = load(f"{'e2e_adapt' if adapt else 'e2e'}_{num_nodes}x{per_node}.npz")
        self.M, self.P, self.iters, self.t_freeze = (int(x) for x in self.d["meta"])
        self.world = self.M * self.P
        self.names = [n for n, *_ in E2E_LAYERS]

    def p0(self):
        return {n: self.d[f"p0/{n}"].astype(np.float64) for n in self.names}

    def theta(self, k, r):
        return {n: self.d[f"theta/{k}/{r}/{n}"].astype(np.float64) for n in self.names}

    def u(self, k, r):
        return {n: self.d[f"u/{k}/{r}/{n}"] for n in self.names}

    def node_state(self, grp, k, node):
        return {n: self.d[f"{grp}/{k}/{node}/{n}"] for n in self.names}

    def masks(self, k, node):
        return {n: self.d[f"mask/{k}/{node}/{n}"] for n, _, _, c in E2E_LAYERS if c}

    def frozen(self, k, node):
        return bool(self.d[f"frozen/{k}/{node}"])

    def cache(self, k, r):
        return tuple(int(x) for x in self.d[f"cache/{k}/{r}"])

    def zsync(self, k):
        return json.loads(str(self.d[f"zsync/{k}"]))

    # phase 5 (adaptive runs only): the report packed as consensus.pack_report
    # (per layer r_intra, s_intra, r_inter, s_inter, eps_pri_intra, eps_dual_intra,
    # eps_pri_inter, eps_dual_inter; then r_pri, r_dual, eps_pri, eps_dual, converged),
    # the penalties iteration k ran with, and each rank's local r_intra
    def report(self, k):
        return self.d[f"report/{k}"]

    def rho(self, k):
        return self.d[f"rho1/{k}"], self.d[f"rho2/{k}"]

    def r_intra(self, k, r):
        return self.d[f"r_intra/{k}/{r}"]

    def rho_final(self):
        return self.d["rho_final"]

    def ledger(self, k):
        """Every ledger entry of iteration k (adaptive runs only)."""
        return json.loads(str(self.d[f"ledger/{k}"]))


def prox_case():
    """proximal_sgd fixture (make_golden.gen_prox): inputs, gradient sequence, output."""
    d = load("prox_sgd.npz")
    names = [n for n, *_ in E2E_LAYERS]
    lr, mom, steps = d["meta"]
    f64 = lambda key: {n: d[f"{key}/{n}"].astype(np.float64) for n in names}
    return dict(names=names, lr=float(lr), momentum=float(mom), rho1=dict(zip(names, d["rho1"].tolist())),
                w0=f64("w0"), z=f64("z"), u=f64("u"), out={n: d[f"out/{n}"] for n in names},
                grads=[{n: d[f"g/{i}/{n}"].astype(np.float64) for n in names} for i in range(int(steps))])


FLAT_CASES = [(2, False), (1, True), (2, True), (4, True)]   # (world, adapt)
DENSE_WORLDS = [1, 2, 4]


class Flat:
    """run_flat_consensus (baselines.py:151-293) with phase 1 replaced (make_golden.gen_flat):
    state after iteration k per rank (z, u post-rescale, masks, frozen, rho1 after
    adaptation), rank 0's report / rho1 / drift / mask popcounts, each rank's r_intra,
    the ledger of every iteration."""

    def __init__(self, world, adapt):
        self.d = load(f"flat_{'adapt_' if adapt else ''}{world}.npz")
        self.world, self.iters, self.t_freeze, adapt_ = (int(x) for x in self.d["meta"])
        self.adapt = bool(adapt_)
        self.names = [n for n, *_ in E2E_LAYERS]

    def p0(self):
        return {n: self.d[f"p0/{n}"].astype(np.float64) for n in self.names}

    def theta(self, k, r):
        return {n: self.d[f"theta/{k}/{r}/{n}"].astype(np.float64) for n in self.names}

    def state(self, key, k, r):
        return {n: self.d[f"{key}/{k}/{r}/{n}"] for n in self.names}

    def masks(self, k, r):
        return {n: self.d[f"mask/{k}/{r}/{n}"] for n, _, _, c in E2E_LAYERS if c}

    def frozen(self, k):
        return bool(self.d[f"frozen/{k}/0"])

    def report(self, k):
        return self.d[f"report/{k}"]

    def rho1(self, k):
        return self.d[f"rho1/{k}"]

    def rho1_after(self, k):
        return self.d[f"rho1_after/{k}/0"]

    def r_intra(self, k, r):
        return self.d[f"r_intra/{k}/{r}"]

    def drift(self, k):
        return json.loads(str(self.d[f"drift/{k}"]))

    def ledger(self, k):
        return json.loads(str(self.d[f"ledger/{k}"]))


class Dense:
    """run_dense_sync (baselines.py:77-98) with recorded per-rank gradients (make_golden.gen_dense)."""

    def __init__(self, world):
        self.d = load(f"dense_{world}.npz")
        self.world, self.steps = (int(x) for x in self.d["meta"])
        self.lr, self.momentum, self.weight_decay = (float(x) for x in self.d["solver"])
        self.names = [n for n, *_ in E2E_LAYERS]

    def p0(self):
        return {n: self.d[f"p0/{n}"].astype(np.float64) for n in self.names}

    def grads(self, s, r):
        return {n: self.d[f"g/{s}/{r}/{n}"].astype(np.float64) for n in self.names}

    def out(self):
        return {n: self.d[f"out/{n}"] for n in self.names}

    def ledger(self):
        return json.loads(str(self.d["ledger"]))


class TopK(Dense):
    """run_topk (baselines.py:101-148) with recorded gradients (make_golden.gen_topk):
    also every rank's selected indices per step and layer."""

    def __init__(self, world):
        self.d = load(f"topk_{world}.npz")
        self.world, self.steps = (int(x) for x in self.d["meta"])
        self.lr, self.momentum, self.weight_decay, self.rate = (float(x) for x in self.d["solver"])
        self.names = [n for n, *_ in E2E_LAYERS]

    def sel(self, s, r, n):
        return self.d[f"sel/{s}/{r}/{n}"]
