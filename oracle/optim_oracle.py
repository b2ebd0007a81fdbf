"""CPU float64 oracle for the training-step caller of the hot path (SURVEY
8(f) item 1): Adam over the parameter groups, the constraint projections,
the positional-gradient accumulator and the density-aware densify / prune
rules of the reference's `optim.py`.

TEST INFRASTRUCTURE ONLY (see volgauss_oracle.py's header): a numpy
restatement of `pkg/src/volgauss/optim.py` (paths relative to the
reference's `pkg/src/volgauss/`), pinned bit-for-bit against golden vectors
that `tests/golden/make_golden_optim.py` produced by running the reference's
own `Trainer.step` and `densify_and_prune` (tests/test_optim_pins.py).
The product package never imports it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .volgauss_oracle import SCALE_FLOOR, THETA_CEILING, kappa_of, quat_to_rotmat

GROUPS = ("position", "scale", "rotation", "color", "density")


@dataclass
class TrainConfig:
    """The optimizer / densification fields of optim.TrainConfig (optim.py:24-53)."""
    iterations: int = 1000
    lr_position: float = 1.6e-4
    lr_position_final: float = 1e-5
    lr_theta: float = 0.03
    lr_color: float = 0.003
    lr_scale: float = 5e-3
    lr_rotation: float = 1e-3
    split_grad_threshold: float = 1e-8
    clone_grad_threshold: float = 5e-5
    prune_theta_min: float = 0.005
    prune_scale_fraction: float = 0.01
    high_kappa_split_fraction: float = 0.9
    max_primitives: int = 20000


class Adam:
    """optim.Adam (optim.py:84-107): per-array moments, bias-corrected update."""

    def __init__(self, shape, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        self.m = np.zeros(shape)
        self.v = np.zeros(shape)
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps
        self.t = 0

    def step(self, grad, lr=None):
        self.t += 1
        g = np.asarray(grad, dtype=float)
        self.m = self.beta1 * self.m + (1 - self.beta1) * g
        self.v = self.beta2 * self.v + (1 - self.beta2) * g * g
        mhat = self.m / (1 - self.beta1 ** self.t)
        vhat = self.v / (1 - self.beta2 ** self.t)
        return (self.lr if lr is None else lr) * mhat / (np.sqrt(vhat) + self.eps)

    def surgery(self, keep, n_new):
        """optim.py:104-107: drop rows not kept, append zero moments."""
        self.m = np.concatenate([self.m[keep], np.zeros((n_new,) + self.m.shape[1:])])
        self.v = np.concatenate([self.v[keep], np.zeros((n_new,) + self.v.shape[1:])])


def softplus(x):
    """optim._softplus (optim.py:110-111), sharpness 10."""
    return np.logaddexp(0.0, 10.0 * x) / 10.0


def softplus_inv(y):
    """optim._softplus_inv (optim.py:114-116)."""
    y = np.asarray(y, dtype=float)
    return y + np.log1p(-np.exp(-10.0 * y)) / 10.0


def sigmoid(x):
    """scipy.special.expit, as optim.py:148 uses it (bit-identical)."""
    from scipy.special import expit
    return expit(x)


class Trainer:
    """optim.Trainer, analytic mode (optim.py:119-175): raw colours live
    pre-softplus; after every step theta is clipped to [0, 1], scales are
    floored and quaternions renormalised."""

    def __init__(self, scene, config: TrainConfig, extent):
        self.scene = scene
        self.config = config
        self.extent = extent
        self.color_raw = softplus_inv(np.clip(scene.colors, 1e-6, None))
        n = len(scene.means)
        c = config
        self.opts = {"position": Adam((n, 3), c.lr_position), "scale": Adam((n, 3), c.lr_scale),
                     "rotation": Adam((n, 4), c.lr_rotation), "color": Adam((n, 3), c.lr_color),
                     "density": Adam((n,), c.lr_theta)}

    def lr_position_at(self, iteration):
        """optim.py:140-144: exponential decay, scaled by the scene extent."""
        c = self.config
        frac = iteration / max(c.iterations - 1, 1)
        return c.lr_position * (c.lr_position_final / c.lr_position) ** frac * self.extent

    def step(self, grads, iteration):
        """optim.py:146-175; raises FloatingPointError (the reference's
        DivergenceError) on a non-finite update, naming group and primitive."""
        s = self.scene
        d_color_raw = grads.d_colors * sigmoid(10.0 * self.color_raw)
        updates = {
            "position": self.opts["position"].step(grads.d_means, lr=self.lr_position_at(iteration)),
            "scale": self.opts["scale"].step(grads.d_scales),
            "rotation": self.opts["rotation"].step(grads.d_rotations),
            "color": self.opts["color"].step(d_color_raw),
            "density": self.opts["density"].step(grads.d_thetas),
        }
        for name, u in updates.items():
            bad = ~np.isfinite(u)
            if bad.any():
                raise FloatingPointError(f"non-finite {name} update for primitive {int(np.argwhere(bad)[0][0])}")
        s.means = s.means - updates["position"]
        s.scales = np.maximum(s.scales - updates["scale"], SCALE_FLOOR)
        s.rotations = s.rotations - updates["rotation"]
        s.rotations = s.rotations / np.linalg.norm(s.rotations, axis=1, keepdims=True)
        self.color_raw = self.color_raw - updates["color"]
        s.colors = softplus(self.color_raw)
        s.thetas = np.clip(s.thetas - updates["density"], 0.0, 1.0)


class GradAccum:
    """optim.GradAccum (optim.py:194-206): windowed positional-gradient norms
    of the primitives visible in each step."""

    def __init__(self, n):
        self.norm_sum = np.zeros(n)
        self.count = np.zeros(n)

    def update(self, grads):
        norms = np.linalg.norm(grads.d_means, axis=1)
        vis = np.asarray(grads.visible, dtype=bool)
        self.norm_sum[vis] += norms[vis]
        self.count[vis] += 1

    def averages(self):
        return self.norm_sum / np.maximum(self.count, 1.0)


def theta_for_kappa(kappa, scales):
    """core.theta_for_kappa (core.py:146-153)."""
    s = np.maximum(np.asarray(scales, dtype=float), SCALE_FLOOR)
    inv_mean = np.mean(1.0 / s, axis=-1)
    return np.clip(-np.expm1(-np.asarray(kappa, dtype=float) / inv_mean) / THETA_CEILING, 0.0, 1.0)


def densify_masks(scene, accum: GradAccum, config: TrainConfig, extent):
    """The split / clone / prune decisions of densify_and_prune
    (optim.py:218-240, 292-297), including the primitive budget."""
    n = len(scene.means)
    avg = accum.averages()
    kappas = kappa_of(scene.thetas, scene.scales)
    ceilings = kappa_of(np.ones(n), scene.scales)
    max_scale = scene.scales.max(axis=1)
    big = max_scale > config.prune_scale_fraction * extent
    split = ((avg > config.split_grad_threshold) & big) | (kappas > config.high_kappa_split_fraction * ceilings)
    clone = (avg > config.clone_grad_threshold) & ~big & ~split
    budget = max(config.max_primitives - n, 0)
    grow = np.flatnonzero(split | clone)
    if len(grow) > budget:
        drop = grow[budget:]
        split[drop] = False
        clone[drop] = False
    prune = (scene.thetas < config.prune_theta_min) | (max_scale > config.prune_scale_fraction * extent)
    return split, clone, prune & ~(split | clone), kappas


def densify_and_prune(scene, trainer: Trainer, accum: GradAccum, config: TrainConfig, extent, rng):
    """optim.densify_and_prune, analytic mode (optim.py:218-317) without the
    event log: splits draw rng.standard_normal((2, 3)) per split parent in
    index order, children halve kappa (theta clamped at the ceiling), parents
    of splits / clones are replaced, pruned primitives dropped; Adam moments
    keep the surviving rows and start at zero for the children."""
    split, clone, prune, kappas = densify_masks(scene, accum, config, extent)
    rot = quat_to_rotmat(scene.rotations)
    new = {k: [] for k in ("means", "scales", "rotations", "thetas", "colors")}

    def emit(parent, child_means, child_scales):
        for cm, cs in zip(child_means, child_scales):
            target = 0.5 * kappas[parent]
            ceiling = kappa_of(np.ones(1), cs[None])[0]
            th = 1.0 if target > ceiling * (1.0 + 1e-12) else float(theta_for_kappa(target, cs))
            new["means"].append(cm)
            new["scales"].append(cs)
            new["rotations"].append(scene.rotations[parent].copy())
            new["thetas"].append(th)
            new["colors"].append(scene.colors[parent].copy())

    for p in np.flatnonzero(split):
        cs = scene.scales[p] / 1.6
        xi = rng.standard_normal((2, 3))
        means = scene.means[p] + (rot[p] @ (scene.scales[p] * xi).T).T
        emit(p, list(means), [cs.copy(), cs.copy()])
    for p in np.flatnonzero(clone):
        cs = scene.scales[p].copy()
        emit(p, [scene.means[p].copy(), scene.means[p].copy()], [cs, cs.copy()])
    keep = ~(split | clone | prune)
    n_new = len(new["means"])
    scene.means = np.concatenate([scene.means[keep], np.array(new["means"]).reshape(n_new, 3)])
    scene.scales = np.concatenate([scene.scales[keep], np.array(new["scales"]).reshape(n_new, 3)])
    scene.rotations = np.concatenate([scene.rotations[keep], np.array(new["rotations"]).reshape(n_new, 4)])
    scene.thetas = np.concatenate([scene.thetas[keep], np.array(new["thetas"])])
    scene.colors = np.concatenate([scene.colors[keep], np.array(new["colors"]).reshape(n_new, 3)])
    for opt in trainer.opts.values():
        opt.surgery(keep, n_new)
    trainer.color_raw = np.concatenate(
        [trainer.color_raw[keep], softplus_inv(np.clip(scene.colors[len(scene.means) - n_new:], 1e-6, None))])
    return split, clone, prune
