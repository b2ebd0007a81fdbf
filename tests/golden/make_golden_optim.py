"""Generate tests/golden/optim.npz by running the REFERENCE training-step code
(volgauss 0.1.0 optim.Trainer.step, GradAccum, densify_and_prune) itself.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src:. \\
        python tests/golden/make_golden_optim.py

A 300-primitive scene (float32-rounded inputs, some primitives below the
prune density, some larger than the prune scale, some at high kappa) takes
three Trainer.step calls with seeded synthetic gradients, accumulating the
positional-gradient norms of the visible primitives; then one
densify_and_prune with a seeded Philox generator and a primitive budget that
truncates the growth.  The fixture stores the inputs, the scene and the Adam
moments after every step, and the densified scene.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from volgauss import grad, optim, raster  # noqa: E402  (reference)


def f32(a):
    return np.asarray(np.asarray(a, dtype=np.float32), dtype=np.float64)


def main():
    rng = np.random.default_rng(7)
    n = 300
    means = f32(rng.uniform(-1, 1, (n, 3)))
    scales = f32(np.exp(rng.uniform(np.log(0.004), np.log(0.06), (n, 3))))
    q = rng.standard_normal((n, 4))
    rots = f32(q / np.linalg.norm(q, axis=1, keepdims=True))
    thetas = f32(rng.uniform(0.0, 0.4, n))
    thetas[:10] = f32(rng.uniform(0.0, 0.004, 10))          # prune by theta
    thetas[10:20] = f32(rng.uniform(0.97, 1.0, 10))         # high kappa -> split
    colors = f32(rng.uniform(0.02, 0.98, (n, 3)))
    scene = raster.Scene(means.copy(), scales.copy(), rots.copy(), thetas.copy(), colors.copy())
    cfg = optim.TrainConfig(iterations=50, max_primitives=330)
    extent = 4.0
    trainer = optim.Trainer(scene, cfg, "analytic", extent)
    accum = optim.GradAccum(n)
    out = dict(means=means, scales=scales, rotations=rots, thetas=thetas, colors=colors,
               extent=np.array(extent), max_primitives=np.array(cfg.max_primitives),
               iterations=np.array(cfg.iterations))
    for it in range(3):
        g = grad.SceneGrads(n, "analytic")
        g.d_means = f32(rng.standard_normal((n, 3)) * 3e-4)
        g.d_scales = f32(rng.standard_normal((n, 3)) * 1e-3)
        g.d_rotations = f32(rng.standard_normal((n, 4)) * 1e-3)
        g.d_thetas = f32(rng.standard_normal(n) * 1e-2)
        g.d_colors = f32(rng.standard_normal((n, 3)) * 1e-2)
        g.visible = rng.uniform(0, 1, n) < 0.8
        for k in ("d_means", "d_scales", "d_rotations", "d_thetas", "d_colors", "visible"):
            out[f"g{it}_{k}"] = getattr(g, k)
        accum.update(g)
        trainer.step(g, it)
        for k in ("means", "scales", "rotations", "thetas", "colors"):
            out[f"s{it}_{k}"] = getattr(scene, k).copy()
        out[f"s{it}_color_raw"] = trainer.color_raw.copy()
        for name, opt in trainer.opts.items():
            out[f"s{it}_{name}_m"] = opt.m.copy()
            out[f"s{it}_{name}_v"] = opt.v.copy()
    out["accum_norm"] = accum.norm_sum.copy()
    out["accum_count"] = accum.count.copy()
    drng = np.random.Generator(np.random.Philox(key=11))
    events = optim.densify_and_prune(scene, trainer, accum, cfg, extent, drng, 3, "analytic")
    for k in ("means", "scales", "rotations", "thetas", "colors"):
        out[f"d_{k}"] = getattr(scene, k).copy()
    out["d_color_raw"] = trainer.color_raw.copy()
    for name, opt in trainer.opts.items():
        out[f"d_{name}_m"] = opt.m.copy()
        out[f"d_{name}_v"] = opt.v.copy()
    out["d_event_kinds"] = np.array([{"split": 0, "clone": 1, "prune": 2}[e.kind] for e in events])
    out["d_event_parents"] = np.array([e.parent for e in events])
    np.savez_compressed(os.path.join(HERE, "optim.npz"), **out)
    kinds = out["d_event_kinds"]
    print(f"optim.npz: {n} -> {len(scene)} primitives; splits {int((kinds == 0).sum())}, "
          f"clones {int((kinds == 1).sum())}, prunes {int((kinds == 2).sum())}")


if __name__ == "__main__":
    sys.exit(main())
