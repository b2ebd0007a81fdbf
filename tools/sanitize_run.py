"""Exercise every device path once on small inputs, for compute-sanitizer
(racecheck / memcheck on the tiny config):

    PYTORCH_NO_CUDA_MEMORY_CACHING=1 compute-sanitizer --tool memcheck \\
        python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Paths: BASELINE config 1 (N=1024, 64x64) render + backward (atomic and
deterministic, explicit gradient and fused L2), sort_by="gamma", mode="splat",
cone-beam and parallel-beam tomography forward + adjoint (atomic and
deterministic), an SH-3 multi-view step through the pipelined
ViewShardedStep (three contexts, side stream, two blend streams), the fused
Adam step, the ray marcher and the voxelizer.  Prints one line per path.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2412_03378_b200 as vg
    from types import SimpleNamespace
    from paper_2412_03378_b200 import configs, groundtruth, tomo
    from paper_2412_03378_b200.engine import Engine
    from paper_2412_03378_b200.multiview import ViewShardedStep
    cfg = configs.tiny()
    s, cam = cfg.scene, cfg.cameras[0]
    scene = SimpleNamespace(means=s.means.astype(np.float64), scales=s.scales.astype(np.float64),
                            rotations=s.rotations.astype(np.float64), thetas=s.thetas.astype(np.float64),
                            colors=s.colors.astype(np.float64), splat_opacities=np.full(len(s.means), 0.6),
                            background=np.array([0.1, 0.2, 0.3]))
    dc = np.random.default_rng(0).uniform(-1, 1, (64, 64, 3))
    out = vg.render(scene, cam)
    print("render", float(out.color.sum()))
    for det in (False, True):
        g = vg.backward(scene, cam, dc, deterministic=det)
        print("backward det" if det else "backward atomic", float(np.abs(g.d_means).sum()))
    gg = vg.backward(scene, cam, dc, sort_by="gamma")
    print("gamma", float(np.abs(gg.d_means).sum()))
    sp = vg.render(scene, cam, mode="splat")
    gs = vg.backward(scene, cam, dc, mode="splat")
    print("splat", float(sp.color.sum()), float(np.abs(gs.d_means).sum()))
    w = np.random.default_rng(1).uniform(0.1, 1.0, (64, 64))
    for parallel in (False, True):
        img = vg.tomo_forward(scene, cam, parallel=parallel)
        for det in (False, True):
            gt = vg.tomo_backward(scene, cam, w, parallel=parallel, deterministic=det)
            print(f"tomo parallel={parallel} det={det}", float(img.sum()), float(np.abs(gt.d_means).sum()))
    big = configs.large(n=3000, width=96, height=64, n_views=4)
    for det in (False, True):
        eng = Engine(deterministic=det)
        targets = {v: torch.from_numpy(big.target(v, (64, 96, 3))).cuda() for v in range(4)}
        step = ViewShardedStep(eng, eng.upload(big.scene), big.cameras, targets)
        print(f"multiview SH det={det}", float(step()))
    from paper_2412_03378_b200 import optim
    tc = optim.TrainConfig(iterations=2, loss="l2")
    _, rep = optim.fit_image([cfg.target(0, (64, 64, 3))], [cam], tc, init_scene=scene)
    print("fit_image", rep.losses)
    col, tf = groundtruth.raymarch_image(scene, vg.look_at([0, 0, -3.0], [0, 0, 0], width=16, height=16,
                                                            fov_x_deg=60.0))
    print("raymarch", float(col.sum()))
    grid = tomo.voxelize(scene, resolution=12)
    print("voxelize", float(grid.values.sum()))
    torch.cuda.synchronize()
    print("sanitize_run done")


if __name__ == "__main__":
    main()
