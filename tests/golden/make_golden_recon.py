"""Generate tests/golden/recon.npz by running the REFERENCE tomography
reconstruction and voxelizer (volgauss 0.1.0 tomo.reconstruct, tomo.voxelize)
themselves.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src:. \\
        python tests/golden/make_golden_recon.py

Inputs: six 24x24 cone-beam projections of the reference's blob phantom (the
projections themselves are stored, so the test needs no phantom code), an
L2 TrainConfig with 16 initial primitives and 24 iterations (no densify
before iteration 24), seed 0; and the same run with loss="mixed" (the
reference's default: 0.8 L1 + 0.2 D-SSIM), mixed_* keys.  Stored: the projections and cameras, the loss
of every iteration, the final scene, its voxel grid at resolution 20, the
psnr_3d / ssim_3d against the phantom grid, and a separate voxelize case
(anisotropic rotated primitives, anisotropic resolution, box partly outside),
and a density grid written by tomo.save_density_grid (io_grid.raw / .txt).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from volgauss import raster, tomo  # noqa: E402  (reference)
from volgauss.optim import TrainConfig  # noqa: E402


def main():
    ph = tomo.blob_phantom()
    geo = tomo.TomoGeometry(width=24, height=24)
    projs = tomo.make_phantom_projections(ph, 6, geo)
    ref_grid = tomo.grid_from_phantom(ph, resolution=20, bbox=(-np.ones(3), np.ones(3)))
    cfg = TrainConfig(iterations=24, loss="l2", n_init=16, seed=0)
    scene, grid, rep = tomo.reconstruct(projs, cfg, resolution=20, reference=ref_grid)
    out = {}
    for k, p in enumerate(projs):
        c = p.camera
        out[f"p{k}_image"] = p.image
        out[f"p{k}_cam"] = np.array([c.width, c.height, c.fx, c.fy, c.cx, c.cy, c.z_near])
        out[f"p{k}_rot"] = np.asarray(c.rotation, dtype=float)
        out[f"p{k}_trans"] = np.asarray(c.translation, dtype=float)
    out["n_proj"] = np.array(len(projs))
    out["ref_grid"] = ref_grid.values
    out["losses"] = np.array(rep["losses"])
    out["counts"] = np.array(rep["primitive_counts"])
    for k in ("means", "scales", "rotations", "thetas"):
        out[f"final_{k}"] = getattr(scene, k)
    out["grid"] = grid.values
    out["psnr_3d"] = np.array(rep["psnr_3d"])
    out["ssim_3d"] = np.array(rep["ssim_3d"])
    # the same run with the reference's default loss, mixed (0.8 L1 + 0.2 D-SSIM)
    cfg_m = TrainConfig(iterations=24, loss="mixed", n_init=16, seed=0)
    scene_m, grid_m, rep_m = tomo.reconstruct(projs, cfg_m, resolution=20, reference=ref_grid)
    out["mixed_losses"] = np.array(rep_m["losses"])
    for k in ("means", "scales", "rotations", "thetas"):
        out[f"mixed_final_{k}"] = getattr(scene_m, k)
    out["mixed_grid"] = grid_m.values
    out["mixed_psnr_3d"] = np.array(rep_m["psnr_3d"])
    # voxelize on its own
    rng = np.random.default_rng(5)
    n = 40
    q = rng.standard_normal((n, 4))
    vs = raster.Scene(means=rng.uniform(-1.1, 1.1, (n, 3)),
                      scales=np.exp(rng.uniform(np.log(0.03), np.log(0.3), (n, 3))),
                      rotations=q / np.linalg.norm(q, axis=1, keepdims=True),
                      thetas=rng.uniform(0.02, 0.9, n), colors=np.full((n, 3), 0.5))
    bmin, bmax = np.array([-1.0, -0.8, -1.2]), np.array([0.9, 1.1, 1.0])
    vg = tomo.voxelize(vs, resolution=(18, 14, 22), bbox=(bmin, bmax))
    out.update(vox_means=vs.means, vox_scales=vs.scales, vox_rotations=vs.rotations,
               vox_thetas=vs.thetas, vox_bmin=bmin, vox_bmax=bmax, vox_values=vg.values)
    # boxes tomo.voxelize accepts unchecked: a flat one (zero spacing on y) and a
    # reversed one (bbox_max < bbox_min on x)
    for tag, lo, hi in (("flat", [-1.0, 0.1, -1.2], [0.9, 0.1, 1.0]),
                        ("reversed", [0.9, -0.8, -1.2], [-1.0, 1.1, 1.0])):
        g = tomo.voxelize(vs, resolution=(9, 7, 11), bbox=(np.array(lo), np.array(hi)))
        out[f"vox_{tag}_bmin"], out[f"vox_{tag}_bmax"] = np.array(lo), np.array(hi)
        out[f"vox_{tag}_values"] = g.values
    np.savez_compressed(os.path.join(HERE, "recon.npz"), **out)
    # density grid I/O (tomo.save_density_grid): a 5x6x7 grid with negative and
    # awkward values and an asymmetric box -> io_grid.raw / io_grid.txt
    gv = rng.normal(size=(5, 6, 7)) / 3.0
    tomo.save_density_grid(os.path.join(HERE, "io_grid"),
                           tomo.DensityGrid(values=gv, bbox_min=np.array([-1.0, -0.5, -2.0 / 3.0]),
                                            bbox_max=np.array([1.25, 0.1, 0.7])))
    np.save(os.path.join(HERE, "io_grid_values.npy"), gv)
    print(f"recon.npz: losses {rep['losses'][0]:.4g} -> {rep['losses'][-1]:.4g}, "
          f"psnr_3d {rep['psnr_3d']:.3f}, ssim_3d {rep['ssim_3d']:.4f}, vox max {vg.values.max():.4g}")


if __name__ == "__main__":
    sys.exit(main())
