"""Generate tests/golden/camera.npz by running the REFERENCE camera helpers
(volgauss 0.1.0 camera.Camera.pixel_directions / view_to_pixel /
ray_through_pixel, look_at) and raster.Scene.gaussian.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src:. \\
        python tests/golden/make_golden_camera.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from volgauss import camera, raster  # noqa: E402  (reference)


def main():
    cam = camera.look_at([0.7, -1.1, -2.6], [0.1, 0.2, 0.0], up=(0.0, 1.0, 0.0), width=19, height=13,
                         fov_x_deg=47.0)
    rng = np.random.default_rng(3)
    v = rng.normal(size=(7, 3)) + np.array([0.0, 0.0, 3.0])
    ray = cam.ray_through_pixel(4, 11)
    s = raster.Scene(means=rng.normal(size=(3, 3)), scales=rng.uniform(0.1, 0.3, (3, 3)),
                     rotations=rng.normal(size=(3, 4)), thetas=rng.uniform(0.1, 0.9, 3),
                     colors=rng.uniform(0, 1, (3, 3)), splat_opacities=rng.uniform(0, 1, 3))
    g = s.gaussian(2)
    np.savez_compressed(
        os.path.join(HERE, "camera.npz"), R=cam.rotation, t=cam.translation, f=np.array([cam.fx, cam.fy]),
        c=np.array([cam.cx, cam.cy]), dirs=cam.pixel_directions(), v=v, px=cam.view_to_pixel(v),
        ray_o=ray.origin, ray_d=ray.direction, s_means=s.means, s_scales=s.scales, s_rot=s.rotations,
        s_thetas=s.thetas, s_colors=s.colors, s_opac=s.splat_opacities,
        g=np.concatenate([g.mean, g.scale, g.rotation, [g.theta], g.color, [g.splat_opacity]]))
    print("camera.npz written")


if __name__ == "__main__":
    sys.exit(main())
