"""Generate the I/O and ray-march fixtures by running the REFERENCE:

* io_scene.txt / io_camera.txt: volgauss.sceneio.save_scene / save_camera of a
  seeded 7-primitive scene with two named cameras (repr floats, exact round
  trip) -- the byte-level contract of the text formats (sceneio.py:16-170);
* raymarch.npz: volgauss.oracle.raymarch_image (oracle.py:80-161; midpoint
  rule, 10 000 steps, auto-fitted bounds) of the config-1 miniature and of
  the reference's golden scene (inputs from golden_scene.npz) -- the ground
  truth the GPU ray marcher reproduces.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src:. \\
        python tests/golden/make_golden_io.py
"""

from __future__ import annotations

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from volgauss import oracle, raster, scenes, sceneio  # noqa: E402  (reference)


def main():
    rng = scenes.make_rng(61)
    n = 7
    q = rng.standard_normal((n, 4))
    scene = raster.Scene(means=rng.uniform(-1, 1, (n, 3)), scales=rng.uniform(0.05, 0.3, (n, 3)),
                         rotations=q, thetas=rng.uniform(0, 1, n), colors=rng.uniform(0, 1, (n, 3)),
                         splat_opacities=rng.uniform(0, 1, n), background=(0.05, 0.1, 0.2))
    cam_a = scenes.Camera(width=40, height=30, fx=35.5, fy=36.25, cx=20.0, cy=15.0,
                          rotation=np.eye(3), translation=np.array([0.0, 0.0, 3.0]), z_near=0.02)
    cam_b = scenes.Camera(width=33, height=21, fx=29.0, fy=29.0, cx=16.5, cy=10.5,
                          rotation=np.array([[0.0, 0.0, -1.0], [0.0, 1.0, 0.0], [1.0, 0.0, 0.0]]),
                          translation=np.array([0.1, -0.2, 4.0]))
    sceneio.save_scene(os.path.join(HERE, "io_scene.txt"), scene, {"front": cam_a, "side": cam_b})
    sceneio.save_camera(os.path.join(HERE, "io_camera.txt"), cam_b)

    out = {}
    g = np.load(os.path.join(HERE, "golden_scene.npz"))
    gscene = raster.Scene(g["means"], g["scales"], g["rotations"], g["thetas"], g["colors"],
                          background=g["background"])
    w, h = (int(v) for v in g["cam_wh"])
    fx, fy, cx, cy, zn = g["cam_f"]
    gcam = scenes.Camera(width=w, height=h, fx=fx, fy=fy, cx=cx, cy=cy, rotation=g["cam_R"],
                         translation=g["cam_t"])
    col, tf = oracle.raymarch_image(gscene, gcam)
    out.update(golden_color=col, golden_T=tf)
    # a denser miniature: 40 primitives of config 1 at 24x24
    t = np.load(os.path.join(HERE, "tiny.npz"))
    sel = np.arange(0, 1024, 26)[:40]
    mscene = raster.Scene(t["means"][sel], t["scales"][sel], t["rotations"][sel], t["thetas"][sel],
                          t["colors"][sel], background=(0.1, 0.2, 0.3))
    mcam = scenes.Camera(width=24, height=24, fx=20.78, fy=20.78, cx=12.0, cy=12.0,
                         rotation=np.eye(3), translation=np.array([0.0, 0.0, 3.0]))
    col, tf = oracle.raymarch_image(mscene, mcam)
    out.update(mini_sel=sel, mini_color=col, mini_T=tf, mini_cam_f=np.array([20.78, 20.78, 12.0, 12.0]))
    np.savez_compressed(os.path.join(HERE, "raymarch.npz"), **out)
    print("io_scene.txt, io_camera.txt, raymarch.npz written")


if __name__ == "__main__":
    main()
