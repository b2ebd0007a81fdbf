"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
implementation (volgauss 0.1.0) itself.

Run in the build container, where the read-only reference is present:

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src:. \
        python tests/golden/make_golden.py

Each case stores its float32-rounded inputs (widened to float64 for the
reference), the camera, the flags, and the reference outputs of
raster.prepare / render, grad.backward and tomo.tomo_forward / tomo_backward.
Nothing at test time reads /root/reference; the tests read only these files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from volgauss import core, grad, raster, scenes, sceneio, tomo  # noqa: E402  (reference)

from paper_2412_03378_b200 import configs  # noqa: E402


def f32(a):
    return np.asarray(np.asarray(a, dtype=np.float32), dtype=np.float64)


def ref_scene(means, scales, rots, thetas, colors, bg=(0.0, 0.0, 0.0)):
    n = len(means)
    return raster.Scene(means=f32(means).reshape(n, 3), scales=f32(scales).reshape(n, 3),
                        rotations=f32(rots).reshape(n, 4), thetas=f32(thetas).reshape(n),
                        colors=f32(colors).reshape(n, 3), background=np.asarray(bg, dtype=float))


def cam_dict(cam):
    return dict(cam_wh=np.array([cam.width, cam.height]),
                cam_f=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.z_near]),
                cam_R=np.asarray(cam.rotation, dtype=float), cam_t=np.asarray(cam.translation, dtype=float))


def scene_dict(s):
    return dict(means=s.means, scales=s.scales, rotations=s.rotations, thetas=s.thetas,
                colors=s.colors, background=s.background)


def lists_dict(prefix, grid):
    flat = np.concatenate([np.asarray(t, dtype=np.int64) for t in grid.tiles]) if grid.tiles else np.zeros(0, np.int64)
    off = np.concatenate([[0], np.cumsum([len(t) for t in grid.tiles])]).astype(np.int64)
    return {f"{prefix}_prims": flat, f"{prefix}_offsets": off}


def grads_dict(prefix, g):
    return {f"{prefix}_d_means": g.d_means, f"{prefix}_d_scales": g.d_scales,
            f"{prefix}_d_rotations": g.d_rotations, f"{prefix}_d_thetas": g.d_thetas,
            f"{prefix}_d_colors": g.d_colors, f"{prefix}_d_background": g.d_background,
            f"{prefix}_d_kappas": g.d_kappas, f"{prefix}_visible": g.visible}


def raster_case(name, scene, cam, *, flags=None, d_color=None, d_trans=None, tomo_w=None, extra=None):
    flags = flags or {}
    es = flags.get("early_stop", raster.EARLY_STOP_T)
    ac = flags.get("alpha_cut", raster.ALPHA_CUT)
    out = {"flag_early_stop": np.array(-1.0 if es is None else es), "flag_alpha_cut": np.array(ac)}
    out.update(scene_dict(scene))
    out.update(cam_dict(cam))
    prep = raster.prepare(scene, cam, "analytic", alpha_cut=ac)
    out.update(lists_dict("tiles", prep.grid))
    out.update(depth=prep.depth, valid=prep.valid, mean2d=prep.mean2d, radius=prep.radius,
               kappa=prep.kappa)
    r = raster.render(scene, cam, early_stop=es, alpha_cut=ac, prep=prep)
    out.update(color=r.color, final_transmittance=r.final_transmittance, n_contrib=r.n_contrib)
    if d_color is not None:
        g = grad.backward(scene, cam, d_color, early_stop=es, alpha_cut=ac,
                          d_transmittance=d_trans, prep=prep)
        out["d_color"] = d_color
        if d_trans is not None:
            out["d_transmittance"] = d_trans
        out.update(grads_dict("bwd", g))
    if tomo_w is not None:
        tprep = raster.prepare(scene, cam, "analytic", alpha_cut=tomo.TOMO_BIN_CUT)
        out.update(lists_dict("tomo_tiles", tprep.grid))
        out["tomo_image"] = tomo.tomo_forward(scene, cam, prep=tprep)
        out["tomo_weights"] = tomo_w
        out.update(grads_dict("tomo", tomo.tomo_backward(scene, cam, tomo_w, prep=tprep)))
    if extra:
        out.update(extra)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: n={len(scene)} pairs={len(out['tiles_prims'])}")
    return r


def main():
    # config 1 (BASELINE configs[0])
    cfg = configs.tiny()
    s = cfg.scene
    cam = cfg.cameras[0]
    scene = ref_scene(s.means, s.scales, s.rotations, s.thetas, s.colors)
    rcam = scenes.Camera(width=cam.width, height=cam.height, fx=cam.fx, fy=cam.fy, cx=cam.cx,
                         cy=cam.cy, rotation=cam.rotation, translation=cam.translation)
    target = f32(cfg.target(0, (cam.height, cam.width, 3)))
    r0 = raster.render(scene, rcam)
    loss, d_img = grad.loss_and_grad(r0.color, target, grad.LossSpec("l2"))
    rng = scenes.make_rng(777)
    tomo_w = rng.uniform(0.1, 1.0, (cam.height, cam.width))
    raster_case("tiny", scene, rcam, d_color=d_img, tomo_w=tomo_w,
                extra={"target": target, "l2_loss": np.array(loss)})

    # config 1 with the gradient-check flags (no early stop, no alpha skip)
    flags = dict(early_stop=None, alpha_cut=0.0)
    d_color = rng.uniform(-1.0, 1.0, (cam.height, cam.width, 3))
    d_trans = rng.uniform(-1.0, 1.0, (cam.height, cam.width))
    raster_case("tiny_nostop", scene, rcam, flags=flags, d_color=d_color, d_trans=d_trans)

    # the reference's golden scene file (tests/data/golden_scene.txt) and its PFM
    gs, gcams = sceneio.load_scene("/root/reference/pkg/tests/data/golden_scene.txt")
    gcam = gcams["golden"]
    gscene = ref_scene(gs.means, gs.scales, gs.rotations, gs.thetas, gs.colors, gs.background)
    rr = raster_case("golden_scene", gscene, gcam,
                     d_color=scenes.make_rng(5).uniform(-1, 1, (gcam.height, gcam.width, 3)))
    sceneio.write_pfm(os.path.join(HERE, "golden_render.pfm"), rr.color)

    # ragged image (37x23: partial tiles), off-screen and behind-camera primitives
    rng = scenes.make_rng(12345, 9)
    n = 80
    means = rng.uniform(-1.2, 1.2, (n, 3))
    means[:4, 2] = -4.0                       # behind the camera (z_view < 0)
    means[4:8, 0] = rng.uniform(1.6, 2.2, 4)   # beyond the right edge
    sc = rng.uniform(0.03, 0.3, (n, 3))
    rc = look_at_ref([0.3, -0.2, -3.2], [0, 0, 0], 37, 23, 55.0)
    rscene = ref_scene(means, sc, scenes.random_quaternions(rng, n), rng.uniform(0.05, 0.95, n),
                       rng.uniform(0, 1, (n, 3)), (0.2, 0.3, 0.4))
    raster_case("ragged", rscene, rc, d_color=rng.uniform(-1, 1, (23, 37, 3)),
                d_trans=rng.uniform(-1, 1, (23, 37)), tomo_w=rng.uniform(0.1, 1.0, (23, 37)))

    # early termination buries a far primitive (test_grad.py:190-206)
    fronts = [core.Gaussian3D(mean=np.array([0.0, 0.0, z]), scale=np.full(3, 0.4), theta=1.0,
                              color=np.array([1.0, 0.0, 0.0])) for z in (1.5, 1.6, 1.7)]
    back = core.Gaussian3D(mean=np.array([0.0, 0.0, 30.0]), scale=np.full(3, 0.01), theta=0.8,
                           color=np.array([0.0, 1.0, 0.0]))
    es = raster.Scene.from_gaussians(fronts + [back])
    es = ref_scene(es.means, es.scales, es.rotations, es.thetas, es.colors)
    raster_case("early_stop", es, scenes.zscale_camera(), d_color=np.ones((65, 65, 3)))

    # one-pixel lone primitive: zero theta and d_transmittance paths (test_grad.py:62-121)
    one = scenes.front_camera(width=1, height=1)
    lone0 = ref_scene([[0.0, 0.0, 2.0]], [[0.25] * 3], [[1.0, 0, 0, 0]], [0.0], [[1.0, 1.0, 1.0]])
    d1 = 2.0 * (raster.render(lone0, one, early_stop=None, alpha_cut=0.0).color - 1.0) / 3.0
    raster_case("lone_zero_theta", lone0, one, flags=flags, d_color=d1)
    lone = ref_scene([[0.05, 0.02, 2.0]], [[0.25] * 3], [[1.0, 0, 0, 0]], [0.5], [[1.0, 1.0, 1.0]])
    raster_case("lone_transmittance", lone, one, flags=flags, d_color=np.zeros((1, 1, 3)),
                d_trans=np.ones((1, 1)))

    # empty scene, behind-camera only, tiny centre-tile primitive (test_raster.py:23-42, 122-127)
    e = raster.Scene.empty(background=(0.1, 0.5, 0.9))
    e16 = scenes.front_camera(width=16, height=16)
    out = {"background": e.background}
    out.update(cam_dict(e16))
    np.savez_compressed(os.path.join(HERE, "empty.npz"), **out)
    beh = ref_scene([[0.0, 0.0, -10.0]], [[0.2] * 3], [[1.0, 0, 0, 0]], [0.6], [[1.0, 1.0, 1.0]])
    raster_case("behind", beh, scenes.front_camera(), d_color=np.ones((64, 64, 3)))
    tin = ref_scene([[0.0, 0.0, 0.0]], [[1e-3] * 3], [[1.0, 0, 0, 0]], [0.5], [[1.0, 1.0, 1.0]])
    raster_case("centre_tile", tin, scenes.front_camera(width=48, height=48),
                d_color=np.ones((48, 48, 3)))

    # unit Gaussian tomography centre ray = sqrt(2 pi) (test_tomo.py:35-45)
    tc = scenes.front_camera(width=33, height=33, distance=5.0)
    th = core.theta_for_kappa(1.0, [1.0, 1.0, 1.0])
    unit = ref_scene([[0.0, 0.0, 0.0]], [[1.0] * 3], [[1, 0, 0, 0]], [th], [[1.0] * 3])
    raster_case("tomo_unit", unit, tc, tomo_w=np.ones((33, 33)))

    # a miniature of config 4 (opaque disks, early termination on most pixels)
    mo = configs.opaque(seed=41, n=6000, size=96, n_views=2)
    ms = mo.scene
    mscene = ref_scene(ms.means, ms.scales, ms.rotations, ms.thetas, ms.colors)
    mc = mo.cameras[1]
    mcam = scenes.Camera(width=mc.width, height=mc.height, fx=mc.fx, fy=mc.fy, cx=mc.cx, cy=mc.cy,
                         rotation=mc.rotation, translation=mc.translation)
    raster_case("mini_opaque", mscene, mcam,
                d_color=scenes.make_rng(41).uniform(-1, 1, (96, 96, 3)))


def look_at_ref(pos, target, w, h, fov):
    from volgauss.camera import look_at
    return look_at(pos, target, width=w, height=h, fov_x_deg=fov)


if __name__ == "__main__":
    main()
