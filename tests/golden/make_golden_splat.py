"""Generate tests/golden/splat.npz by running the REFERENCE with mode="splat"
(the EWA comparator: raster.py:154-219, 353-361; grad.py:170-177, 262-302)
on the config-1 and ragged scenes of make_golden.py (inputs read back from
tiny.npz / ragged.npz) with seeded splat opacities.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src:. \\
        python tests/golden/make_golden_splat.py
"""

from __future__ import annotations

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from volgauss import grad, raster, scenes  # noqa: E402  (reference)


def main():
    out = {}
    for k, name in enumerate(("tiny", "ragged")):
        d = np.load(os.path.join(HERE, f"{name}.npz"))
        n = len(d["means"])
        opac = np.asarray(scenes.make_rng(41 + k).uniform(0.2, 0.95, n).astype(np.float32), dtype=np.float64)
        scene = raster.Scene(d["means"], d["scales"], d["rotations"], d["thetas"], d["colors"],
                             splat_opacities=opac, background=d["background"])
        w, h = (int(v) for v in d["cam_wh"])
        fx, fy, cx, cy, zn = d["cam_f"]
        cam = scenes.Camera(width=w, height=h, fx=fx, fy=fy, cx=cx, cy=cy, rotation=d["cam_R"],
                            translation=d["cam_t"])
        prep = raster.prepare(scene, cam, mode="splat")
        flat = np.concatenate([np.asarray(t, dtype=np.int64) for t in prep.grid.tiles])
        off = np.concatenate([[0], np.cumsum([len(t) for t in prep.grid.tiles])]).astype(np.int64)
        r = raster.render(scene, cam, mode="splat", prep=prep)
        dc = scenes.make_rng(51 + k).uniform(-1, 1, (h, w, 3))
        g = grad.backward(scene, cam, dc, mode="splat", prep=prep)
        out.update({f"{name}_opac": opac, f"{name}_prims": flat, f"{name}_offsets": off,
                    f"{name}_radius": prep.radius, f"{name}_color": r.color,
                    f"{name}_T": r.final_transmittance, f"{name}_ncontrib": r.n_contrib,
                    f"{name}_dcolor": dc, f"{name}_visible": g.visible})
        for f in ("d_means", "d_scales", "d_rotations", "d_colors", "d_background",
                  "d_splat_opacities", "d_thetas"):
            out[f"{name}_{f}"] = getattr(g, f)
    np.savez_compressed(os.path.join(HERE, "splat.npz"), **out)
    print("splat.npz written")


if __name__ == "__main__":
    main()
