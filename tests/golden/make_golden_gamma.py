"""Generate tests/golden/gamma.npz by running the REFERENCE with
sort_by="gamma" (raster.prepare / _resort_by_gamma, raster.py:291-312):
per-tile lists re-sorted by gamma along each tile's central ray, plus the
image and gradients rendered in that order, for the config-1 scene and the
ragged scene of make_golden.py (inputs read back from tiny.npz / ragged.npz).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src:. \\
        python tests/golden/make_golden_gamma.py
"""

from __future__ import annotations

import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from volgauss import grad, raster, scenes  # noqa: E402  (reference)


def main():
    out = {}
    for name in ("tiny", "ragged"):
        d = np.load(os.path.join(HERE, f"{name}.npz"))
        scene = raster.Scene(d["means"], d["scales"], d["rotations"], d["thetas"], d["colors"],
                             background=d["background"])
        w, h = (int(v) for v in d["cam_wh"])
        fx, fy, cx, cy, zn = d["cam_f"]
        cam = scenes.Camera(width=w, height=h, fx=fx, fy=fy, cx=cx, cy=cy, rotation=d["cam_R"],
                            translation=d["cam_t"])
        prep = raster.prepare(scene, cam, sort_by="gamma")
        flat = np.concatenate([np.asarray(t, dtype=np.int64) for t in prep.grid.tiles])
        off = np.concatenate([[0], np.cumsum([len(t) for t in prep.grid.tiles])]).astype(np.int64)
        r = raster.render(scene, cam, sort_by="gamma", prep=prep)
        dc = scenes.make_rng(31).uniform(-1, 1, (h, w, 3))
        g = grad.backward(scene, cam, dc, sort_by="gamma", prep=prep)
        out.update({f"{name}_prims": flat, f"{name}_offsets": off, f"{name}_color": r.color,
                    f"{name}_T": r.final_transmittance, f"{name}_ncontrib": r.n_contrib,
                    f"{name}_dcolor": dc})
        for k in ("d_means", "d_scales", "d_rotations", "d_thetas", "d_colors", "d_background"):
            out[f"{name}_{k}"] = getattr(g, k)
    np.savez_compressed(os.path.join(HERE, "gamma.npz"), **out)
    print("gamma.npz written")


if __name__ == "__main__":
    main()
