"""Drop-in mirror of the reference tomography projector (tomo.py:34-103):
`tomo_forward` / `tomo_backward`, plus the parallel-beam (orthographic
detector) geometry BASELINE config 5 asks for, which the reference only has
for phantom projections (`tomo._parallel_rays`, tomo.py:272-282).

The line integral of each binned Gaussian is summed per pixel with no
compositing, cut, clamp or early stop (tomo.py:43-47); bins use the generous
TOMO_BIN_CUT = 1e-12 radii (tomo.py:26-28).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .grad import GradBuffers, _dev_image, _finite_or_raise
from .raster import TILE_SIZE, DeviceScene, _out, _stream, prepare

TOMO_BIN_CUT = 1e-12   # tomo.py:28


def tomo_prepare(scene, camera, *, tile_size=TILE_SIZE, parallel=False, extent=1.6, _ctx=None):
    """raster.prepare(..., alpha_cut=TOMO_BIN_CUT) for either ray model."""
    return prepare(scene, camera, "analytic", tile_size, "depth", TOMO_BIN_CUT, _ctx=_ctx,
                   _kind="tomo", _bin_cut=TOMO_BIN_CUT,
                   _projection=_lib.VG_PARALLEL if parallel else _lib.VG_PINHOLE,
                   _extent=extent if parallel else 0.0)


def _tomo_prep(scene, camera, tile_size, prep, parallel, extent):
    if prep is not None:
        return prep
    dscene = DeviceScene(scene)
    return tomo_prepare(dscene, camera, tile_size=tile_size, parallel=parallel, extent=extent,
                        _ctx=_lib.scratch_context(dscene.device.index))


def tomo_forward(scene, camera, *, tile_size=TILE_SIZE, threads=None, prep=None, parallel=False,
                 extent=1.6, intensity=False):
    """Line-integral image I(p) = sum_j kappa_j sqrt(2 pi) beta_j peak_j
    (tomo.py:34-57).  With intensity=True also returns exp(-I)."""
    import torch
    prep = _tomo_prep(scene, camera, tile_size, prep, parallel, extent)
    H, W = int(camera.height), int(camera.width)
    dev = prep.dscene.device
    img = torch.empty((H, W), dtype=torch.float32, device=dev)
    inten = torch.empty((H, W), dtype=torch.float32, device=dev) if intensity else None
    _lib.check(_lib.load().vg_tomo_forward(prep.ctx.handle, _lib.ptr(img), _lib.ptr(inten),
                                           _stream(dev)), "vg_tomo_forward")
    ti = prep.dscene.torch_in
    if intensity:
        return _out(img, ti), _out(inten, ti)
    return _out(img, ti)


def tomo_backward(scene, camera, d_image, *, tile_size=TILE_SIZE, threads=None, prep=None,
                  parallel=False, extent=1.6, deterministic=True):
    """Gradients of sum(d_image * tomo_forward) for every scene parameter
    (tomo.py:60-103); colour gradients are zero.  deterministic=True (the
    default, like the reference's fixed tile-order reduction) sums with
    fixed-order reductions: bitwise reproducible."""
    _finite_or_raise(d_image)
    prep = _tomo_prep(scene, camera, tile_size, prep, parallel, extent)
    H, W = int(camera.height), int(camera.width)
    dev = prep.dscene.device
    di = _dev_image(d_image, (H, W), dev)
    bufs = GradBuffers(prep.dscene.n, dev)
    g = bufs.struct(accumulate=False)
    opt = _lib.make_options(TILE_SIZE, None, TOMO_BIN_CUT, 0.99, TOMO_BIN_CUT,
                            deterministic=deterministic)
    _lib.check(_lib.load().vg_set_options(prep.ctx.handle, ctypes.byref(opt)), "vg_set_options")
    _lib.check(_lib.load().vg_tomo_backward(prep.ctx.handle, _lib.ptr(di), ctypes.byref(g),
                                            _stream(dev)), "vg_tomo_backward")
    return bufs.to_scene_grads("analytic", prep.dscene.torch_in)


def attenuation(image):
    """Beer-Lambert intensity exp(-I) (host helper for numpy images)."""
    return np.exp(-np.asarray(image, dtype=float))
