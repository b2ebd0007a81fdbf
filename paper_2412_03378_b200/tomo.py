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


class DensityGrid:
    """tomo.DensityGrid (tomo.py:314-327): a voxel grid of the mixture
    density with its world bounding box (cell-centred samples, C order)."""

    def __init__(self, values, bbox_min, bbox_max):
        self.values = values
        self.bbox_min = np.asarray(bbox_min, dtype=float)
        self.bbox_max = np.asarray(bbox_max, dtype=float)

    def voxel_centers(self):
        axes = [self.bbox_min[i] + (np.arange(n) + 0.5) * ((self.bbox_max[i] - self.bbox_min[i]) / n)
                for i, n in enumerate(self.values.shape)]
        return np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1)


def voxelize(scene, resolution=64, bbox=None):
    """tomo.voxelize (tomo.py:345-389) on the GPU (vg_voxelize): the density
    sum_i kappa_i exp(-q_i/2) at the cell centres, each primitive culled to
    5 of its largest standard deviations.  Returns a DensityGrid (numpy)."""
    import torch
    if bbox is None:
        bbox = (-np.ones(3), np.ones(3))
    bmin = np.asarray(bbox[0], dtype=np.float64).reshape(3)
    bmax = np.asarray(bbox[1], dtype=np.float64).reshape(3)
    shape = (int(resolution),) * 3 if np.isscalar(resolution) else tuple(int(r) for r in resolution)
    dscene = scene if isinstance(scene, DeviceScene) else DeviceScene(scene)
    dev = dscene.device
    out = torch.empty(shape, dtype=torch.float64, device=dev)
    s = dscene.struct()
    lo = (ctypes.c_double * 3)(*bmin)
    hi = (ctypes.c_double * 3)(*bmax)
    sh = (ctypes.c_int32 * 3)(*shape)
    _lib.check(_lib.load().vg_voxelize(ctypes.byref(s), lo, hi, sh, _lib.ptr(out), _stream(dev)),
               "vg_voxelize")
    return DensityGrid(out.cpu().numpy(), bmin, bmax)


def _tomo_init(config, bbox, rng):
    """tomo._tomo_init (tomo.py:428-439): n_init isotropic primitives uniform
    in the box (the same Philox draws as the reference)."""
    from .raster import Scene
    lo, hi = bbox
    n = config.n_init
    means = rng.uniform(0.0, 1.0, (n, 3)) * (hi - lo) + lo
    size = float(np.max(hi - lo))
    return Scene(means=means, scales=np.full((n, 3), config.init_scale_pixels * size / 16.0),
                 rotations=np.tile([1.0, 0.0, 0.0, 0.0], (n, 1)), thetas=np.full(n, config.init_theta),
                 colors=np.full((n, 3), 0.5), splat_opacities=np.full(n, config.init_theta))


def reconstruct(projections, config, *, bbox=None, resolution=64, reference=None, threads=None,
                init_scene=None, callback=None, deterministic=True):
    """tomo.reconstruct (tomo.py:442-519) on the GPU: fit a mixture to
    cone-beam log-intensity projections with the device Trainer (fused Adam,
    GradAccum, densify/prune) -- one projection per iteration in the
    reference's seeded order, targets normalised by their joint maximum, the
    projector and adjoint on the device; returns (DeviceScene, DensityGrid,
    report dict).  L2 is fused into the adjoint; l1 / dssim / mixed (the
    reference's default) are formed by grad.loss_and_grad on the normalised
    projection on the device and pulled back through the explicit-gradient
    adjoint.  deterministic (default): fixed-order gradient sums, so the run
    is bitwise reproducible (densify / prune decisions cannot flip on
    summation order)."""
    import math

    import torch

    from .engine import Engine
    from .optim import DivergenceError, GradAccum, Trainer, _clone_scene, densify_and_prune, scene_extent
    from . import metrics
    if len(projections) < 2:
        raise ValueError("need at least two projections")
    for p in projections:
        if np.any(np.asarray(p.image) < 0):
            raise ValueError("projections must be non-negative log-intensities")
    from .grad import loss_and_grad
    if bbox is None:
        bbox = (-np.ones(3), np.ones(3))
    bbox = (np.asarray(bbox[0], dtype=float), np.asarray(bbox[1], dtype=float))
    rng = np.random.Generator(np.random.Philox(key=config.seed))
    scene = DeviceScene(init_scene if init_scene is not None else _tomo_init(config, bbox, rng))
    dev = scene.device
    cameras = [p.camera for p in projections]
    norm = max(float(np.max([np.max(p.image) for p in projections])), 1e-12)
    targets = [torch.as_tensor(np.asarray(p.image, dtype=np.float64) / norm, dtype=torch.float32).to(dev)
               for p in projections]
    extent = scene_extent(cameras, scene, config.scene_extent_multiplier)
    trainer = Trainer(scene, config, "analytic", extent)
    accum = GradAccum(scene.n, dev.index)
    report = {"losses": [], "primitive_counts": [], "events": [], "diverged": False}
    n_views = len(projections)
    epochs = -(-config.iterations // n_views)
    order = np.concatenate([rng.permutation(n_views) for _ in range(epochs)])[:config.iterations]
    eng = Engine(dev.index, deterministic=deterministic)
    grads = eng.new_grads(scene)
    checkpoint = _clone_scene(scene)
    densify_stop = config.densify_stop_fraction * config.iterations
    for it in range(config.iterations):
        v = int(order[it])
        cam = cameras[v]
        eng.prepare(scene, cam, tomo=True)
        image = eng.tomo_forward()
        # the loss of image / norm against the normalised target; its gradient
        # is chained through the scale (tomo.py:486-494)
        if config.loss.kind == "l2":
            r = image / norm - targets[v]
            n = r.numel()
            value_t = (r.double() ** 2).sum() / n
            d_img = (r * (2.0 / (n * norm))).contiguous()
        else:
            value_t, d = loss_and_grad(image / norm, targets[v], config.loss)
            d_img = (d / norm).to(torch.float32).contiguous()
        eng.tomo_backward(d_img, grads, accumulate=False)
        trainer.step(grads, it, accum=accum, check=False)
        value = float(value_t)                       # the one host sync of the iteration
        if not math.isfinite(value):
            report["diverged"] = True
            scene = checkpoint
            break
        try:
            trainer.check_divergence()
        except DivergenceError:
            report["diverged"] = True
            scene = checkpoint
            break
        report["losses"].append(value)
        report["primitive_counts"].append(scene.n)
        if callback is not None:
            callback(it, scene, value)
        step_no = it + 1
        if config.densify and step_no % config.densify_interval == 0 \
                and config.densify_start <= step_no <= densify_stop:
            scene, events = densify_and_prune(scene, trainer, accum, config, extent, rng, step_no,
                                              "analytic")
            report["events"].extend(events)
            accum = GradAccum(scene.n, dev.index)
            grads = eng.new_grads(scene)
            checkpoint = _clone_scene(scene)
    grid = voxelize(scene, resolution=resolution, bbox=bbox)
    report["final_count"] = scene.n
    if reference is not None:
        ref = reference.values if hasattr(reference, "values") else np.asarray(reference)
        report["psnr_3d"] = metrics.psnr_volume(grid.values, ref)
        report["ssim_3d"] = metrics.ssim_volume(grid.values, ref)
    return scene, grid, report


def attenuation(image):
    """Beer-Lambert intensity exp(-I) (host helper for numpy images)."""
    return np.exp(-np.asarray(image, dtype=float))
