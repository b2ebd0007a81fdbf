"""GPU training-step caller of the rasterizer: the
reference's `volgauss.optim` hot loop -- Adam over the parameter groups with
the bounded-density constraint projections (`Trainer.step`, optim.py:119-175),
the positional-gradient accumulator (`GradAccum`, optim.py:194-206), the
density-aware `densify_and_prune` (optim.py:218-317) and the image-fitting
loop `fit_image` (optim.py:343-416) -- with the scene, gradients and Adam
moments resident in HBM.

`Trainer.step` is one fused sm_100a kernel (vg_adam_step: Adam on all five
groups + GradAccum.update + projections).  `densify_and_prune` decides on
the device (vg_densify_plan), draws the split offsets on the host with the
reference's generator calls (rng.standard_normal((2, 3)) per split parent,
in index order, so the children are the reference's), and compacts on the
device (vg_densify_apply); the DensifyEvent log is assembled on the host from
the decisions.  Only the analytic mode exists here (the splat comparator is
outside the hot path).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .grad import GradBuffers, LossSpec
from .raster import DeviceScene

SCALE_FLOOR = 1e-7
THETA_CEILING = 0.99
GROUPS = ("position", "scale", "rotation", "color", "density")


class DivergenceError(RuntimeError):
    """Raised when an optimizer update goes non-finite (optim.py:19-20)."""


@dataclass
class TrainConfig:
    """optim.TrainConfig (optim.py:24-53), same fields and defaults."""
    iterations: int = 1000
    loss: LossSpec = field(default_factory=LossSpec)
    lr_position: float = 1.6e-4
    lr_position_final: float = 1e-5
    lr_theta: float = 0.03
    lr_color: float = 0.003
    lr_scale: float = 5e-3
    lr_rotation: float = 1e-3
    densify: bool = False
    densify_interval: int = 200
    densify_start: int = 200
    densify_stop_fraction: float = 0.7
    split_grad_threshold: float = 1e-8
    clone_grad_threshold: float = 5e-5
    prune_theta_min: float = 0.005
    prune_scale_fraction: float = 0.01
    scene_extent_multiplier: float = 1.0
    high_kappa_split_fraction: float = 0.9
    max_primitives: int = 20000
    seed: int = 0
    n_init: int = 200
    init_theta: float = 0.1
    init_scale_pixels: float = 1.0

    def __post_init__(self):
        if isinstance(self.loss, str):
            self.loss = LossSpec.parse(self.loss)


@dataclass
class DensifyEvent:
    """optim.DensifyEvent (optim.py:56-71)."""
    iteration: int
    kind: str
    parent: int
    parent_kappa: float = 0.0
    parent_theta: float = 0.0
    child_thetas: tuple = ()
    child_scales: tuple = ()
    child_kappas: tuple = ()
    clamped: bool = False
    reason: str = ""
    theta: float = 0.0
    max_scale: float = 0.0
    theta_bound: float = 0.0
    scale_bound: float = 0.0


@dataclass
class FitReport:
    """optim.FitReport (optim.py:74-81)."""
    mode: str
    losses: list = field(default_factory=list)
    primitive_counts: list = field(default_factory=list)
    events: list = field(default_factory=list)
    final_metrics: list = field(default_factory=list)
    diverged: bool = False
    iterations_run: int = 0


def _softplus_inv(y):
    y = np.asarray(y, dtype=np.float64)
    return y + np.log1p(-np.exp(-10.0 * y)) / 10.0


class GradAccum:
    """optim.GradAccum on the device: windowed positional-gradient norms of
    the visible primitives.  Trainer.step(accum=...) updates it inside the
    fused Adam kernel; update() is the standalone form."""

    def __init__(self, n, device=None):
        torch = _lib._require_cuda()
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.norm_sum = torch.zeros(max(n, 0), dtype=torch.float32, device=dev)
        self.count = torch.zeros(max(n, 0), dtype=torch.float32, device=dev)

    def update(self, grads):
        d = _grad_tensor(grads, "d_means")
        vis = _grad_tensor(grads, "visible").bool()
        self.norm_sum += d.norm(dim=1) * vis
        self.count += vis.float()

    def averages(self):
        return self.norm_sum / self.count.clamp(min=1.0)


def _grad_tensor(grads, name):
    if isinstance(grads, GradBuffers):
        return grads.visible[:grads.n] if name == "visible" else grads.views[name]
    return getattr(grads, name)


class Trainer:
    """optim.Trainer (optim.py:119-175) with the state on the device: the
    DeviceScene's tensors are updated in place, raw (pre-softplus) colours
    and the 14+14 Adam moments per primitive live in HBM."""

    def __init__(self, scene: DeviceScene, config: TrainConfig, mode="analytic", extent=1.0):
        if mode != "analytic":
            raise NotImplementedError("only the analytic mode is on the device")
        torch = _lib._require_cuda()
        self.torch = torch
        self.scene = scene
        self.config = config
        self.mode = mode
        self.extent = float(extent)
        self.t = 0
        n = scene.n
        dev = scene.device
        cols = scene.colors.double().clamp(min=1e-6)
        self.color_raw = (cols + torch.log1p(-torch.exp(-10.0 * cols)) / 10.0).float().contiguous()
        self.moments = torch.zeros((max(n, 1), 28), dtype=torch.float32, device=dev)
        self._bad = torch.empty(5, dtype=torch.int32, device=dev)
        self.lib = _lib.load()

    def lr_position_at(self, iteration):
        """optim.py:140-144."""
        c = self.config
        frac = iteration / max(c.iterations - 1, 1)
        return c.lr_position * (c.lr_position_final / c.lr_position) ** frac * self.extent

    def state(self, accum=None):
        s = self.scene
        st = _lib.VgTrainState()
        st.means, st.scales = _lib.ptr(s.means).value, _lib.ptr(s.scales).value
        st.rotations, st.thetas = _lib.ptr(s.rotations).value, _lib.ptr(s.thetas).value
        st.colors, st.color_raw = _lib.ptr(s.colors).value, _lib.ptr(self.color_raw).value
        st.moments = _lib.ptr(self.moments).value
        if accum is not None:
            st.accum_norm, st.accum_count = _lib.ptr(accum.norm_sum).value, _lib.ptr(accum.count).value
        st.n = s.n
        return st

    def step(self, grads, iteration, accum=None, check=True):
        """One Adam step on every group (optim.py:146-175).  grads: a
        GradBuffers (or SceneGrads with device tensors).  With check=True the
        divergence flag is read back (host sync) and DivergenceError raised;
        check=False defers that to check_divergence()."""
        c = self.config
        self.t += 1
        hp = _lib.VgAdamHparams()
        for k, v in enumerate((self.lr_position_at(iteration), c.lr_scale, c.lr_rotation, c.lr_color,
                               c.lr_theta)):
            hp.lr[k] = v
        hp.beta1, hp.beta2, hp.eps, hp.t = 0.9, 0.999, 1e-8, self.t
        g = grads.struct(False) if isinstance(grads, GradBuffers) else _scene_grads_struct(grads)
        st = self.state(accum)
        _lib.check(self.lib.vg_adam_step(ctypes.byref(st), ctypes.byref(g), ctypes.byref(hp),
                                         _lib.ptr(self._bad), _stream(self.scene.device)),
                   "vg_adam_step")
        if check:
            self.check_divergence()

    def check_divergence(self):
        bad = self._bad.cpu().numpy()
        for name, b in zip(GROUPS, bad):
            if b != np.iinfo(np.int32).max:
                raise DivergenceError(f"non-finite {name} update for primitive {int(b)}")


def _stream(dev):
    import torch
    return torch.cuda.current_stream(dev).cuda_stream


def _scene_grads_struct(sg):
    g = _lib.VgGrads()
    for name in ("d_means", "d_scales", "d_rotations", "d_thetas", "d_colors"):
        setattr(g, name, _lib.ptr(getattr(sg, name)).value)
    vis = getattr(sg, "visible", None)
    g.visible = _lib.ptr(vis.to(dtype=__import__("torch").uint8)).value if vis is not None else None
    return g


def scene_extent(cameras, scene, multiplier=1.0):
    """optim.scene_extent (optim.py:178-191)."""
    centers = np.array([c.center for c in cameras])
    r = float(np.linalg.norm(centers - centers.mean(axis=0), axis=1).max())
    if r < 1e-9:
        if scene.n:
            m = scene.means.double()
            diag = float((m.max(dim=0).values - m.min(dim=0).values).norm())
        else:
            diag = 0.0
        r = max(diag, 1.0)
    return multiplier * r


def densify_and_prune(scene: DeviceScene, trainer: Trainer, accum: GradAccum, config: TrainConfig,
                      extent, rng, iteration, mode="analytic", events=True):
    """optim.densify_and_prune (optim.py:218-317), analytic mode.  Returns the
    new DeviceScene (trainer.scene, trainer moments and raw colours are
    replaced) and the list of DensifyEvents."""
    torch = trainer.torch
    lib = trainer.lib
    n = scene.n
    if n == 0:
        return scene, []
    dev = scene.device
    st = _stream(dev)
    args = _lib.VgDensifyArgs()
    args.n = n
    args.means, args.scales = _lib.ptr(scene.means).value, _lib.ptr(scene.scales).value
    args.rotations, args.thetas = _lib.ptr(scene.rotations).value, _lib.ptr(scene.thetas).value
    args.colors, args.color_raw = _lib.ptr(scene.colors).value, _lib.ptr(trainer.color_raw).value
    args.moments = _lib.ptr(trainer.moments).value
    args.accum_norm, args.accum_count = _lib.ptr(accum.norm_sum).value, _lib.ptr(accum.count).value
    args.extent = float(extent)
    args.split_grad_threshold = config.split_grad_threshold
    args.clone_grad_threshold = config.clone_grad_threshold
    args.prune_theta_min = config.prune_theta_min
    args.prune_scale_fraction = config.prune_scale_fraction
    args.high_kappa_split_fraction = config.high_kappa_split_fraction
    args.max_primitives = int(config.max_primitives)
    scratch = torch.empty(int(lib.vg_densify_scratch_bytes(n)), dtype=torch.uint8, device=dev)
    counts = torch.empty(4, dtype=torch.int32, device=dev)
    _lib.check(lib.vg_densify_plan(ctypes.byref(args), _lib.ptr(scratch), _lib.ptr(counts), st),
               "vg_densify_plan")
    c = counts.cpu().numpy().astype(np.uint32)       # {grown, kept, splits, clones}
    kept, n_split, n_clone = int(c[1]), int(c[2]), int(c[3])
    # the reference draws rng.standard_normal((2, 3)) once per split parent, in index order
    xi = rng.standard_normal((n_split, 2, 3)) if n_split else np.zeros((0, 2, 3))
    xi_dev = torch.from_numpy(np.ascontiguousarray(xi)).to(dev)
    n_out = kept + 2 * (n_split + n_clone)
    new = _empty_scene_like(scene, n_out)
    color_raw = torch.empty((max(n_out, 1), 3), dtype=torch.float32, device=dev)
    moments = torch.empty((max(n_out, 1), 28), dtype=torch.float32, device=dev)
    out = _lib.VgTrainState()
    out.means, out.scales = _lib.ptr(new.means).value, _lib.ptr(new.scales).value
    out.rotations, out.thetas = _lib.ptr(new.rotations).value, _lib.ptr(new.thetas).value
    out.colors, out.color_raw = _lib.ptr(new.colors).value, _lib.ptr(color_raw).value
    out.moments = _lib.ptr(moments).value
    out.n = n_out
    hc = (ctypes.c_uint32 * 4)(*[int(v) for v in c])
    _lib.check(lib.vg_densify_apply(ctypes.byref(args), _lib.ptr(scratch), hc, _lib.ptr(xi_dev),
                                    ctypes.byref(out), st), "vg_densify_apply")
    ev = _events(scene, scratch, n, accum, config, extent, iteration, lib, new, kept) if events else []
    trainer.scene = new
    trainer.color_raw = color_raw[:n_out] if n_out else color_raw[:0]
    trainer.moments = moments
    return new, ev


def _empty_scene_like(scene, n):
    from types import SimpleNamespace
    import torch
    dev = scene.device
    z = SimpleNamespace(means=torch.empty((n, 3), device=dev), scales=torch.empty((n, 3), device=dev),
                        rotations=torch.empty((n, 4), device=dev), thetas=torch.empty((n,), device=dev),
                        colors=torch.empty((n, 3), device=dev), background=scene.background)
    return DeviceScene(z, dev.index)


def _events(scene, scratch, n, accum, config, extent, iteration, lib, new, kept):
    """The DensifyEvent log (optim.py:245-300) from the device decisions."""
    flags = scratch[:n].cpu().numpy()                 # first n bytes: decision flags
    split = np.flatnonzero(flags & 1)
    clone = np.flatnonzero(flags & 2)
    prune = np.flatnonzero(flags & 4)
    thetas = scene.thetas.double().cpu().numpy()
    scales = np.maximum(scene.scales.double().cpu().numpy(), SCALE_FLOOR)
    raw_scales = scene.scales.double().cpu().numpy()
    inv_mean = np.mean(1.0 / scales, axis=1)
    kappas = -np.log1p(-THETA_CEILING * thetas) * inv_mean
    ceilings = -np.log1p(-THETA_CEILING) * inv_mean
    avg = (accum.averages().double().cpu().numpy())
    big = raw_scales.max(axis=1) > config.prune_scale_fraction * extent
    child_th = new.thetas.double().cpu().numpy()
    child_sc = new.scales.double().cpu().numpy()
    events = []

    def child_kappa(th, cs):
        cs = np.maximum(cs, SCALE_FLOOR)
        return float(-np.log1p(-THETA_CEILING * th) * np.mean(1.0 / cs))

    def emit(parent, slot, kind):
        ths = (float(child_th[slot]), float(child_th[slot + 1]))
        css = (tuple(child_sc[slot]), tuple(child_sc[slot + 1]))
        target = 0.5 * kappas[parent]
        clamped = any(target > -np.log1p(-THETA_CEILING) * np.mean(1.0 / np.maximum(np.array(cs), SCALE_FLOOR))
                      * (1.0 + 1e-12) for cs in css)
        high = kappas[parent] > config.high_kappa_split_fraction * ceilings[parent]
        grad_rule = avg[parent] > config.split_grad_threshold and big[parent]
        events.append(DensifyEvent(
            iteration=iteration, kind=kind, parent=int(parent), parent_kappa=float(kappas[parent]),
            parent_theta=float(thetas[parent]), child_thetas=ths, child_scales=css,
            child_kappas=tuple(child_kappa(t, np.array(cs)) for t, cs in zip(ths, css)),
            clamped=bool(clamped),
            reason="high_kappa" if kind == "split" and high and not grad_rule else "gradient"))

    for r, p in enumerate(split):
        emit(p, kept + 2 * r, "split")
    for r, p in enumerate(clone):
        emit(p, kept + 2 * len(split) + 2 * r, "clone")
    max_scale = raw_scales.max(axis=1)
    for i in prune:
        events.append(DensifyEvent(
            iteration=iteration, kind="prune", parent=int(i), theta=float(thetas[i]),
            max_scale=float(max_scale[i]), theta_bound=config.prune_theta_min,
            scale_bound=config.prune_scale_fraction * extent,
            reason="theta" if thetas[i] < config.prune_theta_min else "scale"))
    return events


def fit_image(targets, cameras, config: TrainConfig, mode="analytic", init_scene=None,
              threads=None, background=(0, 0, 0), callback=None, deterministic=True):
    """optim.fit_image (optim.py:343-416) on the GPU, analytic mode: one
    camera per iteration in the reference's seeded order, the loss and
    backward (L2 fused into the backward blend; l1 / dssim / mixed formed by
    grad.loss_and_grad on the rendered image on the device, then the
    explicit-gradient backward), the fused Adam step, periodic
    densify/prune; the loss is read back once per iteration (the reference's
    finite check) and the scene restored from the last checkpoint on
    divergence.  deterministic (default): fixed-order gradient sums, so a run
    is bitwise reproducible like the reference's (its densify decisions
    cannot flip on summation order).  Returns (DeviceScene, FitReport);
    final_metrics holds the per-view mse/psnr."""
    import torch
    from .engine import Engine
    from .grad import loss_and_grad
    if mode != "analytic":
        raise NotImplementedError("only the analytic mode is on the device")
    fused = config.loss.kind == "l2"
    if not isinstance(targets, (list, tuple)):
        targets = [targets]
        cameras = [cameras] if not isinstance(cameras, (list, tuple)) else cameras
    if len(targets) != len(cameras) or not cameras:
        raise ValueError("need one camera per target image")
    if init_scene is None:
        raise NotImplementedError("pass init_scene (the seeded default init is outside the hot path)")
    rng = np.random.Generator(np.random.Philox(key=config.seed))
    scene = DeviceScene(init_scene)
    dev = scene.device
    tgts = [torch.as_tensor(np.asarray(t, dtype=np.float32)).to(dev) for t in targets]
    extent = scene_extent(cameras, scene, config.scene_extent_multiplier)
    trainer = Trainer(scene, config, mode, extent)
    accum = GradAccum(scene.n, dev.index)
    report = FitReport(mode=mode)
    if len(cameras) > 1:
        epochs = -(-config.iterations // len(cameras))
        order = np.concatenate([rng.permutation(len(cameras)) for _ in range(epochs)])[:config.iterations]
    else:
        order = np.zeros(config.iterations, dtype=int)
    eng = Engine(dev.index, deterministic=deterministic)
    grads = eng.new_grads(scene)
    loss = torch.zeros((), dtype=torch.float64, device=dev)
    checkpoint = _clone_scene(scene)
    densify_stop = config.densify_stop_fraction * config.iterations
    for it in range(config.iterations):
        cam = cameras[order[it]]
        H, W = int(cam.height), int(cam.width)
        eng.prepare(scene, cam)
        color, tfin, _ = eng.forward(counts=False)
        if fused:
            loss.zero_()
            eng.backward_l2(color, tfin, tgts[order[it]], grads, accumulate=False, loss=loss)
        else:
            value, d_img = loss_and_grad(color, tgts[order[it]], config.loss)
            eng.backward(color, tfin, d_img.to(torch.float32).contiguous(), grads, accumulate=False)
        trainer.step(grads, it, accum=accum, check=False)
        if fused:
            value = float(loss) / (H * W * 3)      # the one sync of the iteration
        if not math.isfinite(value):
            report.diverged = True
            scene = checkpoint
            break
        try:
            trainer.check_divergence()
        except DivergenceError:
            report.diverged = True
            scene = checkpoint
            break
        report.losses.append(value)
        report.primitive_counts.append(scene.n)
        if callback is not None:
            callback(it, scene, value)
        step_no = it + 1
        if config.densify and step_no % config.densify_interval == 0 \
                and config.densify_start <= step_no <= densify_stop:
            scene, events = densify_and_prune(scene, trainer, accum, config, extent, rng, step_no, mode)
            report.events.extend(events)
            accum = GradAccum(scene.n, dev.index)
            grads = eng.new_grads(scene)
            checkpoint = _clone_scene(scene)
        report.iterations_run = step_no
    for cam, t in zip(cameras, tgts):
        eng.prepare(scene, cam)
        color, _, _ = eng.forward(counts=False)
        mse = float(((color.double() - t.double()) ** 2).mean())
        psnr = float(10.0 * math.log10(1.0 / max(float(((color.clamp(0, 1).double() - t.clamp(0, 1).double()) ** 2).mean()), 1e-30)))
        report.final_metrics.append({"mse": mse, "psnr": psnr})
    return scene, report


def _clone_scene(s):
    from types import SimpleNamespace
    z = SimpleNamespace(means=s.means.clone(), scales=s.scales.clone(), rotations=s.rotations.clone(),
                        thetas=s.thetas.clone(), colors=s.colors.clone(), background=s.background)
    return DeviceScene(z, s.device.index)
