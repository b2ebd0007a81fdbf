"""Drop-in mirror of the reference `volgauss.grad` hot path (grad.py):
`SceneGrads`, `ParamGrad`, `backward`, `loss_and_grad` (L2 / L1).

`backward` runs the sm_100a backward blend (front-to-back replay, warp-reduced
per-Gaussian accumulators) and the float64 parameter chain through the C ABI.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib, hostio
from .raster import (ALPHA_CLAMP, ALPHA_CUT, EARLY_STOP_T, TILE_SIZE, DeviceScene, _check_mode,
                     _forward, _stream, prepare)


@dataclass
class ParamGrad:
    index: int
    d_mean: object
    d_scale: object
    d_rotation: object
    d_theta: float
    d_color: object
    d_splat_opacity: float


class SceneGrads:
    """Struct-of-arrays gradients (grad.py:41-69)."""

    FIELDS = ("d_means", "d_scales", "d_rotations", "d_thetas", "d_colors", "d_kappas")

    def __init__(self, n, mode):
        self.mode = mode
        self.d_means = np.zeros((n, 3))
        self.d_scales = np.zeros((n, 3))
        self.d_rotations = np.zeros((n, 4))
        self.d_thetas = np.zeros(n)
        self.d_colors = np.zeros((n, 3))
        self.d_splat_opacities = np.zeros(n)
        self.d_background = np.zeros(3)
        self.d_kappas = np.zeros(n)
        self.visible = np.zeros(n, dtype=bool)
        self.d_sh = None

    def __len__(self):
        return len(self.d_thetas)

    def __getitem__(self, i) -> ParamGrad:
        return ParamGrad(index=i, d_mean=self.d_means[i], d_scale=self.d_scales[i],
                         d_rotation=self.d_rotations[i], d_theta=float(self.d_thetas[i]),
                         d_color=self.d_colors[i], d_splat_opacity=float(self.d_splat_opacities[i]))

    def __iter__(self):
        return (self[i] for i in range(len(self)))

    def position_norms(self):
        if _lib_is_torch(self.d_means):
            return self.d_means.norm(dim=1)
        return np.linalg.norm(self.d_means, axis=1)


def _lib_is_torch(x):
    try:
        import torch
        return isinstance(x, torch.Tensor)
    except ImportError:
        return False


class GradBuffers:
    """One flat float32 device buffer holding every per-Gaussian gradient
    (so a multi-GPU step all-reduces it with a single collective), plus
    d_background and the visibility mask."""

    LAYOUT = (("d_means", 3), ("d_scales", 3), ("d_rotations", 4), ("d_thetas", 1),
              ("d_colors", 3), ("d_kappas", 1), ("d_splat_opacities", 1))

    def __init__(self, n, device, with_sh=False):
        import torch
        self.n = n
        width = sum(w for _, w in self.LAYOUT) + (48 if with_sh else 0)
        self.flat = torch.zeros(max(n, 1) * width + 3, dtype=torch.float32, device=device)
        self.views = {}
        off = 0
        for name, w in self.LAYOUT:
            self.views[name] = self.flat[off:off + n * w].view(n, w) if w > 1 else self.flat[off:off + n]
            off += n * w
        self.views["d_sh"] = self.flat[off:off + n * 48].view(n, 16, 3) if with_sh else None
        off += n * 48 if with_sh else 0
        self.views["d_background"] = self.flat[off:off + 3]
        self.visible = torch.zeros(max(n, 1), dtype=torch.uint8, device=device)

    def struct(self, accumulate=False):
        """vg_grads view; accumulate: False/VG_OVERWRITE, True/VG_ADD or VG_DEFER."""
        g = _lib.VgGrads()
        for name in ("d_means", "d_scales", "d_rotations", "d_thetas", "d_colors", "d_kappas",
                     "d_background", "d_splat_opacities"):
            setattr(g, name, _lib.ptr(self.views[name]).value)
        g.d_sh = _lib.ptr(self.views["d_sh"]).value if self.views["d_sh"] is not None else None
        g.visible = _lib.ptr(self.visible).value
        g.accumulate = int(accumulate) if not isinstance(accumulate, bool) else (1 if accumulate else 0)
        return g

    def zero_(self):
        self.flat.zero_()
        self.visible.zero_()

    def to_scene_grads(self, mode, torch_out):
        n = self.n
        sg = SceneGrads(0, mode)
        if torch_out:
            for name, _ in self.LAYOUT:
                setattr(sg, name, self.views[name])
            sg.d_background = self.views["d_background"]
            sg.visible = self.visible[:n].bool()
            if self.views["d_sh"] is not None:
                sg.d_sh = self.views["d_sh"]
            return sg
        # one download of the whole flat buffer (float64 on the host), fields
        # as views into it
        flat = hostio.to_host(self.flat, np.float64)
        off = 0
        for name, w in self.LAYOUT:
            setattr(sg, name, flat[off:off + n * w].reshape((n, w) if w > 1 else (n,)))
            off += n * w
        if self.views["d_sh"] is not None:
            sg.d_sh = flat[off:off + n * 48].reshape(n, 16, 3)
            off += n * 48
        sg.d_background = flat[off:off + 3]
        sg.visible = hostio.to_host(self.visible[:n], np.uint8).astype(bool)
        return sg


def _finite_or_raise(*arrays):
    """ValueError on a non-finite upstream gradient (grad.py:121-125); device
    tensors are checked with one reduction on the device."""
    import torch
    for a in arrays:
        if a is None:
            continue
        ok = hostio.all_finite(a) if isinstance(a, torch.Tensor) else bool(np.all(np.isfinite(a)))
        if not ok:
            raise ValueError("non-finite upstream pixel gradient")


def _dev_image(a, shape, dev):
    import torch
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=torch.float32).reshape(shape).contiguous()
    return hostio.to_device(np.asarray(a), dev, shape)


def backward(scene, camera, d_color, mode="analytic", *, d_transmittance=None,
             tile_size=TILE_SIZE, sort_by="depth", early_stop=EARLY_STOP_T, alpha_cut=ALPHA_CUT,
             alpha_clamp=ALPHA_CLAMP, threads=None, prep=None, deterministic=True) -> SceneGrads:
    """grad.backward (grad.py:107-213), analytic mode.  Flags must match the
    forward render they differentiate.  Raises ValueError on a non-finite
    upstream gradient (grad.py:121-125).  deterministic=True (the default,
    like the reference's thread-count-invariant result, grad.py:188-204)
    reduces with fixed-order sums instead of float atomics: bitwise
    reproducible; False is the faster training-loop path."""
    _check_mode(mode, sort_by, tile_size)
    torch = _lib._require_cuda()
    dev0 = prep.dscene.device if prep is not None else torch.device("cuda", torch.cuda.current_device())
    H, W = int(camera.height), int(camera.width)
    # the upstream gradient goes to the device first; its finiteness is then
    # one reduction there (a host isfinite pass costs more than the upload)
    dc = _dev_image(d_color, (H, W, 3), dev0)
    dt = _dev_image(d_transmittance, (H, W), dev0) if d_transmittance is not None else None
    _finite_or_raise(dc, dt)
    if prep is None:
        dscene = DeviceScene(scene)
        prep = prepare(dscene, camera, mode, tile_size, sort_by, alpha_cut,
                       _ctx=_lib.scratch_context(dscene.device.index))
    dscene = prep.dscene
    _, color, tfin, _ = _forward(prep, early_stop, alpha_cut, alpha_clamp)
    dev = dscene.device
    bufs = GradBuffers(dscene.n, dev, with_sh=dscene.sh is not None)
    g = bufs.struct(accumulate=False)
    opt = _lib.make_options(TILE_SIZE, early_stop, alpha_cut, alpha_clamp, prep.alpha_cut,
                            deterministic=deterministic, mode=prep.mode)
    _lib.check(_lib.load().vg_set_options(prep.ctx.handle, ctypes.byref(opt)), "vg_set_options")
    _lib.check(_lib.load().vg_render_backward(prep.ctx.handle, _lib.ptr(color), _lib.ptr(tfin),
                                              _lib.ptr(dc), _lib.ptr(dt), ctypes.byref(g),
                                              _stream(dev)), "vg_render_backward")
    return bufs.to_scene_grads(mode, dscene.torch_in)


@dataclass
class LossSpec:
    """Photometric loss (grad.py:308-320): 'l1', 'l2', 'dssim', or 'mixed'
    ((1 - lam) L1 + lam D-SSIM), the reference's default.  The device fuses
    L2 into the backward blend (vg_render_backward_l2); the other kinds are
    formed by loss_and_grad on the rendered image (torch on its device, or
    numpy) and enter through the explicit-gradient backward."""
    kind: str = "mixed"
    lam: float = 0.2

    @classmethod
    def parse(cls, text):
        if ":" in text:
            kind, lam = text.split(":", 1)
            return cls(kind=kind.strip(), lam=float(lam))
        return cls(kind=text.strip())


_KINDS = ("l1", "l2", "dssim", "mixed")


def loss_value(image, target, spec: LossSpec = None):
    """grad.loss_value (grad.py:323-335)."""
    return loss_and_grad(image, target, spec)[0]


def loss_and_grad(image, target, spec: LossSpec = None):
    """Loss value and dL/d(image) (grad.py:338-358) for every loss kind; numpy
    in -> float, numpy float64 gradient; torch in -> float, torch float64
    gradient on the image's device.  D-SSIM = 1 - mean SSIM
    (metrics.ssim_with_grad)."""
    from . import metrics
    spec = spec or LossSpec()
    if spec.kind not in _KINDS:
        raise ValueError(f"unknown loss kind {spec.kind!r}")
    if _lib_is_torch(image):
        import torch
        x = image.to(torch.float64)
        t = target.to(device=x.device, dtype=torch.float64) if _lib_is_torch(target) else \
            torch.as_tensor(np.asarray(target, dtype=float), device=x.device)
        r = x - t
        n = r.numel()
        if spec.kind == "l2":
            return float((r * r).mean()), 2.0 * r / n
        l1, g1 = float(r.abs().mean()), torch.sign(r) / n
    else:
        import torch
        x = np.asarray(image, dtype=float)
        t = np.asarray(target, dtype=float)
        # elementwise work on torch CPU tensors sharing the numpy memory
        # (multi-threaded: a 1080p RGB L2 gradient 40 -> a few ms)
        r_t = torch.from_numpy(np.ascontiguousarray(x)) - torch.from_numpy(np.ascontiguousarray(t))
        n = r_t.numel()
        if spec.kind == "l2":
            flat = r_t.reshape(-1)
            value = float(torch.dot(flat, flat)) / n
            return value, r_t.mul_(2.0 / n).numpy()
        l1, g1 = float(r_t.abs().sum()) / n, torch.sign(r_t).div_(n).numpy()
    if spec.kind == "l1":
        return l1, g1
    sv, ds = metrics.ssim_with_grad(x, t)
    sv = float(sv)
    if spec.kind == "dssim":
        return 1.0 - sv, -ds
    return (1.0 - spec.lam) * l1 + spec.lam * (1.0 - sv), (1.0 - spec.lam) * g1 - spec.lam * ds


# ---------------------------------------------------------------------------
# finite-difference verification (grad.py:361-467)

@dataclass
class FdRecord:
    """grad.FdRecord (grad.py:365-381)."""
    primitive: int
    param: str
    analytic: float
    numeric: float

    @property
    def abs_err(self):
        return abs(self.analytic - self.numeric)

    @property
    def rel_err(self):
        return self.abs_err / max(abs(self.analytic), abs(self.numeric), 1e-8)

    def within(self, tol):
        return self.rel_err <= tol


@dataclass
class FdReport:
    """grad.FdReport (grad.py:384-404)."""
    mode: str
    loss: str
    records: list = field(default_factory=list)

    def fraction_within(self, tol):
        if not self.records:
            return 1.0
        return sum(r.within(tol) for r in self.records) / len(self.records)

    def worst(self):
        failing = [r for r in self.records if not r.within(1e-3)]
        pool = failing or self.records
        return max(pool, key=lambda r: r.rel_err, default=None)

    def rows(self):
        for r in self.records:
            yield (self.mode, r.primitive, r.param, r.analytic, r.numeric, r.abs_err, r.rel_err)


_FD_SLOTS = [("mean", i) for i in range(3)] + [("scale", i) for i in range(3)] + \
    [("rotation", i) for i in range(4)] + [("theta", 0)] + [("color", i) for i in range(3)]
_FD_ARRAYS = {"mean": "means", "scale": "scales", "rotation": "rotations", "theta": "thetas",
              "color": "colors"}


def fd_check(scene, camera, target, loss_spec: LossSpec = None, mode="analytic",
             tile_size=TILE_SIZE, h_min=1e-3, h_rel=1e-2) -> FdReport:
    """grad.fd_check (grad.py:420-467) on the device, analytic mode: the
    device backward against five-point central differences of the device
    render's loss, every scalar parameter of every primitive, with the
    reference's smooth flags (no early stop, no alpha skip).  The renders are
    float32, so the step is h = max(h_min, h_rel |p|) (the reference's float64
    1e-5 / 1e-4 would sit at float32 rounding); the report never raises."""
    from types import SimpleNamespace
    from .raster import render
    if mode != "analytic":
        raise NotImplementedError("fd_check runs the analytic mode on the device")
    loss_spec = loss_spec or LossSpec()
    flags = dict(early_stop=None, alpha_cut=0.0, tile_size=tile_size)
    base = {k: np.array(np.asarray(getattr(scene, k), dtype=np.float64)) for k in _FD_ARRAYS.values()}
    bg = np.asarray(getattr(scene, "background", np.zeros(3)), dtype=np.float64)

    def make(arrs):
        return SimpleNamespace(**arrs, background=bg)

    out = render(make(base), camera, mode, **flags)
    _, d_img = loss_and_grad(out.color, target, loss_spec)
    grads = backward(make(base), camera, d_img, mode, **flags)
    analytic = {"mean": grads.d_means, "scale": grads.d_scales, "rotation": grads.d_rotations,
                "theta": grads.d_thetas, "color": grads.d_colors}

    def loss_of(arrs):
        return loss_value(render(make(arrs), camera, mode, **flags).color, target, loss_spec)

    report = FdReport(mode=mode, loss=loss_spec.kind)
    for prim in range(len(base["means"])):
        for name, comp in _FD_SLOTS:
            key = _FD_ARRAYS[name]
            arr = base[key]
            p0 = float(arr[prim]) if arr.ndim == 1 else float(arr[prim, comp])
            h = max(h_min, h_rel * abs(p0))
            vals = []
            for step in (h, -h, 2.0 * h, -2.0 * h):
                pert = dict(base)
                a = arr.copy()
                if a.ndim == 1:
                    a[prim] += step
                else:
                    a[prim, comp] += step
                pert[key] = a
                vals.append(loss_of(pert))
            numeric = (8.0 * (vals[0] - vals[1]) - (vals[2] - vals[3])) / (12.0 * h)
            an = analytic[name]
            a_val = float(an[prim]) if an.ndim == 1 else float(an[prim, comp])
            label = name if an.ndim == 1 else f"{name}[{comp}]"
            report.records.append(FdRecord(prim, label, a_val, numeric))
    return report
