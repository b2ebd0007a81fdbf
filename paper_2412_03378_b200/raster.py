"""Drop-in mirror of the reference `volgauss.raster` hot path (raster.py).

Same names, signatures, flag defaults and error behaviour as the reference:
`Scene`, `TileGrid`, `RenderOutput`, `prepare`, `bin_tiles`, `render`,
`composite_pixel`.  All compute runs in the sm_100a library through the C ABI
(include/volgauss_b200.h); there is no CPU fallback.

Array types: a scene whose arrays are numpy (e.g. a reference
`volgauss.Scene`) gets numpy float64 outputs, exactly like the reference; a
scene whose arrays are CUDA torch tensors gets CUDA torch outputs with no host
round trip.  sort_by='gamma' re-sorts every tile list by gamma along the
tile's central ray on the device (raster.py:299-312); mode='splat' runs the
EWA comparator (raster.py:353-361) on the same tile pipeline.  tile_size != 16
raises NotImplementedError; unknown modes / sort keys raise ValueError as in
raster.py:268-269, 293-294.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, hostio

TILE_SIZE = 16            # raster.py:26
ALPHA_CLAMP = 0.99        # raster.py:27
ALPHA_CUT = 1.0 / 255.0   # raster.py:28
EARLY_STOP_T = 1e-4       # raster.py:29
COV2D_DILATION = 0.3      # raster.py:30
BASE_RADIUS_SIGMA = 3.0   # raster.py:35


class Scene:
    """Struct-of-arrays Gaussian mixture plus a background colour
    (raster.py:38-97).  Arrays may be numpy or CUDA torch tensors.  `sh`
    optionally holds (N, 16, 3) degree-3 SH coefficients whose DC band is the
    view-independent RGB (BASELINE config 3; no reference counterpart)."""

    def __init__(self, means, scales, rotations, thetas, colors, splat_opacities=None,
                 background=(0.0, 0.0, 0.0), sh=None):
        if _is_torch(means):
            n = means.shape[0]
            self.means, self.scales, self.rotations = means, scales, rotations
            self.thetas, self.colors = thetas, colors
            self.splat_opacities = splat_opacities
        else:
            self.means = np.atleast_2d(np.asarray(means, dtype=float))
            n = len(self.means)
            self.scales = np.broadcast_to(np.asarray(scales, dtype=float), (n, 3)).copy()
            self.rotations = np.broadcast_to(np.asarray(rotations, dtype=float), (n, 4)).copy()
            self.thetas = np.broadcast_to(np.asarray(thetas, dtype=float), (n,)).copy()
            self.colors = np.broadcast_to(np.asarray(colors, dtype=float), (n, 3)).copy()
            if splat_opacities is None:
                splat_opacities = np.full(n, 0.5)
            self.splat_opacities = np.broadcast_to(np.asarray(splat_opacities, dtype=float), (n,)).copy()
        self.background = np.asarray(background, dtype=float)
        self.sh = sh

    @classmethod
    def empty(cls, background=(0.0, 0.0, 0.0)):
        return cls(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0),
                   np.zeros((0, 3)), np.zeros(0), background)

    @classmethod
    def from_gaussians(cls, gaussians, background=(0.0, 0.0, 0.0)):
        gs = list(gaussians)
        if not gs:
            return cls.empty(background)
        return cls([g.mean for g in gs], [g.scale for g in gs], [g.rotation for g in gs],
                   [g.theta for g in gs], [g.color for g in gs],
                   [getattr(g, "splat_opacity", 0.5) for g in gs], background)

    def __len__(self):
        return int(self.means.shape[0])

    def gaussian(self, i):
        """Primitive i as a camera.Gaussian3D (raster.py:85-89), host copies."""
        from .camera import Gaussian3D

        def host(a):
            return a.detach().cpu().numpy().astype(np.float64) if _is_torch(a) else np.asarray(a, dtype=float)
        op = self.splat_opacities
        return Gaussian3D(mean=host(self.means[i]).copy(), scale=host(self.scales[i]).copy(),
                          rotation=host(self.rotations[i]).copy(), theta=float(host(self.thetas[i])),
                          color=host(self.colors[i]).copy(),
                          splat_opacity=float(host(op[i])) if op is not None else 0.5)

    def copy(self):
        if _is_torch(self.means):
            return Scene(self.means.clone(), self.scales.clone(), self.rotations.clone(),
                         self.thetas.clone(), self.colors.clone(), None, self.background.copy(),
                         None if self.sh is None else self.sh.clone())
        return Scene(self.means.copy(), self.scales.copy(), self.rotations.copy(),
                     self.thetas.copy(), self.colors.copy(), self.splat_opacities.copy(),
                     self.background.copy(), None if self.sh is None else np.array(self.sh))

    def kappas(self):
        """core.density_kappa (core.py:132-143)."""
        if _is_torch(self.thetas):
            import torch
            s = self.scales.double().clamp_min(1e-7)
            return -torch.log1p(-0.99 * self.thetas.double()) * (1.0 / s).mean(dim=1)
        s = np.maximum(self.scales, 1e-7)
        return -np.log1p(-0.99 * self.thetas) * np.mean(1.0 / s, axis=-1)


@dataclass
class TileGrid:
    """Per-tile primitive lists, each sorted by view depth (raster.py:100-112)."""
    tile_size: int
    n_tiles_x: int
    n_tiles_y: int
    tiles: list
    sort_keys: np.ndarray

    def entries(self, tx, ty):
        ids = self.tiles[ty * self.n_tiles_x + tx]
        return [(int(i), float(self.sort_keys[i])) for i in ids]


@dataclass
class RenderOutput:
    color: object               # (H, W, 3)
    final_transmittance: object  # (H, W)
    n_contrib: object           # (H, W) int32
    mode: str


def _is_torch(x):
    try:
        import torch
        return isinstance(x, torch.Tensor)
    except ImportError:
        return False


def _check_mode(mode, sort_by, tile_size):
    if mode not in ("analytic", "splat"):
        raise ValueError(f"unknown mode {mode!r}")
    if sort_by not in ("depth", "gamma"):
        raise ValueError(f"unknown sort key {sort_by!r}")
    if int(tile_size) != TILE_SIZE:
        raise NotImplementedError("only tile_size=16 is supported")


class DeviceScene:
    """float32 CUDA copies (or zero-copy views) of a scene's arrays."""

    def __init__(self, scene, device=None):
        torch = _lib._require_cuda()
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.device = dev
        self.torch_in = _is_torch(scene.means)
        n = int(scene.means.shape[0]) if hasattr(scene.means, "shape") else len(scene.means)
        self.n = n

        def conv(a, shape):
            if _is_torch(a):
                t = a.to(device=dev, dtype=torch.float32)
            else:
                # pinned float64 staging + a cast on the device (hostio)
                t = hostio.to_device(np.asarray(a), dev, shape)
            return t.reshape(shape).contiguous()

        self.means = conv(scene.means, (n, 3))
        self.scales = conv(scene.scales, (n, 3))
        self.rotations = conv(scene.rotations, (n, 4))
        self.thetas = conv(scene.thetas, (n,))
        colors = getattr(scene, "colors", None)
        self.colors = conv(colors, (n, 3)) if colors is not None else None
        sh = getattr(scene, "sh", None)
        self.sh = conv(sh, (n, 16, 3)) if sh is not None else None
        op = getattr(scene, "splat_opacities", None)
        # raster.Scene's default splat opacity is 0.5 (raster.py:49-50)
        self.splat_opacities = conv(op, (n,)) if op is not None else \
            torch.full((n,), 0.5, dtype=torch.float32, device=dev)
        bg = scene.background
        self.background = np.asarray(bg.detach().cpu().numpy() if _is_torch(bg) else bg,
                                     dtype=np.float64).reshape(3)

    def struct(self):
        s = _lib.VgScene()
        s.means = _lib.ptr(self.means).value
        s.scales = _lib.ptr(self.scales).value
        s.rotations = _lib.ptr(self.rotations).value
        s.thetas = _lib.ptr(self.thetas).value
        s.colors = _lib.ptr(self.colors).value if self.colors is not None else None
        s.sh = _lib.ptr(self.sh).value if self.sh is not None else None
        s.splat_opacities = _lib.ptr(self.splat_opacities).value
        s.n = self.n
        for i in range(3):
            s.background[i] = float(self.background[i])
        return s


class Prep:
    """Device-side analogue of the reference `_Prep` (raster.py:123-145): the
    context that holds the blend records, sorted tile lists and (after a
    render) the per-pixel forward state that backward reuses."""

    def __init__(self, ctx, dscene, camera, mode, tile_size, alpha_cut, kind="render",
                 projection=_lib.VG_PINHOLE, extent=0.0):
        self.ctx = ctx
        self.dscene = dscene
        self.camera = camera
        self.mode = mode
        self.tile_size = tile_size
        self.alpha_cut = alpha_cut
        self.kind = kind
        self.projection = projection
        self.extent = extent
        self.fwd = None          # (flags, color, final_t, n_contrib) device tensors
        self._grid = None
        self._pooled = False     # ctx came from _lib.pooled_context (returned on collection)

    def __del__(self):
        if getattr(self, "_pooled", False):
            try:
                _lib.release_context(self.ctx)
            except Exception:
                pass

    @property
    def n_tiles_x(self):
        return (int(self.camera.width) + TILE_SIZE - 1) // TILE_SIZE

    @property
    def n_tiles_y(self):
        return (int(self.camera.height) + TILE_SIZE - 1) // TILE_SIZE

    def pair_count(self):
        import ctypes
        out = ctypes.c_int64()
        _lib.check(_lib.load().vg_pair_count(self.ctx.handle, ctypes.byref(out)), "vg_pair_count")
        return int(out.value)

    def n_active(self):
        """Per-pixel count of active entries (transmittance in front >=
        early_stop, raster.py:384-385) of the last render on this prep, as an
        int32 (H, W) array on the host (diagnostic: the parity tests use it to
        find early-stop decisions float32 took differently from float64)."""
        torch = _lib._require_cuda()
        if self.fwd is None:
            raise ValueError("n_active: render on this prep first")
        H, W = int(self.camera.height), int(self.camera.width)
        out = torch.empty((H, W), dtype=torch.int32, device=self.dscene.device)
        _lib.check(_lib.load().vg_n_active(self.ctx.handle, _lib.ptr(out), _stream(self.dscene.device)),
                   "vg_n_active")
        return out.cpu().numpy()

    def tile_lists_device(self):
        """(prims int32[P], offsets int32[n_tiles+1]) on the device."""
        torch = _lib._require_cuda()
        P = self.pair_count()
        dev = self.dscene.device
        prims = torch.empty(max(P, 1), dtype=torch.int32, device=dev)
        offs = torch.empty(self.n_tiles_x * self.n_tiles_y + 1, dtype=torch.int32, device=dev)
        st = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(_lib.load().vg_tile_lists(self.ctx.handle, _lib.ptr(prims), _lib.ptr(offs), st),
                   "vg_tile_lists")
        return prims[:P], offs

    @property
    def grid(self):
        if self._grid is None:
            prims, offs = self.tile_lists_device()
            p = prims.cpu().numpy().astype(np.int64)
            o = offs.cpu().numpy().astype(np.int64)
            tiles = [p[o[t]:o[t + 1]] for t in range(len(o) - 1)]
            self._grid = TileGrid(TILE_SIZE, self.n_tiles_x, self.n_tiles_y, tiles, self.depth())
        return self._grid

    def depth(self):
        """View-space depth of every primitive (TileGrid.sort_keys)."""
        torch = _lib._require_cuda()
        R = torch.tensor(np.asarray(self.camera.rotation, dtype=np.float64), device=self.dscene.device)
        t = torch.tensor(np.asarray(self.camera.translation, dtype=np.float64), device=self.dscene.device)
        z = self.dscene.means.double() @ R[2] + t[2]
        return z.cpu().numpy()


def _options(tile_size, early_stop, alpha_cut, alpha_clamp, bin_cut, sort_by="depth",
             mode="analytic"):
    return _lib.make_options(tile_size, early_stop, alpha_cut, alpha_clamp, bin_cut, sort_by,
                             mode=mode)


def _stream(dev):
    import torch
    return torch.cuda.current_stream(dev).cuda_stream


def prepare(scene, camera, mode="analytic", tile_size=TILE_SIZE, sort_by="depth",
            alpha_cut=ALPHA_CUT, *, _ctx=None, _kind="render", _bin_cut=None,
            _projection=_lib.VG_PINHOLE, _extent=0.0) -> Prep:
    """raster.prepare (raster.py:263-296): project, bin and sort on the GPU.
    Returns a Prep that owns its own device context."""
    _check_mode(mode, sort_by, tile_size)
    dscene = scene if isinstance(scene, DeviceScene) else DeviceScene(scene)
    ctx = _ctx if _ctx is not None else _lib.pooled_context(dscene.device.index)
    bin_cut = alpha_cut if _bin_cut is None else _bin_cut
    opt = _options(tile_size, EARLY_STOP_T, alpha_cut, ALPHA_CLAMP, bin_cut, sort_by, mode)
    cam = _lib.make_camera(camera, _projection, _extent)
    s = dscene.struct()
    import ctypes
    _lib.check(_lib.load().vg_prepare(ctx.handle, ctypes.byref(s), ctypes.byref(cam),
                                      ctypes.byref(opt), _stream(dscene.device)), "vg_prepare")
    prep = Prep(ctx, dscene, camera, mode, tile_size, alpha_cut, _kind, _projection, _extent)
    prep._pooled = _ctx is None
    return prep


def bin_tiles(scene, camera, tile_size=TILE_SIZE, mode="analytic", sort_by="depth") -> TileGrid:
    """raster.bin_tiles (raster.py:315-319)."""
    return prepare(scene, camera, mode=mode, tile_size=tile_size, sort_by=sort_by).grid


def _forward(prep, early_stop, alpha_cut, alpha_clamp):
    import ctypes
    torch = _lib._require_cuda()
    flags = (early_stop, alpha_cut, alpha_clamp)
    if prep.fwd is not None and prep.fwd[0] == flags:
        return prep.fwd
    lib = _lib.load()
    opt = _options(TILE_SIZE, early_stop, alpha_cut, alpha_clamp, prep.alpha_cut)
    _lib.check(lib.vg_set_options(prep.ctx.handle, ctypes.byref(opt)), "vg_set_options")
    H, W = int(prep.camera.height), int(prep.camera.width)
    dev = prep.dscene.device
    color = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
    tfin = torch.empty((H, W), dtype=torch.float32, device=dev)
    ncon = torch.empty((H, W), dtype=torch.int32, device=dev)
    _lib.check(lib.vg_render_forward(prep.ctx.handle, _lib.ptr(color), _lib.ptr(tfin), _lib.ptr(ncon),
                                     _stream(dev)), "vg_render_forward")
    prep.fwd = (flags, color, tfin, ncon)
    return prep.fwd


def _out(x, torch_in):
    if torch_in:
        return x
    return hostio.to_host(x, np.float64 if x.dtype.is_floating_point else np.int32)


def render(scene, camera, mode="analytic", *, tile_size=TILE_SIZE, threads=None, sort_by="depth",
           early_stop=EARLY_STOP_T, alpha_cut=ALPHA_CUT, alpha_clamp=ALPHA_CLAMP,
           prep: Prep = None) -> RenderOutput:
    """raster.render (raster.py:410-439), analytic mode.  `threads` is
    accepted and ignored (the GPU result does not depend on it)."""
    _check_mode(mode, sort_by, tile_size)
    if prep is None:
        dscene = DeviceScene(scene)
        prep = prepare(dscene, camera, mode, tile_size, sort_by, alpha_cut,
                       _ctx=_lib.scratch_context(dscene.device.index))
        torch_in = dscene.torch_in
    else:
        torch_in = prep.dscene.torch_in
    _, color, tfin, ncon = _forward(prep, early_stop, alpha_cut, alpha_clamp)
    return RenderOutput(_out(color, torch_in), _out(tfin, torch_in), _out(ncon, torch_in), mode)


def composite_pixel(contributions, background, early_stop=EARLY_STOP_T):
    """Scalar compositing specification (raster.py:442-454): an entry is
    composited iff the transmittance in front of it is >= early_stop.  A
    host-side helper for tests and documentation, not a compute path."""
    color = np.zeros(3)
    t = 1.0
    stop = early_stop if early_stop is not None else 0.0
    for alpha, c in contributions:
        if t < stop:
            break
        color += t * alpha * np.asarray(c, dtype=float)
        t *= 1.0 - alpha
    return color + t * np.asarray(background, dtype=float), t
