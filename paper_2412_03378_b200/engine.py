"""Low-level device engine: one vg_context plus reusable device buffers.

The drop-in functions in raster/grad/tomo are built for reference
compatibility (numpy in, numpy out).  Training loops, the multi-GPU step
and the benchmark use this engine instead: scene tensors stay resident in
HBM, per-view outputs reuse cached buffers, gradients of many views
accumulate into one flat buffer (GradBuffers) that a single NCCL
all-reduce can sum across GPUs, and the L2 loss is fused into the backward
blend (vg_render_backward_l2).  No call here synchronises the host.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .grad import GradBuffers
from .raster import ALPHA_CLAMP, ALPHA_CUT, EARLY_STOP_T, TILE_SIZE, DeviceScene
from .tomo import TOMO_BIN_CUT


class Engine:
    def __init__(self, device=None, early_stop=EARLY_STOP_T, alpha_cut=ALPHA_CUT,
                 alpha_clamp=ALPHA_CLAMP, deterministic=False, sort_by="depth", mode="analytic"):
        torch = _lib._require_cuda()
        self.torch = torch
        self.ctx = _lib.Context(device)
        self.device = torch.device("cuda", self.ctx.device)
        self.flags = (early_stop, alpha_cut, alpha_clamp)
        self.deterministic = deterministic   # fixed-order gradient sums (vg_det.cu)
        self.sort_by = sort_by
        self.mode = mode                     # "analytic" or "splat" (the EWA comparator)
        self.lib = _lib.load()
        self._bufs = {}
        self.cam = None
        self.dscene = None

    # -- helpers -----------------------------------------------------------
    def stream(self):
        return self.torch.cuda.current_stream(self.device).cuda_stream

    def _buf(self, key, shape, dtype):
        b = self._bufs.get(key)
        if b is None or tuple(b.shape) != tuple(shape) or b.dtype != dtype:
            b = self.torch.empty(shape, dtype=dtype, device=self.device)
            self._bufs[key] = b
        return b

    def upload(self, scene):
        return scene if isinstance(scene, DeviceScene) else DeviceScene(scene, self.ctx.device)

    def new_grads(self, ds):
        return GradBuffers(ds.n, self.device, with_sh=ds.sh is not None)

    def launches(self):
        return self.ctx.launches()

    # -- pipeline ----------------------------------------------------------
    def prepare(self, ds, cam, *, tomo=False, parallel=False, extent=1.6):
        self.prepare_async(ds, cam, tomo=tomo, parallel=parallel, extent=extent)
        self.prepare_finish()

    def prepare_async(self, ds, cam, *, tomo=False, parallel=False, extent=1.6):
        """First half of prepare (no host wait); see vg_prepare_async."""
        es, ac, cl = self.flags
        bin_cut = TOMO_BIN_CUT if tomo else ac
        opt = _lib.make_options(TILE_SIZE, es, ac, cl, bin_cut, sort_by=self.sort_by,
                                deterministic=self.deterministic, mode=self.mode)
        c = _lib.make_camera(cam, _lib.VG_PARALLEL if parallel else _lib.VG_PINHOLE,
                             extent if parallel else 0.0)
        s = ds.struct()
        _lib.check(self.lib.vg_prepare_async(self.ctx.handle, ctypes.byref(s), ctypes.byref(c),
                                             ctypes.byref(opt), self.stream()), "vg_prepare_async")
        self.cam = cam
        self.dscene = ds

    def prepare_finish(self):
        _lib.check(self.lib.vg_prepare_finish(self.ctx.handle, self.stream()), "vg_prepare_finish")

    def forward(self, slot=0, counts=True):
        """Forward blend -> (color, final_T, n_contrib).  counts=False skips
        the per-pixel counts (n_contrib is then None): the training step."""
        H, W = int(self.cam.height), int(self.cam.width)
        t = self.torch
        color = self._buf(("color", slot), (H, W, 3), t.float32)
        tfin = self._buf(("T", slot), (H, W), t.float32)
        ncon = self._buf(("nc", slot), (H, W), t.int32) if counts else None
        _lib.check(self.lib.vg_render_forward(self.ctx.handle, _lib.ptr(color), _lib.ptr(tfin),
                                              _lib.ptr(ncon), self.stream()), "vg_render_forward")
        return color, tfin, ncon

    def n_active(self, slot=0):
        """Per-pixel active-entry counts of the last forward (device int32)."""
        H, W = int(self.cam.height), int(self.cam.width)
        out = self._buf(("na", slot), (H, W), self.torch.int32)
        _lib.check(self.lib.vg_n_active(self.ctx.handle, _lib.ptr(out), self.stream()), "vg_n_active")
        return out

    def pair_count(self):
        """(tile, Gaussian) pairs of the last prepare (synchronises)."""
        out = ctypes.c_int64()
        _lib.check(self.lib.vg_pair_count(self.ctx.handle, ctypes.byref(out)), "vg_pair_count")
        return int(out.value)

    def visible_pairs(self):
        """(entry, 64-pixel warp block) pairs the last forward marked visible:
        the pairs the backward walks (synchronises; diagnostic)."""
        out = ctypes.c_int64()
        _lib.check(self.lib.vg_visible_pairs(self.ctx.handle, ctypes.byref(out)), "vg_visible_pairs")
        return int(out.value)

    def forward_stats(self):
        """Roofline counts of the prepared view (diagnostic, synchronises):
        (evaluated forward (entry, warp-block) pairs, of which visible, list
        entries walked per warp); runs an extra counting forward."""
        H, W = int(self.cam.height), int(self.cam.width)
        t = self.torch
        color = self._buf(("color", "stats"), (H, W, 3), t.float32)
        tfin = self._buf(("T", "stats"), (H, W), t.float32)
        ncon = self._buf(("nc", "stats"), (H, W), t.int32)
        out = (ctypes.c_ulonglong * 4)()
        _lib.check(self.lib.vg_debug_forward_stats(self.ctx.handle, _lib.ptr(color), _lib.ptr(tfin),
                                                   _lib.ptr(ncon), out, self.stream()),
                   "vg_debug_forward_stats")
        return int(out[0]), int(out[1]), int(out[2])

    def backward(self, color, tfin, d_color, grads, d_t=None, accumulate=False):
        g = grads.struct(accumulate)
        _lib.check(self.lib.vg_render_backward(self.ctx.handle, _lib.ptr(color), _lib.ptr(tfin),
                                               _lib.ptr(d_color), _lib.ptr(d_t), ctypes.byref(g),
                                               self.stream()), "vg_render_backward")

    def backward_l2(self, color, tfin, target, grads, accumulate=False, loss=None):
        """Fused L2: returns the device scalar mean((color-target)^2) (or adds
        the sum of squares into `loss`, a float64 device scalar, if given)."""
        out = loss if loss is not None else self.torch.zeros((), dtype=self.torch.float64,
                                                              device=self.device)
        g = grads.struct(accumulate)
        _lib.check(self.lib.vg_render_backward_l2(self.ctx.handle, _lib.ptr(color), _lib.ptr(tfin),
                                                  _lib.ptr(target), _lib.ptr(out), ctypes.byref(g),
                                                  self.stream()), "vg_render_backward_l2")
        if loss is None:
            return out / color.numel()
        return out

    def merge_deferred(self, other):
        """Move `other`'s deferred (VG_DEFER) accumulators into this engine's,
        so that one finalize covers both (same scene, same device)."""
        _lib.check(self.lib.vg_merge_deferred(self.ctx.handle, other.ctx.handle, self.stream()),
                   "vg_merge_deferred")

    def finalize(self, grads, accumulate=True):
        """Write the geometry gradients of all VG_DEFER backward calls since
        the last finalize into `grads` (added unless accumulate=False)."""
        g = grads.struct(accumulate)
        _lib.check(self.lib.vg_finalize_grads(self.ctx.handle, ctypes.byref(g), self.stream()),
                   "vg_finalize_grads")

    def tomo_forward(self, slot=0, intensity=False):
        H, W = int(self.cam.height), int(self.cam.width)
        img = self._buf(("img", slot), (H, W), self.torch.float32)
        inten = self._buf(("inten", slot), (H, W), self.torch.float32) if intensity else None
        _lib.check(self.lib.vg_tomo_forward(self.ctx.handle, _lib.ptr(img), _lib.ptr(inten),
                                            self.stream()), "vg_tomo_forward")
        return (img, inten) if intensity else img

    def tomo_backward(self, d_image, grads, accumulate=False):
        g = grads.struct(accumulate)
        _lib.check(self.lib.vg_tomo_backward(self.ctx.handle, _lib.ptr(d_image), ctypes.byref(g),
                                             self.stream()), "vg_tomo_backward")

    def tomo_backward_l2(self, image, target, grads, accumulate=False, loss=None):
        out = loss if loss is not None else self.torch.zeros((), dtype=self.torch.float64,
                                                              device=self.device)
        g = grads.struct(accumulate)
        _lib.check(self.lib.vg_tomo_backward_l2(self.ctx.handle, _lib.ptr(image), _lib.ptr(target),
                                                _lib.ptr(out), ctypes.byref(g), self.stream()),
                   "vg_tomo_backward_l2")
        if loss is None:
            return out / image.numel()
        return out
