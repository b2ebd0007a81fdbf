"""ctypes binding of libvolgauss_b200.so (include/volgauss_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is present, every entry point raises RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# VG_LIB: an alternative build of the same library (the checking variant of
# tools/debug_checks.py); the default is the in-tree release build
LIB_PATH = os.environ.get("VG_LIB") or os.path.join(_HERE, "libvolgauss_b200.so")

VG_OK, VG_EINVAL, VG_ECUDA, VG_ENOMEM = 0, 1, 2, 3
VG_PINHOLE, VG_PARALLEL = 0, 1
VG_OVERWRITE, VG_ADD, VG_DEFER = 0, 1, 2
ABI_VERSION = 1


class VgCamera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("projection", C.c_int32),
                ("_pad", C.c_int32), ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double),
                ("cy", C.c_double), ("rotation", C.c_double * 9), ("translation", C.c_double * 3),
                ("z_near", C.c_double), ("extent", C.c_double)]


class VgOptions(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("_pad", C.c_int32), ("early_stop", C.c_double),
                ("alpha_cut", C.c_double), ("alpha_clamp", C.c_double), ("bin_cut", C.c_double),
                ("sort_by", C.c_int32), ("deterministic", C.c_int32), ("mode", C.c_int32),
                ("_pad3", C.c_int32)]


class VgScene(C.Structure):
    _fields_ = [("means", C.c_void_p), ("scales", C.c_void_p), ("rotations", C.c_void_p),
                ("thetas", C.c_void_p), ("colors", C.c_void_p), ("sh", C.c_void_p),
                ("n", C.c_int64), ("background", C.c_double * 3), ("splat_opacities", C.c_void_p)]


class VgGrads(C.Structure):
    _fields_ = [("d_means", C.c_void_p), ("d_scales", C.c_void_p), ("d_rotations", C.c_void_p),
                ("d_thetas", C.c_void_p), ("d_colors", C.c_void_p), ("d_kappas", C.c_void_p),
                ("d_sh", C.c_void_p), ("d_background", C.c_void_p), ("visible", C.c_void_p),
                ("accumulate", C.c_int32), ("_pad", C.c_int32), ("d_splat_opacities", C.c_void_p)]


class VgTrainState(C.Structure):
    _fields_ = [("means", C.c_void_p), ("scales", C.c_void_p), ("rotations", C.c_void_p),
                ("thetas", C.c_void_p), ("colors", C.c_void_p), ("color_raw", C.c_void_p),
                ("moments", C.c_void_p), ("accum_norm", C.c_void_p), ("accum_count", C.c_void_p),
                ("n", C.c_int64)]


class VgAdamHparams(C.Structure):
    _fields_ = [("lr", C.c_double * 5), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("t", C.c_int64)]


class VgDensifyArgs(C.Structure):
    _fields_ = [("n", C.c_int64), ("means", C.c_void_p), ("scales", C.c_void_p),
                ("rotations", C.c_void_p), ("thetas", C.c_void_p), ("colors", C.c_void_p),
                ("color_raw", C.c_void_p), ("moments", C.c_void_p), ("accum_norm", C.c_void_p),
                ("accum_count", C.c_void_p), ("extent", C.c_double),
                ("split_grad_threshold", C.c_double), ("clone_grad_threshold", C.c_double),
                ("prune_theta_min", C.c_double), ("prune_scale_fraction", C.c_double),
                ("high_kappa_split_fraction", C.c_double), ("max_primitives", C.c_int64)]


EXPORTS = {
    "vg_abi_version": (C.c_int, []),
    "vg_last_error": (C.c_char_p, []),
    "vg_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32]),
    "vg_destroy": (None, [C.c_void_p]),
    "vg_prepare": (C.c_int, [C.c_void_p, C.POINTER(VgScene), C.POINTER(VgCamera),
                             C.POINTER(VgOptions), C.c_void_p]),
    "vg_prepare_async": (C.c_int, [C.c_void_p, C.POINTER(VgScene), C.POINTER(VgCamera),
                                   C.POINTER(VgOptions), C.c_void_p]),
    "vg_prepare_finish": (C.c_int, [C.c_void_p, C.c_void_p]),
    "vg_set_options": (C.c_int, [C.c_void_p, C.POINTER(VgOptions)]),
    "vg_pair_count": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "vg_tile_lists": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vg_render_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vg_render_backward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.POINTER(VgGrads), C.c_void_p]),
    "vg_render_backward_l2": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.POINTER(VgGrads), C.c_void_p]),
    "vg_n_active": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "vg_visible_pairs": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "vg_merge_deferred": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "vg_copy_streaming": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int32, C.c_void_p]),
    "vg_voxelize": (C.c_int, [C.POINTER(VgScene), C.POINTER(C.c_double), C.POINTER(C.c_double),
                              C.POINTER(C.c_int32), C.c_void_p, C.c_void_p]),
    "vg_tomo_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vg_tomo_backward": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(VgGrads), C.c_void_p]),
    "vg_tomo_backward_l2": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.POINTER(VgGrads), C.c_void_p]),
    "vg_launch_count": (C.c_int64, [C.c_void_p]),
    "vg_finalize_grads": (C.c_int, [C.c_void_p, C.POINTER(VgGrads), C.c_void_p]),
    "vg_profile": (C.c_int, [C.c_void_p, C.c_int32]),
    "vg_profile_read": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "vg_probe_peaks": (C.c_int, [C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "vg_raymarch": (C.c_int, [C.POINTER(VgScene), C.POINTER(VgCamera), C.c_int32, C.c_double,
                              C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]),
    "vg_debug_forward_stats": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p]),
    "vg_debug_cta_log": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "vg_debug_segments": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "vg_nccl_available": (C.c_int, []),
    "vg_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "vg_nccl_comm_init": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.c_void_p, C.c_int32, C.c_int32]),
    "vg_nccl_comm_destroy": (C.c_int, [C.c_void_p]),
    "vg_allreduce_grads": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                     C.c_void_p, C.c_void_p]),
    "vg_adam_step": (C.c_int, [C.POINTER(VgTrainState), C.POINTER(VgGrads), C.POINTER(VgAdamHparams),
                               C.c_void_p, C.c_void_p]),
    "vg_densify_scratch_bytes": (C.c_size_t, [C.c_int64]),
    "vg_densify_plan": (C.c_int, [C.POINTER(VgDensifyArgs), C.c_void_p, C.c_void_p, C.c_void_p]),
    "vg_densify_apply": (C.c_int, [C.POINTER(VgDensifyArgs), C.c_void_p, C.POINTER(C.c_uint32),
                                   C.c_void_p, C.POINTER(VgTrainState), C.c_void_p]),
}

KERNEL_KINDS = ("preprocess", "scan", "duplicate", "sort", "ranges", "render_fwd", "render_bwd",
                "finalize", "tomo_fwd", "tomo_bwd")

_lib = None
_lock = threading.Lock()


def load():
    """Load the shared library (no CUDA calls).  Raises RuntimeError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build the CUDA extension with "
                    "`python -m paper_2412_03378_b200.build` (there is no CPU fallback)")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in EXPORTS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.vg_abi_version() != ABI_VERSION:
                raise RuntimeError("libvolgauss_b200.so ABI version mismatch; rebuild it")
            _lib = lib
    return _lib


def check(code, what=""):
    if code == VG_OK:
        return
    msg = (load().vg_last_error() or b"").decode(errors="replace")
    if code == VG_EINVAL:
        raise ValueError(f"{what}: {msg}" if what else msg)
    raise RuntimeError(f"{what}: {msg} (code {code})" if what else msg)


def _require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("volgauss_b200 needs a CUDA device (B200); no CPU fallback exists")
    return torch


class Context:
    """One vg_context: the device-side `prep` state (records, sorted tile
    lists, per-pixel forward state).  Not thread-safe."""

    def __init__(self, device=None):
        torch = _require_cuda()
        lib = load()
        self.device = torch.cuda.current_device() if device is None else int(device)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            check(lib.vg_create(C.byref(h), self.device), "vg_create")
        self._h = h
        self._lib = lib

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.vg_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launches(self):
        return int(self._lib.vg_launch_count(self._h))

    def profile(self, enable=True):
        check(self._lib.vg_profile(self._h, 1 if enable else 0), "vg_profile")

    def profile_read(self):
        """{kind: (total_ms, launches)} for the events recorded since profile(True)."""
        n = len(KERNEL_KINDS)
        ms = (C.c_double * n)()
        cnt = (C.c_int64 * n)()
        check(self._lib.vg_profile_read(self._h, ms, cnt), "vg_profile_read")
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNEL_KINDS)}


_tls = threading.local()
_ctx_pool = {}          # device -> contexts released by collected Prep objects
_ctx_pool_lock = threading.Lock()
_CTX_POOL_MAX = 4


def pooled_context(device):
    """A context for a new Prep (raster.prepare without _ctx): one released
    by a collected Prep if available -- its device buffers are already
    sized, so a prepare -> render -> backward sequence per iteration (the
    reference's optim.py:379-386 pattern) does not re-create and re-grow a
    context every call -- else a new one.  Reuse is stream-ordered on the
    caller's stream."""
    with _ctx_pool_lock:
        pool = _ctx_pool.get(int(device))
        if pool:
            return pool.pop()
    return Context(device)


def release_context(ctx):
    """Return a Prep's context to the pool (called when the Prep is collected)."""
    if ctx is None or not getattr(ctx, "_h", None) or not ctx._h.value:
        return
    with _ctx_pool_lock:
        pool = _ctx_pool.setdefault(ctx.device, [])
        if len(pool) < _CTX_POOL_MAX:
            pool.append(ctx)
            return
    ctx.close()


def scratch_context(device):
    """Per-thread, per-device context for calls made without `prep=`."""
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    if device not in cache:
        cache[device] = Context(device)
    return cache[device]


def make_camera(cam, projection=VG_PINHOLE, extent=0.0):
    c = VgCamera()
    c.width = int(cam.width)
    c.height = int(cam.height)
    c.projection = projection
    c.fx, c.fy, c.cx, c.cy = (float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy))
    R = np.asarray(cam.rotation, dtype=np.float64).reshape(9)
    t = np.asarray(cam.translation, dtype=np.float64).reshape(3)
    for i in range(9):
        c.rotation[i] = float(R[i])
    for i in range(3):
        c.translation[i] = float(t[i])
    c.z_near = float(getattr(cam, "z_near", 0.01))
    c.extent = float(extent)
    return c


VG_SORT_DEPTH, VG_SORT_GAMMA = 0, 1


VG_MODE_ANALYTIC, VG_MODE_SPLAT = 0, 1


def make_options(tile_size, early_stop, alpha_cut, alpha_clamp, bin_cut, sort_by="depth",
                 deterministic=False, mode="analytic"):
    o = VgOptions()
    o.mode = VG_MODE_SPLAT if mode == "splat" else VG_MODE_ANALYTIC
    o.deterministic = 1 if deterministic else 0
    o.sort_by = VG_SORT_GAMMA if sort_by == "gamma" else VG_SORT_DEPTH
    o.tile_size = int(tile_size)
    o.early_stop = -1.0 if early_stop is None else float(early_stop)
    o.alpha_cut = float(alpha_cut)
    o.alpha_clamp = float(alpha_clamp)
    o.bin_cut = float(bin_cut)
    return o


def ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)
