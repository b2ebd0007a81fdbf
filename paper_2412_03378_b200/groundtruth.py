"""Ground-truth renderer on the GPU: the reference's
validation oracle `volgauss.oracle.raymarch_image` (oracle.py:80-161) --
midpoint-rule quadrature of the volume rendering equation through the full
Gaussian mixture density, independent of the closed-form transmittance path
the rasterizer uses -- as one sm_100a kernel (vg_raymarch, one CTA per pixel
ray, float64).  For accuracy studies of the analytic renderer at image sizes
the CPU oracle cannot reach.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass


from . import _lib
from .raster import DeviceScene, _out, _stream


@dataclass
class MarchConfig:
    """oracle.MarchConfig (oracle.py:21-30): None bounds auto-fit the mixture
    support (the hull of [gamma - k beta, gamma + k beta] per ray, t >= 0)."""
    n_steps: int = 10_000
    t_min: float = None
    t_max: float = None
    support_sigmas: float = 8.0


def raymarch_image(scene, camera, cfg: MarchConfig = None):
    """Quadrature render of a full camera -> (color (H,W,3), final_T (H,W)),
    numpy float64 for numpy scenes (like the reference), CUDA tensors for
    CUDA-tensor scenes."""
    cfg = cfg or MarchConfig()
    torch = _lib._require_cuda()
    ds = scene if isinstance(scene, DeviceScene) else DeviceScene(scene)
    H, W = int(camera.height), int(camera.width)
    color = torch.empty((H, W, 3), dtype=torch.float32, device=ds.device)
    tfin = torch.empty((H, W), dtype=torch.float32, device=ds.device)
    s = ds.struct()
    cam = _lib.make_camera(camera, _lib.VG_PINHOLE, 0.0)
    nan = math.nan
    _lib.check(_lib.load().vg_raymarch(ctypes.byref(s), ctypes.byref(cam), int(cfg.n_steps),
                                       float(cfg.support_sigmas),
                                       nan if cfg.t_min is None else float(cfg.t_min),
                                       nan if cfg.t_max is None else float(cfg.t_max),
                                       _lib.ptr(color), _lib.ptr(tfin), _stream(ds.device)),
               "vg_raymarch")
    return _out(color, ds.torch_in), _out(tfin, ds.torch_in)
