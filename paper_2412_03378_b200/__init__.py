"""B200-native analytic-transmittance Gaussian rasterizer (arXiv 2412.03378).

Drop-in for the hot path of the reference package `volgauss` 0.1.0:
`render`, `prepare`, `bin_tiles`, `backward`, `tomo_forward`,
`tomo_backward` keep the reference signatures; the compute runs in
hand-written sm_100a kernels behind the C ABI in include/volgauss_b200.h.
Importing the package does not touch CUDA; the first call loads
libvolgauss_b200.so and raises RuntimeError if it (or a GPU) is missing.
"""

from .camera import Camera, look_at
from .grad import (FdRecord, FdReport, LossSpec, ParamGrad, SceneGrads, backward, fd_check, loss_and_grad,
                   loss_value)
from .raster import (ALPHA_CLAMP, ALPHA_CUT, EARLY_STOP_T, TILE_SIZE, Prep, RenderOutput, Scene,
                     TileGrid, bin_tiles, composite_pixel, prepare, render)
from .tomo import TOMO_BIN_CUT, tomo_backward, tomo_forward, tomo_prepare

__version__ = "0.1.0"

__all__ = [
    "ALPHA_CLAMP", "ALPHA_CUT", "Camera", "EARLY_STOP_T", "LossSpec", "ParamGrad", "Prep",
    "RenderOutput", "Scene", "SceneGrads", "TILE_SIZE", "TOMO_BIN_CUT", "TileGrid", "backward",
    "bin_tiles", "composite_pixel", "look_at", "loss_and_grad", "loss_value", "fd_check", "FdReport", "FdRecord", "prepare", "render",
    "tomo_backward", "tomo_forward", "tomo_prepare",
]
