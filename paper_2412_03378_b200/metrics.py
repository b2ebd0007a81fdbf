"""Image / volume quality numbers used by the reconstruction report
(metrics.psnr_volume / ssim_volume of the reference, metrics.py:98-122).

Host-side numpy: an 11-tap Gaussian window (sigma 1.5, normalised), separable
zero-padded filtering over the two image axes, C1 = 0.01^2, C2 = 0.03^2 for a
unit data range; the volume SSIM averages slice SSIMs along each axis, then
over the three axes, after scaling both volumes by the reference's peak.
"""

from __future__ import annotations

import math

import numpy as np
from scipy.ndimage import correlate1d

_C1, _C2 = 1e-4, 9e-4


def _window(size=11, sigma=1.5):
    x = np.arange(size, dtype=float) - 0.5 * (size - 1)
    w = np.exp(-0.5 * (x / sigma) ** 2)
    return w / np.sum(w)


def _blur(img, w):
    return correlate1d(correlate1d(img, w, axis=0, mode="constant"), w, axis=1, mode="constant")


def ssim(x, y):
    """Mean SSIM of two images sharing a unit data range."""
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=float)
    w = _window()
    mx, my = _blur(x, w), _blur(y, w)
    vx = _blur(x * x, w) - mx * mx
    vy = _blur(y * y, w) - my * my
    cxy = _blur(x * y, w) - mx * my
    num = (2.0 * mx * my + _C1) * (2.0 * cxy + _C2)
    den = (mx * mx + my * my + _C1) * (vx + vy + _C2)
    return float(np.mean(num / den))


def psnr_volume(recon, reference):
    """10 log10(peak^2 / MSE) with peak = the reference's maximum."""
    recon = np.asarray(recon, dtype=float)
    reference = np.asarray(reference, dtype=float)
    err = float(np.mean((recon - reference) ** 2))
    if err == 0.0:
        return math.inf
    peak = float(np.max(reference))
    return 10.0 * math.log10(peak * peak / err)


def ssim_volume(a, b):
    """Slice SSIM averaged along each axis, then over the axes (b's peak = 1)."""
    peak = max(float(np.max(b)), 1e-12)
    a = np.asarray(a, dtype=float) / peak
    b = np.asarray(b, dtype=float) / peak
    per_axis = []
    for ax in range(3):
        sa, sb = np.moveaxis(a, ax, 0), np.moveaxis(b, ax, 0)
        per_axis.append(float(np.mean([ssim(sa[k], sb[k]) for k in range(sa.shape[0])])))
    return float(np.mean(per_axis))
