"""Image / volume quality numbers used by the reconstruction report
(metrics.psnr_volume / ssim_volume of the reference, metrics.py:98-122) and
the SSIM term of the photometric losses (metrics.ssim / ssim_with_grad,
metrics.py:60-95: the D-SSIM / mixed losses of grad.loss_and_grad).

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


def ssim_with_grad(x, y):
    """(mean SSIM, d mean-SSIM / dx) for images sharing a unit data range
    (reference metrics.ssim_with_grad, metrics.py:70-95).  SSIM per pixel is
    A1 A2 / (B1 B2) with A1 = 2 mx my + C1, A2 = 2 cxy + C2,
    B1 = mx^2 + my^2 + C1, B2 = vx + vy + C2 over the blurred moments
    mx = F(x), F(x^2), F(xy); the zero-padded separable Gaussian blur F is
    self-adjoint, so the gradient is F applied to the per-pixel sensitivities
    of mx, F(x^2) and F(xy), times 1, 2x and y.  numpy arrays, or torch
    tensors (computed in float64 on their device)."""
    if not isinstance(x, np.ndarray) and hasattr(x, "device"):
        return _ssim_with_grad_torch(x, y)
    x = np.asarray(x, dtype=float)
    y = np.asarray(y, dtype=float)
    w = _window()
    mx, my = _blur(x, w), _blur(y, w)
    a1 = 2.0 * mx * my + _C1
    a2 = 2.0 * (_blur(x * y, w) - mx * my) + _C2
    b1 = mx * mx + my * my + _C1
    b2 = (_blur(x * x, w) - mx * mx) + (_blur(y * y, w) - my * my) + _C2
    smap = a1 * a2 / (b1 * b2)
    inv_n = 1.0 / smap.size
    # sensitivities of mean SSIM to mx, to F(x^2) and to F(xy)
    d_a1, d_a2 = a2 / (b1 * b2), a1 / (b1 * b2)
    d_b1, d_b2 = -smap / b1, -smap / b2
    g_mx = inv_n * (2.0 * my * d_a1 - 2.0 * my * d_a2 + 2.0 * mx * d_b1 - 2.0 * mx * d_b2)
    g_xx = inv_n * d_b2
    g_xy = inv_n * 2.0 * d_a2
    dx = _blur(g_mx, w) + 2.0 * x * _blur(g_xx, w) + y * _blur(g_xy, w)
    return float(np.mean(smap)), dx


def _ssim_with_grad_torch(x, y):
    import torch
    x = x.to(torch.float64)
    y = y.to(y.device if hasattr(y, "device") else x.device, torch.float64) if hasattr(y, "device") \
        else torch.as_tensor(np.asarray(y, dtype=float), device=x.device)
    w = torch.as_tensor(_window(), dtype=torch.float64, device=x.device)

    def blur(a):
        # zero-padded separable correlation over the two image axes
        img = a.unsqueeze(-1) if a.dim() == 2 else a           # (H, W, C)
        t = img.permute(2, 0, 1).unsqueeze(1)                  # (C, 1, H, W)
        k = w.numel()
        t = torch.nn.functional.conv2d(t, w.view(1, 1, k, 1), padding=(k // 2, 0))
        t = torch.nn.functional.conv2d(t, w.view(1, 1, 1, k), padding=(0, k // 2))
        out = t.squeeze(1).permute(1, 2, 0)
        return out.squeeze(-1) if a.dim() == 2 else out

    mx, my = blur(x), blur(y)
    a1 = 2.0 * mx * my + _C1
    a2 = 2.0 * (blur(x * y) - mx * my) + _C2
    b1 = mx * mx + my * my + _C1
    b2 = (blur(x * x) - mx * mx) + (blur(y * y) - my * my) + _C2
    smap = a1 * a2 / (b1 * b2)
    inv_n = 1.0 / smap.numel()
    d_a1, d_a2 = a2 / (b1 * b2), a1 / (b1 * b2)
    d_b1, d_b2 = -smap / b1, -smap / b2
    g_mx = inv_n * (2.0 * my * d_a1 - 2.0 * my * d_a2 + 2.0 * mx * d_b1 - 2.0 * mx * d_b2)
    dx = blur(g_mx) + 2.0 * x * blur(inv_n * d_b2) + y * blur(inv_n * 2.0 * d_a2)
    return smap.mean(), dx


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
