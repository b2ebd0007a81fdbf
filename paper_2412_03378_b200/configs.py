"""Seeded synthetic inputs for the five BASELINE.json configurations.

Every array comes from its own counter-based Philox stream keyed by
(seed, stream), the same construction as the reference's `scenes.make_rng`
(`scenes.py:18-21`), so a config is bit-reproducible on any host.  All
per-Gaussian arrays are rounded to float32 (the device input precision); the
oracle / reference receive exactly those rounded values widened to float64.

Densities are specified as kappa in BASELINE.json but the reference API takes
theta, so kappa is mapped through the reference's inverse
(`core.theta_for_kappa`, `core.py:146-153`), computed here in float64.

Choices BASELINE.json leaves open are frozen here and restated in DESIGN.md:
camera FOV 60 degrees everywhere; config 2 cameras on a Fibonacci sphere of
radius 5; config 3 cameras on a Fibonacci upper hemisphere of radius 6,
elevation 10..70 degrees, clusters centred in [-2,2]^3 with per-axis standard
deviations U(0.1, 0.5) under a random rotation; config 4 disks have their thin
axis along the surface normal, 50/50 sphere/torus, cameras on a radius-4
sphere; config 5 uses 180 parallel views over [0, pi) about the world y axis,
detector half-extent 1.6 (the reference TomoGeometry default, `tomo.py:253`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .camera import look_at

SH_C = None  # filled lazily by sh_basis


def make_rng(seed, stream=0):
    """Independent Philox stream keyed by (seed, stream)."""
    return np.random.Generator(np.random.Philox(key=(np.uint64(seed), np.uint64(stream))))


def random_unit_quats(rng, n):
    q = rng.standard_normal((n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def theta_for_kappa(kappa, scales):
    """core.theta_for_kappa restated (core.py:146-153)."""
    s = np.maximum(np.asarray(scales, dtype=np.float64), 1e-7)
    inv_mean = np.mean(1.0 / s, axis=-1)
    th = -np.expm1(-np.asarray(kappa, dtype=np.float64) / inv_mean) / 0.99
    return np.clip(th, 0.0, 1.0)


@dataclass
class SceneArrays:
    """Host-side struct-of-arrays scene (float32 storage, reference field names)."""
    means: np.ndarray
    scales: np.ndarray
    rotations: np.ndarray
    thetas: np.ndarray
    colors: np.ndarray
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))
    sh: np.ndarray = None      # (N, 16, 3) SH-3 coefficients (config 3 only)

    def __len__(self):
        return len(self.means)


@dataclass
class Config:
    name: str
    scene: SceneArrays
    cameras: list
    targets_seed: int
    tomography: bool = False
    parallel: bool = False
    extent: float = 1.6
    description: str = ""

    def target(self, view, shape):
        """Seeded U(0,1) target for `view` (image shape (H,W,3) or (H,W))."""
        return make_rng(self.targets_seed, 1000 + view).uniform(0.0, 1.0, shape).astype(np.float32)


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _finish(means, scales, quats, kappa, colors, background=(0.0, 0.0, 0.0), sh=None):
    means, scales, quats = _f32(means), _f32(scales), _f32(quats)
    thetas = _f32(theta_for_kappa(kappa, scales.astype(np.float64)))
    return SceneArrays(means, scales, quats, thetas, _f32(colors),
                       np.asarray(background, dtype=np.float64),
                       None if sh is None else _f32(sh))


def fibonacci_dirs(n, hemisphere=False, min_elev_deg=None, max_elev_deg=None):
    """Unit directions on a Fibonacci lattice with +y as the polar axis."""
    k = np.arange(n) + 0.5
    if hemisphere:
        lo = math.sin(math.radians(min_elev_deg if min_elev_deg is not None else 0.0))
        hi = math.sin(math.radians(max_elev_deg if max_elev_deg is not None else 90.0))
        y = lo + (hi - lo) * k / n
    else:
        y = 1.0 - 2.0 * k / n
        y = np.clip(y, -0.95, 0.95)
    r = np.sqrt(1.0 - y * y)
    phi = k * math.pi * (3.0 - math.sqrt(5.0))
    return np.stack([r * np.cos(phi), y, r * np.sin(phi)], axis=1)


def tiny(seed=1):
    """Config 1: N=1024, 64x64, camera (0,0,-3) fov 60, U(0,1) target."""
    n = 1024
    means = make_rng(seed, 0).uniform(-1.0, 1.0, (n, 3))
    scales = np.exp(make_rng(seed, 1).uniform(math.log(0.02), math.log(0.2), (n, 3)))
    quats = random_unit_quats(make_rng(seed, 2), n)
    kappa = make_rng(seed, 3).uniform(0.5, 5.0, n)
    colors = make_rng(seed, 4).uniform(0.0, 1.0, (n, 3))
    cam = look_at([0.0, 0.0, -3.0], [0.0, 0.0, 0.0], width=64, height=64, fov_x_deg=60.0)
    return Config("tiny", _finish(means, scales, quats, kappa, colors), [cam], seed,
                  description="config 1: N=1024, 64x64, 1 view")


def medium(seed=2, n=100_000, size=800, n_views=8):
    """Config 2: N=100k, means in [-2,2]^3, 8 cameras on a radius-5 sphere, 800x800."""
    means = make_rng(seed, 0).uniform(-2.0, 2.0, (n, 3))
    scales = np.exp(make_rng(seed, 1).uniform(math.log(0.02), math.log(0.2), (n, 3)))
    quats = random_unit_quats(make_rng(seed, 2), n)
    kappa = make_rng(seed, 3).uniform(0.5, 5.0, n)
    colors = make_rng(seed, 4).uniform(0.0, 1.0, (n, 3))
    cams = [look_at(5.0 * d, [0.0, 0.0, 0.0], width=size, height=size, fov_x_deg=60.0)
            for d in fibonacci_dirs(n_views)]
    return Config("medium", _finish(means, scales, quats, kappa, colors), cams, seed,
                  description=f"config 2: N={n}, {size}x{size}, {n_views} views")


def sh_basis(dirs):
    """Real spherical-harmonic basis up to degree 3 for unit dirs (K,3) -> (K,16)
    (numpy arrays or torch tensors).
    Band 0 is the constant 1 so the DC coefficient is the view-independent RGB;
    bands 1-3 use the standard real-SH normalisation constants."""
    x, y, z = dirs[:, 0], dirs[:, 1], dirs[:, 2]
    c1 = 0.4886025119029199
    c2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
          -1.0925484305920792, 0.5462742152960396)
    c3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
          0.3731763325901154, -0.4570457994644658, 1.445305721320277, -0.5900435899266435)
    xx, yy, zz = x * x, y * y, z * z
    cols = [x * 0 + 1,
            -c1 * y, c1 * z, -c1 * x,
            c2[0] * x * y, c2[1] * y * z, c2[2] * (2 * zz - xx - yy), c2[3] * x * z, c2[4] * (xx - yy),
            c3[0] * y * (3 * xx - yy), c3[1] * x * y * z, c3[2] * y * (4 * zz - xx - yy),
            c3[3] * z * (2 * zz - 3 * xx - 3 * yy), c3[4] * x * (4 * zz - xx - yy),
            c3[5] * z * (xx - yy), c3[6] * x * (xx - 3 * yy)]
    if not isinstance(dirs, np.ndarray):  # torch tensors (autograd in the tests)
        import torch
        return torch.stack(cols, dim=1)
    return np.stack(cols, axis=1)


def large(seed=3, n=1_000_000, width=1920, height=1080, n_views=64):
    """Config 3: N=1M, 16 anisotropic clusters + 10% uniform background,
    log-scales ~ N(log 0.01, 0.5), kappa ~ LogNormal(0,1), SH-3 colours
    (DC ~ U(0,1), rest ~ N(0, 0.1)), 64 hemisphere cameras at 1920x1080."""
    rng_c = make_rng(seed, 10)
    centres = rng_c.uniform(-2.0, 2.0, (16, 3))
    rots = quat_rotmats(random_unit_quats(rng_c, 16))
    sd = rng_c.uniform(0.1, 0.5, (16, 3))
    n_bg = n // 10
    n_cl = n - n_bg
    rng = make_rng(seed, 0)
    which = rng.integers(0, 16, n_cl)
    local = rng.standard_normal((n_cl, 3)) * sd[which]
    pts = centres[which] + np.einsum("nij,nj->ni", rots[which], local)
    bgp = rng.uniform(-3.0, 3.0, (n_bg, 3))
    means = np.concatenate([pts, bgp], axis=0)
    scales = np.exp(make_rng(seed, 1).normal(math.log(0.01), 0.5, (n, 3)))
    quats = random_unit_quats(make_rng(seed, 2), n)
    kappa = make_rng(seed, 3).lognormal(0.0, 1.0, n)
    sh = make_rng(seed, 4).normal(0.0, 0.1, (n, 16, 3))
    sh[:, 0, :] = make_rng(seed, 5).uniform(0.0, 1.0, (n, 3))
    cams = [look_at(6.0 * d, [0.0, 0.0, 0.0], width=width, height=height, fov_x_deg=60.0)
            for d in fibonacci_dirs(n_views, hemisphere=True, min_elev_deg=10.0, max_elev_deg=70.0)]
    scene = _finish(means, scales, quats, kappa, sh[:, 0, :], sh=sh)
    return Config("large", scene, cams, seed,
                  description=f"config 3: N={n}, {width}x{height}, {n_views} views, SH-3")


def _frame_from_normal(nrm):
    """Quaternion (w,x,y,z) rotating local z onto each normal."""
    z = np.array([0.0, 0.0, 1.0])
    axis = np.cross(np.broadcast_to(z, nrm.shape), nrm)
    s = np.linalg.norm(axis, axis=1)
    c = nrm[:, 2]
    half = 0.5 * np.arctan2(s, c)
    axis = np.where(s[:, None] > 1e-12, axis / np.maximum(s, 1e-12)[:, None], np.array([1.0, 0.0, 0.0]))
    return np.concatenate([np.cos(half)[:, None], np.sin(half)[:, None] * axis], axis=1)


def opaque(seed=4, n=500_000, size=1024, n_views=32):
    """Config 4: flattened disks (thin axis 1e-3 along the surface normal,
    others 0.02) on a unit sphere and a torus (R=1.5, r=0.3), kappa ~ U(20,200)."""
    rng = make_rng(seed, 0)
    n_s = n // 2
    n_t = n - n_s
    p = rng.standard_normal((n_s, 3))
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    nrm_s = p.copy()
    u = rng.uniform(0.0, 2 * math.pi, n_t)
    v = rng.uniform(0.0, 2 * math.pi, n_t)
    R, r = 1.5, 0.3
    tor = np.stack([(R + r * np.cos(v)) * np.cos(u), r * np.sin(v), (R + r * np.cos(v)) * np.sin(u)], axis=1)
    nrm_t = np.stack([np.cos(v) * np.cos(u), np.sin(v), np.cos(v) * np.sin(u)], axis=1)
    means = np.concatenate([p, tor])
    nrm = np.concatenate([nrm_s, nrm_t])
    scales = np.empty((n, 3))
    scales[:, :2] = 0.02
    scales[:, 2] = 1e-3
    quats = _frame_from_normal(nrm)
    kappa = make_rng(seed, 3).uniform(20.0, 200.0, n)
    colors = make_rng(seed, 4).uniform(0.0, 1.0, (n, 3))
    cams = [look_at(4.0 * d, [0.0, 0.0, 0.0], width=size, height=size, fov_x_deg=60.0)
            for d in fibonacci_dirs(n_views)]
    return Config("opaque", _finish(means, scales, quats, kappa, colors), cams, seed,
                  description=f"config 4: N={n}, {size}x{size}, {n_views} views, kappa U(20,200)")


def tomography(seed=5, n=200_000, size=512, n_views=180, extent=1.6):
    """Config 5: isotropic log-scales U(log .01, log .05), kappa ~ U(0.1, 2),
    180 parallel-beam views over [0, pi) about world y, 512x512 detector."""
    means = make_rng(seed, 0).uniform(-1.0, 1.0, (n, 3))
    s = np.exp(make_rng(seed, 1).uniform(math.log(0.01), math.log(0.05), n))
    scales = np.repeat(s[:, None], 3, axis=1)
    quats = np.tile(np.array([1.0, 0.0, 0.0, 0.0]), (n, 1))
    kappa = make_rng(seed, 3).uniform(0.1, 2.0, n)
    colors = np.zeros((n, 3))
    cams = []
    for k in range(n_views):
        ang = math.pi * k / n_views
        pos = 4.0 * np.array([math.sin(ang), 0.0, math.cos(ang)])
        cams.append(look_at(pos, [0.0, 0.0, 0.0], width=size, height=size, fov_x_deg=30.0))
    return Config("tomography", _finish(means, scales, quats, kappa, colors), cams, seed,
                  tomography=True, parallel=True, extent=extent,
                  description=f"config 5: N={n}, {size}x{size}, {n_views} parallel views")


def quat_rotmats(q):
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    return np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                     2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                     2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
                    axis=1).reshape(-1, 3, 3)


BY_NAME = {"tiny": tiny, "medium": medium, "large": large, "opaque": opaque,
           "tomography": tomography}
