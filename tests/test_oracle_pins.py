"""Pin the CPU oracle (oracle/volgauss_oracle.py) against golden vectors the
reference itself produced (tests/golden/make_golden.py), plus the reference's
own known-answer tests for this path.  CPU only."""

from __future__ import annotations

import math
import os

import numpy as np
import pytest

from conftest import RASTER_CASES, TOMO_CASES, case_flags, golden_lists, load_case
from oracle import volgauss_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

GRAD_FIELDS = ["d_means", "d_scales", "d_rotations", "d_thetas", "d_colors", "d_background",
               "d_kappas"]


def close(a, b, rtol=1e-9, atol=1e-12):
    a, b = np.asarray(a, float), np.asarray(b, float)
    scale = max(1.0, float(np.max(np.abs(b)))) if b.size else 1.0
    assert a.shape == b.shape
    np.testing.assert_allclose(a, b, rtol=rtol, atol=atol * scale)


@pytest.mark.parametrize("name", RASTER_CASES)
def test_tile_lists_match_reference(name):
    scene, cam, d = load_case(name)
    prep = O.prepare(scene, cam, alpha_cut=case_flags(d)["alpha_cut"])
    ref = golden_lists(d)
    got = prep.lists()
    assert len(got) == len(ref)
    for t, (g, r) in enumerate(zip(got, ref)):
        assert np.array_equal(g, r), f"tile {t}"
    close(prep.radius, d["radius"], rtol=1e-13)
    close(prep.mean2d, d["mean2d"], rtol=1e-13)
    assert np.array_equal(prep.valid, d["valid"])


@pytest.mark.parametrize("name", RASTER_CASES)
def test_render_matches_reference(name):
    scene, cam, d = load_case(name)
    img = O.render(scene, cam, **case_flags(d))
    close(img.color, d["color"])
    close(img.final_transmittance, d["final_transmittance"])
    assert np.array_equal(img.n_contrib, d["n_contrib"])


@pytest.mark.parametrize("name", [c for c in RASTER_CASES])
def test_backward_matches_reference(name):
    scene, cam, d = load_case(name)
    if "d_color" not in d:
        pytest.skip("no backward in this case")
    g = O.backward(scene, cam, d["d_color"], d_transmittance=d.get("d_transmittance"),
                   **case_flags(d))
    for f in GRAD_FIELDS:
        close(getattr(g, f), d[f"bwd_{f}"], rtol=1e-8, atol=1e-11)
    assert np.array_equal(g.visible, d["bwd_visible"])


@pytest.mark.parametrize("name", TOMO_CASES)
def test_tomo_matches_reference(name):
    scene, cam, d = load_case(name)
    prep = O.tomo_prepare(scene, cam)
    for g_, r_ in zip(prep.lists(), golden_lists(d, "tomo_tiles")):
        assert np.array_equal(g_, r_)
    close(O.tomo_forward(scene, cam, prep=prep), d["tomo_image"])
    g = O.tomo_backward(scene, cam, d["tomo_weights"], prep=prep)
    for f in ["d_means", "d_scales", "d_rotations", "d_thetas", "d_kappas", "d_colors"]:
        close(getattr(g, f), d[f"tomo_{f}"], rtol=1e-8, atol=1e-11)
    assert np.array_equal(g.visible, d["tomo_visible"])


def test_empty_scene():
    scene, cam, d = load_case("empty")
    img = O.render(scene, cam)
    assert np.allclose(img.color, d["background"])
    assert np.all(img.final_transmittance == 1.0) and np.all(img.n_contrib == 0)


def test_known_answers():
    # kappa(theta=0.5, s=1) = -ln(0.505); T(kappa=1, peak=1, beta=1) = exp(-sqrt(2 pi))
    # (reference tests/test_core.py:83-91, 184-191)
    assert O.kappa_of(np.array([0.5]), np.ones((1, 3)))[0] == pytest.approx(-math.log(0.505), rel=1e-14)
    assert O.kappa_of(np.array([1.0]), np.ones((1, 3)))[0] == pytest.approx(4.605170, rel=1e-6)
    assert math.exp(-O.SQRT_2PI) == pytest.approx(0.081543, abs=1e-6)
    # tomography centre ray of a unit Gaussian is sqrt(2 pi) (test_tomo.py:35-45)
    scene, cam, d = load_case("tomo_unit")
    # (theta is stored as float32, so kappa is 1 only to ~1e-7)
    centre = O.tomo_forward(scene, cam)[16, 16]
    assert centre == pytest.approx(O.SQRT_2PI, rel=1e-6)
    assert centre == pytest.approx(d["tomo_image"][16, 16], rel=1e-13)


def test_parallel_beam_matches_quadrature():
    """The orthographic projector has no reference counterpart; pin it with a
    trapezoid integral of the mixture density along each ray (the method of
    the reference's tests/test_tomo.py:14-25, 47-54)."""
    from paper_2412_03378_b200.camera import look_at
    rng = np.random.default_rng(3)
    n = 6
    scene = type("S", (), {})()
    scene.means = rng.uniform(-0.5, 0.5, (n, 3))
    scene.scales = rng.uniform(0.05, 0.25, (n, 3))
    q = rng.standard_normal((n, 4))
    scene.rotations = q
    scene.thetas = rng.uniform(0.1, 0.8, n)
    scene.colors = np.zeros((n, 3))
    scene.background = np.zeros(3)
    cam = look_at([1.0, 0.5, -4.0], [0, 0, 0], width=12, height=10, fov_x_deg=30.0)
    extent = 1.2
    img = O.tomo_forward(scene, cam, parallel=True, extent=extent)
    prec = O.sandwich(O.quat_to_rotmat(q), 1.0 / scene.scales ** 2)
    kap = O.kappa_of(scene.thetas, scene.scales)
    for row, col in [(0, 0), (5, 6), (9, 11), (3, 2)]:
        org, f = O.parallel_pixel_rays(cam, np.array([row]), np.array([col]), extent)
        t = np.linspace(-8.0, 8.0, 200_001)
        pts = org[0][None] + t[:, None] * f[0][None]
        dens = np.zeros_like(t)
        for i in range(n):
            dd = pts - scene.means[i]
            dens += kap[i] * np.exp(-0.5 * np.einsum("ti,ij,tj->t", dd, prec[i], dd))
        assert img[row, col] == pytest.approx(np.trapezoid(dens, t), rel=1e-6, abs=1e-12)


def test_fp32_key_order_differs_only_on_ties():
    """The device sorts 32-bit depth keys; on the golden cases the fp32-key
    order equals the fp64 order except where fp32 depths tie."""
    for name in ["tiny", "mini_opaque", "ragged"]:
        scene, cam, d = load_case(name)
        p64 = O.prepare(scene, cam, alpha_cut=case_flags(d)["alpha_cut"])
        p32 = O.prepare(scene, cam, alpha_cut=case_flags(d)["alpha_cut"], key_dtype=np.float32)
        k32 = p64.depth.astype(np.float32)
        for a, b in zip(p64.lists(), p32.lists()):
            assert np.array_equal(np.sort(a), np.sort(b))
            diff = a != b
            if diff.any():
                assert np.all(np.diff(k32[b]) >= 0)
                assert set(a[diff]) == set(b[diff])
                assert len(np.unique(k32[a[diff]])) < diff.sum()


@pytest.mark.parametrize("name", ["tiny", "ragged"])
def test_gamma_sort_matches_reference(name):
    """sort_by='gamma' (raster.py:291-312): lists re-sorted by gamma along each
    tile's central ray, and the image / gradients composited in that order
    (golden: tests/golden/make_golden_gamma.py)."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "gamma.npz"))
    scene, cam, d = load_case(name)
    prep = O.prepare(scene, cam, sort_by="gamma")
    off = g[f"{name}_offsets"]
    ref = [g[f"{name}_prims"][off[t]:off[t + 1]] for t in range(len(off) - 1)]
    for t, (a, b) in enumerate(zip(prep.lists(), ref)):
        assert np.array_equal(a, b), f"tile {t}"
    out = O.render(scene, cam, prep=prep)
    close(out.color, g[f"{name}_color"], rtol=1e-10, atol=1e-13)
    close(out.final_transmittance, g[f"{name}_T"], rtol=1e-10, atol=1e-13)
    gr = O.backward(scene, cam, g[f"{name}_dcolor"], prep=prep)
    for f in ("d_means", "d_scales", "d_rotations", "d_thetas", "d_colors", "d_background"):
        close(getattr(gr, f), g[f"{name}_{f}"], rtol=1e-8, atol=1e-11)


@pytest.mark.parametrize("name", ["tiny", "ragged"])
def test_splat_mode_matches_reference(name):
    """mode='splat' (the EWA comparator, raster.py:353-361, grad.py:170-177,
    262-302): bin radii, tile lists, image, n_contrib and every gradient
    (golden: tests/golden/make_golden_splat.py)."""
    import os
    from types import SimpleNamespace
    from oracle import splat_oracle as SO
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "splat.npz"))
    scene, cam, d = load_case(name)
    scene = SimpleNamespace(means=scene.means, scales=scene.scales, rotations=scene.rotations,
                            thetas=scene.thetas, colors=scene.colors, background=scene.background,
                            splat_opacities=g[f"{name}_opac"])
    prep = SO.prepare(scene, cam)
    close(prep.radius, g[f"{name}_radius"], rtol=1e-13)
    off = g[f"{name}_offsets"]
    for t in range(len(off) - 1):
        assert np.array_equal(prep.tile_ids(t), g[f"{name}_prims"][off[t]:off[t + 1]]), t
    out = SO.render(scene, cam, prep=prep)
    close(out.color, g[f"{name}_color"], rtol=1e-10, atol=1e-13)
    close(out.final_transmittance, g[f"{name}_T"], rtol=1e-10, atol=1e-13)
    assert np.array_equal(out.n_contrib, g[f"{name}_ncontrib"])
    gr = SO.backward(scene, cam, g[f"{name}_dcolor"], prep=prep)
    for f in ("d_means", "d_scales", "d_rotations", "d_colors", "d_background", "d_splat_opacities"):
        close(getattr(gr, f), g[f"{name}_{f}"], rtol=1e-8, atol=1e-11)
    assert np.array_equal(gr.visible, g[f"{name}_visible"])
    assert not np.any(g[f"{name}_d_thetas"])


def test_voxelize_oracle_pinned_to_reference():
    """oracle.voxelize equals the reference's tomo.voxelize bit for bit
    (tests/golden/make_golden_recon.py: rotated anisotropic primitives,
    anisotropic resolution, a box the primitives partly leave)."""
    d = np.load(os.path.join(GOLDEN, "recon.npz"))
    v = O.voxelize(d["vox_means"], d["vox_scales"], d["vox_rotations"], d["vox_thetas"],
                   d["vox_values"].shape, d["vox_bmin"], d["vox_bmax"])
    assert np.array_equal(v, d["vox_values"])
    # boxes the reference accepts unchecked: flat (zero spacing) and reversed
    for tag in ("flat", "reversed"):
        v = O.voxelize(d["vox_means"], d["vox_scales"], d["vox_rotations"], d["vox_thetas"],
                       d[f"vox_{tag}_values"].shape, d[f"vox_{tag}_bmin"], d[f"vox_{tag}_bmax"])
        assert np.array_equal(v, d[f"vox_{tag}_values"]), tag


def test_volume_metrics_match_reference():
    """metrics.psnr_volume / ssim_volume reproduce the reference's numbers on
    the golden reconstruction grid."""
    from paper_2412_03378_b200 import metrics
    d = np.load(os.path.join(GOLDEN, "recon.npz"))
    assert metrics.psnr_volume(d["grid"], d["ref_grid"]) == pytest.approx(float(d["psnr_3d"]), rel=1e-12)
    assert metrics.ssim_volume(d["grid"], d["ref_grid"]) == pytest.approx(float(d["ssim_3d"]), rel=1e-12)
