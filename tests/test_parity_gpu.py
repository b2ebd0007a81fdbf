"""GPU parity: the sm_100a path (through the C ABI) against the golden vectors
the reference produced and against the pinned CPU oracle.

Contract (tests/parity.py): tile lists and their order bit-exact (order
defined with float32 depth keys); images and gradients within
1e-4 absolute (scaled by the field magnitude for gradients) + 1e-3 relative,
with any out-of-tolerance pixel attributed to a float32/float64 threshold
flip.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import RASTER_CASES, TOMO_CASES, case_flags, cuda_available, golden_lists, load_case
from oracle import volgauss_oracle as O
from parity import (check_field, check_image, device_knife_mask, image_mismatch, knife_cap,
                    near_threshold)

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

GRAD_FIELDS = ["d_means", "d_scales", "d_rotations", "d_thetas", "d_colors", "d_kappas"]


def vg():
    import paper_2412_03378_b200 as m
    return m


def test_library_is_native():
    """The product path is the in-tree .so, not a fallback."""
    import paper_2412_03378_b200._lib as L
    lib = L.load()
    assert lib._name.endswith("libvolgauss_b200.so")
    ctx = L.Context()
    assert ctx.launches() == 0


@pytest.mark.parametrize("name", RASTER_CASES)
def test_tile_lists_bit_exact(name):
    scene, cam, d = load_case(name)
    flags = case_flags(d)
    prep = vg().prepare(scene, cam, alpha_cut=flags["alpha_cut"])
    got = prep.grid.tiles
    ref64 = golden_lists(d)
    ref32 = O.prepare(scene, cam, alpha_cut=flags["alpha_cut"], key_dtype=np.float32).lists()
    assert len(got) == len(ref32)
    ties = 0
    for t, (g, r32, r64) in enumerate(zip(got, ref32, ref64)):
        assert np.array_equal(g, r32), f"tile {t}: order differs from lexsort(prim, f32 depth, tile)"
        assert np.array_equal(np.sort(g), np.sort(r64)), f"tile {t}: set differs from reference"
        ties += int(np.sum(g != r64))
    # any difference from the float64 order is a float32 depth tie
    assert ties <= 2 * max(1, len(scene.means) // 500)


@pytest.mark.parametrize("name", RASTER_CASES)
def test_render_matches_reference(name):
    scene, cam, d = load_case(name)
    flags = case_flags(d)
    dprep = vg().prepare(scene, cam, alpha_cut=flags["alpha_cut"])
    out = vg().render(scene, cam, **flags, prep=dprep)
    prep = O.prepare(scene, cam, alpha_cut=flags["alpha_cut"])
    # pixels whose float32 counts differ from the oracle's (each explained by
    # an entry at a threshold), plus alpha-clamp edges
    knife = device_knife_mask(prep, scene, flags, out.n_contrib, dprep.n_active())
    check_image(out.color, d["color"], prep, scene, flags, f"{name} color", knife=knife)
    check_image(out.final_transmittance, d["final_transmittance"], prep, scene, flags, f"{name} T",
                knife=knife)
    if flags["alpha_cut"] > 0:
        diff = np.argwhere(out.n_contrib != d["n_contrib"])
        bad = [tuple(x) for x in diff if not knife[x[0], x[1]]]
        assert not bad, f"n_contrib differs at {bad[:5]}"


@pytest.mark.parametrize("name", [c for c in RASTER_CASES])
def test_backward_matches_reference(name):
    scene, cam, d = load_case(name)
    if "d_color" not in d:
        pytest.skip("no backward in this case")
    flags = case_flags(d)
    dc, dt = d["d_color"], d.get("d_transmittance")
    ref = {f: d[f"bwd_{f}"] for f in GRAD_FIELDS + ["d_background", "visible"]}
    prep = O.prepare(scene, cam, alpha_cut=flags["alpha_cut"])
    dprep = vg().prepare(scene, cam, alpha_cut=flags["alpha_cut"])
    out = vg().render(scene, cam, **flags, prep=dprep)
    knife = device_knife_mask(prep, scene, flags, out.n_contrib, dprep.n_active())
    knife_cap(int(knife.sum()), knife.size, f"{name} backward")
    if knife.any():
        # float32/float64 threshold flips: take those pixels out of the
        # upstream gradient on both sides (oracle is pinned to the reference)
        dc = dc * ~knife[..., None]
        dt = None if dt is None else dt * ~knife
        g64 = O.backward(scene, cam, dc, d_transmittance=dt, prep=prep, **flags)
        ref = {f: getattr(g64, f) for f in ref}
    g = vg().backward(scene, cam, dc, d_transmittance=dt, **flags, prep=dprep)
    for f in GRAD_FIELDS:
        check_field(getattr(g, f), ref[f], f"{name} {f}")
    check_field(g.d_background, ref["d_background"], f"{name} d_background")
    assert np.array_equal(g.visible, ref["visible"])


@pytest.mark.parametrize("name", TOMO_CASES)
def test_tomo_matches_reference(name):
    scene, cam, d = load_case(name)
    img = vg().tomo_forward(scene, cam)
    check_field(img, d["tomo_image"], f"{name} tomo image", atol=1e-4, rtol=1e-3)
    g = vg().tomo_backward(scene, cam, d["tomo_weights"])
    for f in GRAD_FIELDS:
        check_field(getattr(g, f), d[f"tomo_{f}"], f"{name} tomo {f}")
    assert np.array_equal(g.visible, d["tomo_visible"])


def test_empty_scene_and_background():
    scene, cam, d = load_case("empty")
    out = vg().render(scene, cam)
    assert np.allclose(out.color, d["background"])
    assert np.all(out.final_transmittance == 1.0) and np.all(out.n_contrib == 0)
    dc = np.random.default_rng(0).uniform(-1, 1, (cam.height, cam.width, 3))
    g = vg().backward(scene, cam, dc)
    np.testing.assert_allclose(g.d_background, dc.reshape(-1, 3).sum(axis=0), rtol=1e-5, atol=1e-5)


def test_nan_upstream_raises():
    scene, cam, d = load_case("tiny")
    dc = np.zeros((cam.height, cam.width, 3))
    dc[4, 4, 0] = np.nan
    with pytest.raises(ValueError):
        vg().backward(scene, cam, dc)


def test_fused_l2_equals_explicit():
    """vg_render_backward_l2 == loss_and_grad(l2) + vg_render_backward."""
    import torch
    from paper_2412_03378_b200 import engine
    scene, cam, d = load_case("tiny")
    eng = engine.Engine()
    ds = eng.upload(scene)
    tgt = torch.tensor(d["target"], dtype=torch.float32, device="cuda")
    eng.prepare(ds, cam)
    color, tfin, _ = eng.forward()
    b1 = eng.new_grads(ds)
    loss = eng.backward_l2(color, tfin, tgt, b1)
    ref_loss, dimg = vg().loss_and_grad(color.double().cpu().numpy(), d["target"], vg().LossSpec("l2"))
    assert float(loss) == pytest.approx(ref_loss, rel=1e-5)
    g2 = vg().backward(scene, cam, dimg)
    for f in GRAD_FIELDS:
        check_field(b1.views[f].cpu().numpy(), getattr(g2, f), f"fused {f}", rtol=1e-4, atol=1e-6)


def test_parallel_beam_matches_oracle():
    rng = np.random.default_rng(11)
    n = 300
    from types import SimpleNamespace
    scene = SimpleNamespace(means=rng.uniform(-1, 1, (n, 3)).astype(np.float32).astype(np.float64),
                            scales=np.repeat(np.exp(rng.uniform(np.log(0.02), np.log(0.1), (n, 1))), 3, 1).astype(np.float32).astype(np.float64),
                            rotations=np.tile([1.0, 0, 0, 0], (n, 1)),
                            thetas=rng.uniform(0.05, 0.9, n).astype(np.float32).astype(np.float64),
                            colors=np.zeros((n, 3)), background=np.zeros(3))
    cam = vg().look_at([4.0 * np.sin(0.3), 0.0, 4.0 * np.cos(0.3)], [0, 0, 0], width=40, height=36,
                       fov_x_deg=30.0)
    img = vg().tomo_forward(scene, cam, parallel=True, extent=1.6)
    ref = O.tomo_forward(scene, cam, parallel=True, extent=1.6)
    check_field(img, ref, "parallel image")
    w = rng.uniform(0.1, 1.0, (36, 40))
    g = vg().tomo_backward(scene, cam, w, parallel=True, extent=1.6)
    rg = O.tomo_backward(scene, cam, w, parallel=True, extent=1.6)
    for f in ["d_means", "d_scales", "d_rotations", "d_thetas", "d_kappas"]:
        check_field(getattr(g, f), getattr(rg, f), f"parallel {f}")


def test_multiview_accumulation_and_order_independence():
    """Summing per-view grads with accumulate=True equals the sum of
    separate backward calls (the view-sharded step relies on it)."""
    import torch
    from paper_2412_03378_b200 import configs, engine
    cfg = configs.medium(n=3000, size=64, n_views=3)
    eng = engine.Engine()
    ds = eng.upload(cfg.scene)
    acc = eng.new_grads(ds)
    parts = []
    for v, cam in enumerate(cfg.cameras):
        tgt = torch.tensor(cfg.target(v, (64, 64, 3)), device="cuda")
        eng.prepare(ds, cam)
        color, tfin, _ = eng.forward()
        eng.backward_l2(color, tfin, tgt, acc, accumulate=v > 0)
        one = eng.new_grads(ds)
        eng.prepare(ds, cam)
        color, tfin, _ = eng.forward()
        eng.backward_l2(color, tfin, tgt, one)
        parts.append(one.flat.clone())
    total = sum(parts)
    check_field(acc.flat.cpu().numpy(), total.cpu().numpy(), "accumulated grads", rtol=1e-4, atol=1e-6)
    # the deferred multi-view step (one float64 parameter-chain pass per step)
    from paper_2412_03378_b200.multiview import ViewShardedStep
    targets = {v: torch.tensor(cfg.target(v, (64, 64, 3)), device="cuda") for v in range(3)}
    step = ViewShardedStep(eng, ds, cfg.cameras, targets)
    step()
    check_field(step.grads.flat.cpu().numpy(), total.cpu().numpy(), "deferred step grads",
                rtol=1e-4, atol=1e-6)
    step()   # a second step starts from clean accumulators
    check_field(step.grads.flat.cpu().numpy(), total.cpu().numpy(), "second step grads",
                rtol=1e-4, atol=1e-6)


def _f64_scene(s, colors=True):
    from types import SimpleNamespace
    return SimpleNamespace(means=s.means.astype(np.float64), scales=s.scales.astype(np.float64),
                           rotations=s.rotations.astype(np.float64),
                           thetas=s.thetas.astype(np.float64),
                           colors=s.colors.astype(np.float64), background=np.zeros(3))


def _tile_mask(oprep, tiles, H, W):
    mask = np.zeros((H, W), dtype=bool)
    for t in tiles:
        ty, tx = divmod(t, oprep.tiles_x)
        mask[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = True
    return mask


def _full_size_check(scene, cam, n_random=5, seed=5, n_busy=3):
    """Every tile list bit-exact against the oracle's float32-key order; a
    seeded sample of tiles (incl. the three heaviest) rendered and
    back-propagated against the float64 oracle (d_color vanishes outside the
    sampled tiles and on knife-edge pixels, on both sides)."""
    prep = vg().prepare(scene, cam)
    oprep = O.prepare(scene, cam, key_dtype=np.float32)
    assert prep.pair_count() == len(oprep.pair_prim)
    prims, offs = prep.tile_lists_device()
    assert np.array_equal(offs.cpu().numpy(), oprep.tile_start)
    assert np.array_equal(prims.cpu().numpy(), oprep.pair_prim)
    out = vg().render(scene, cam, prep=prep)
    rng = np.random.default_rng(seed)
    busy = np.argsort(np.diff(oprep.tile_start))[len(oprep.tile_start) - 1 - n_busy:]
    tiles = sorted(set(busy.tolist()) |
                   set(rng.integers(0, oprep.tiles_x * oprep.tiles_y, n_random).tolist()))
    ref = O.render(scene, cam, prep=oprep, tiles=tiles)
    mask = _tile_mask(oprep, tiles, cam.height, cam.width)
    npx = int(mask.sum())
    knife = device_knife_mask(oprep, scene, {}, out.n_contrib, prep.n_active(), tiles=tiles)
    check_image(np.where(mask[..., None], out.color, 0), np.where(mask[..., None], ref.color, 0),
                oprep, scene, {}, "color", n_px=npx, knife=knife)
    check_image(np.where(mask, out.final_transmittance, 0), np.where(mask, ref.final_transmittance, 0),
                oprep, scene, {}, "T", n_px=npx, knife=knife)
    knife_cap(int(knife.sum()), npx, "sampled tiles backward")
    dc = rng.uniform(-1, 1, (cam.height, cam.width, 3)) * (mask & ~knife)[..., None]
    g = vg().backward(scene, cam, dc, prep=prep)
    rg = O.backward(scene, cam, dc, prep=oprep, tiles=tiles)
    for f in GRAD_FIELDS:
        check_field(getattr(g, f), getattr(rg, f), f)
    # the atomic-mode backward on the same context: the earlier forwards left
    # depth statistics, so a tail-bound view now runs the deep-tile forward
    # and the segmented backward
    ga = vg().backward(scene, cam, dc, prep=prep, deterministic=False)
    plan = _segments(prep.ctx)
    for f in GRAD_FIELDS:
        check_field(getattr(ga, f), getattr(rg, f), f"atomic {f}")
    return plan


def test_full_size_large_view_tiles_and_sampled_pixels():
    """Config 3 (N=1M, 1920x1080), first view."""
    from paper_2412_03378_b200 import configs
    cfg = configs.large()
    _full_size_check(_f64_scene(cfg.scene), cfg.cameras[0])


def test_full_size_medium_all_views():
    """Config 2 (BASELINE configs[1]: N=100k, 8 views at 800x800) at full
    size: every view's tile lists bit-exact, and per view the heaviest tile
    plus two seeded tiles rendered and back-propagated against the float64
    oracle (raster.py:410-439, grad.py:107-259)."""
    from paper_2412_03378_b200 import configs
    cfg = configs.medium()
    assert len(cfg.cameras) == 8 and cfg.cameras[0].width == 800
    scene = _f64_scene(cfg.scene)
    for v, cam in enumerate(cfg.cameras):
        _full_size_check(scene, cam, n_random=2, seed=100 + v, n_busy=1)


def test_full_size_opaque_view():
    """Config 4 (N=500k flattened disks, kappa 20-200, 1024x1024): early
    termination on most pixels; three views (a side, top and oblique one)."""
    from paper_2412_03378_b200 import configs
    cfg = configs.opaque()
    scene = _f64_scene(cfg.scene)
    plans = [_full_size_check(scene, cfg.cameras[v], n_random=3, seed=seed, n_busy=2)
             for v, seed in ((3, 7), (11, 8), (26, 9))]
    # the segmented backward ran at full size on the tail-bound views (the
    # drop-in backward's forward counts n_contrib, so it never takes the
    # deep-tile variant -- that is the engine's training forward)
    assert sum(p[0] & 1 for p in plans) >= 2, plans


def test_full_size_tomography_parallel_view():
    """Config 5 (N=200k, 512x512 parallel-beam detector): tile lists exact,
    sampled tiles of the line-integral image and the masked adjoint against
    the float64 oracle."""
    from paper_2412_03378_b200 import configs
    cfg = configs.tomography()
    scene = _f64_scene(cfg.scene)
    cam = cfg.cameras[17]
    prep = vg().tomo_prepare(scene, cam, parallel=True, extent=cfg.extent)
    oprep = O.tomo_prepare(scene, cam, parallel=True, extent=cfg.extent, key_dtype=np.float32)
    prims, offs = prep.tile_lists_device()
    assert np.array_equal(offs.cpu().numpy(), oprep.tile_start)
    assert np.array_equal(np.sort(prims.cpu().numpy()), np.sort(oprep.pair_prim))
    img = vg().tomo_forward(scene, cam, prep=prep)
    rng = np.random.default_rng(3)
    tiles = sorted(set(rng.integers(0, oprep.tiles_x * oprep.tiles_y, 6).tolist()) |
                   set(np.argsort(np.diff(oprep.tile_start))[-2:].tolist()))
    ref = O.tomo_forward(scene, cam, prep=oprep, tiles=tiles)
    mask = _tile_mask(oprep, tiles, cam.height, cam.width)
    check_field(np.where(mask, img, 0), np.where(mask, ref, 0), "tomo image")
    w = rng.uniform(0.1, 1.0, (cam.height, cam.width)) * mask
    g = vg().tomo_backward(scene, cam, w, prep=prep)
    rg = O.tomo_backward(scene, cam, w, prep=oprep, tiles=tiles)
    for f in ["d_means", "d_scales", "d_rotations", "d_thetas", "d_kappas"]:
        check_field(getattr(g, f), getattr(rg, f), f"tomo {f}")


def test_more_than_65536_tiles():
    """4400x4000 = 68750 tiles (275 tile columns, 250 rows in the span
    binning): lists and sampled pixels still match."""
    from paper_2412_03378_b200 import configs
    from paper_2412_03378_b200.camera import look_at
    cfg = configs.medium(n=4000, size=64, n_views=1)
    cam = look_at([0.0, 1.0, -5.0], [0, 0, 0], width=4400, height=4000, fov_x_deg=60.0)
    _full_size_check(_f64_scene(cfg.scene), cam, n_random=4, seed=11)


def test_forward_is_deterministic():
    scene, cam, d = load_case("mini_opaque")
    a = vg().render(scene, cam)
    b = vg().render(scene, cam)
    assert np.array_equal(a.color, b.color)
    assert np.array_equal(a.final_transmittance, b.final_transmittance)
    assert np.array_equal(a.n_contrib, b.n_contrib)


def test_degenerate_inputs():
    """Scales below the 1e-7 floor (dead scale gradients), unnormalised
    quaternions, a primitive straddling the near plane and one covering the
    whole screen: lists, images and gradients still match the oracle."""
    from types import SimpleNamespace
    rng = np.random.default_rng(2)
    n = 40
    means = rng.uniform(-0.8, 0.8, (n, 3))
    scales = rng.uniform(0.05, 0.3, (n, 3))
    scales[0, 1] = 1e-9                      # floored, dead gradient (grad.py:257)
    quats = rng.standard_normal((n, 4)) * 3.0  # unnormalised
    means[1] = [0.0, 0.0, -2.995]            # 5 mm in front of the camera (z_near 0.01)
    scales[2] = [2.5, 2.5, 2.5]              # covers every tile
    means[2] = [0.0, 0.0, 0.5]
    f32 = lambda a: a.astype(np.float32).astype(np.float64)
    scene = SimpleNamespace(means=f32(means), scales=f32(scales), rotations=f32(quats),
                            thetas=f32(rng.uniform(0.05, 0.6, n)), colors=f32(rng.uniform(0, 1, (n, 3))),
                            background=np.array([0.1, 0.2, 0.3]))
    cam = vg().look_at([0, 0, -3.0], [0, 0, 0], width=50, height=34, fov_x_deg=60.0)
    prep = vg().prepare(scene, cam)
    ref_lists = O.prepare(scene, cam, key_dtype=np.float32).lists()
    for gl, rl in zip(prep.grid.tiles, ref_lists):
        assert np.array_equal(gl, rl)
    out = vg().render(scene, cam, prep=prep)
    ref = O.render(scene, cam)
    oprep = O.prepare(scene, cam)
    knife = device_knife_mask(oprep, scene, {}, out.n_contrib, prep.n_active())
    check_image(out.color, ref.color, oprep, scene, {}, "degenerate color", knife=knife)
    knife_cap(int(knife.sum()), knife.size, "degenerate backward")
    dc = rng.uniform(-1, 1, (34, 50, 3)) * ~knife[..., None]
    g = vg().backward(scene, cam, dc)
    rg = O.backward(scene, cam, dc)
    for f in GRAD_FIELDS:
        check_field(getattr(g, f), getattr(rg, f), f"degenerate {f}")
    assert g.d_scales[0, 1] == 0.0


@pytest.mark.parametrize("name", ["tiny", "mini_opaque", "large"])
def test_depth_sort_and_span_lists(name):
    """The hand-written onesweep depth sort (vg_radix.cu) and the span
    binning (vg_span.cu) give bit-exact tile lists and tile starts (many
    tiles of look-back, 68 x 120 tiles on the large config)."""
    if name == "large":
        from paper_2412_03378_b200 import configs
        cfg = configs.large()
        scene, cam = _f64_scene(cfg.scene), cfg.cameras[5]
        flags = {"alpha_cut": O.ALPHA_CUT}
    else:
        scene, cam, d = load_case(name)
        flags = case_flags(d)
    prep = vg().prepare(scene, cam, alpha_cut=flags["alpha_cut"])
    oprep = O.prepare(scene, cam, alpha_cut=flags["alpha_cut"], key_dtype=np.float32)
    prims, offs = prep.tile_lists_device()
    assert np.array_equal(offs.cpu().numpy(), oprep.tile_start)
    assert np.array_equal(prims.cpu().numpy(), oprep.pair_prim)


def sh_direction_grad(means, centre, sh, d_rgb):
    """d/dmeans of sum(d_rgb * RGB(dir)), RGB = sum_l b_l(dir) sh_l, dir =
    (mean - centre)/|.|: float64 torch autograd through configs.sh_basis's
    polynomial (an independent check of k_sh_pull's hand-written VJP)."""
    import torch
    from paper_2412_03378_b200 import configs
    m = torch.tensor(means, dtype=torch.float64, requires_grad=True)
    d = m - torch.tensor(np.asarray(centre, dtype=np.float64))
    d = d / d.norm(dim=1, keepdim=True)
    b = configs.sh_basis(d)
    rgb = torch.einsum("nl,nlc->nc", b, torch.tensor(sh, dtype=torch.float64))
    (rgb * torch.tensor(d_rgb, dtype=torch.float64)).sum().backward()
    return m.grad.numpy()


def test_sh_colour_and_deferred_pullback():
    """SH-3 colour (config 3's colour model; no reference counterpart, so the
    check is against the float64 oracle fed each view's evaluated RGB): the
    multi-view step's geometry gradients equal the sum of the per-view
    oracle gradients, and d_sh equals sum_v basis(d_v) x dL/dRGB_v (the
    deferred per-view slabs folded once per step over both pipelined
    contexts)."""
    import torch
    from types import SimpleNamespace
    from paper_2412_03378_b200 import configs
    from paper_2412_03378_b200.engine import Engine
    from paper_2412_03378_b200.multiview import ViewShardedStep
    cfg = configs.large(n=3000, width=96, height=64, n_views=5)
    s = cfg.scene
    means = s.means.astype(np.float64)
    sh = s.sh.astype(np.float64)
    eng = Engine()
    ds = eng.upload(s)
    targets = {v: torch.from_numpy(cfg.target(v, (64, 96, 3))).cuda() for v in range(5)}
    step = ViewShardedStep(eng, ds, cfg.cameras, targets)
    loss = float(step())
    g = step.grads.to_scene_grads("analytic", torch_out=False)
    tot = {f: 0.0 for f in ["d_means", "d_scales", "d_rotations", "d_thetas", "d_kappas"]}
    d_sh = np.zeros((len(means), 16, 3))
    ref_loss = 0.0
    for v, cam in enumerate(cfg.cameras):
        c = O.cam_center(cam)
        d = means - c
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        basis = configs.sh_basis(d)                                   # (N, 16)
        rgb = np.einsum("nl,nlc->nc", basis, sh)
        scene = SimpleNamespace(means=means, scales=s.scales.astype(np.float64),
                                rotations=s.rotations.astype(np.float64),
                                thetas=s.thetas.astype(np.float64), colors=rgb,
                                background=np.zeros(3))
        out = O.render(scene, cam)
        r = out.color - targets[v].cpu().numpy().astype(np.float64)
        ref_loss += float(np.sum(r * r))
        rg = O.backward(scene, cam, 2.0 * r / r.size)
        for f in tot:
            tot[f] = tot[f] + getattr(rg, f)
        d_sh += basis[:, :, None] * rg.d_colors[:, None, :]
        # the colour's view-direction dependence (torch float64 autograd)
        tot["d_means"] = tot["d_means"] + sh_direction_grad(means, c, sh, rg.d_colors)
    assert abs(loss - ref_loss) <= 1e-4 * ref_loss
    for f in tot:
        check_field(getattr(g, f), tot[f], f"sh step {f}")
    check_field(np.asarray(g.d_sh).reshape(-1, 48), d_sh.reshape(-1, 48), "d_sh")


@pytest.mark.parametrize("name", ["tiny", "ragged"])
def test_gamma_sort_lists_render_and_backward(name):
    """sort_by='gamma' (raster.py:291-312): device lists equal the reference's
    gamma lists (golden: make_golden_gamma.py); positions that differ must
    swap entries whose float64 gammas agree to 1e-12 relative (the device
    evaluates gamma in float64 with a different summation order).  Images
    and gradients composited in that order match the golden ones."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "gamma.npz"))
    scene, cam, d = load_case(name)
    prep = vg().prepare(scene, cam, sort_by="gamma")
    prims, offs = prep.tile_lists_device()
    prims, offs = prims.cpu().numpy(), offs.cpu().numpy()
    ref_off = g[f"{name}_offsets"]
    assert np.array_equal(offs, ref_off)
    ref = g[f"{name}_prims"]
    oprep = O.prepare(scene, cam)
    means = np.asarray(scene.means, dtype=np.float64)
    for t in range(len(ref_off) - 1):
        a, b = prims[ref_off[t]:ref_off[t + 1]], ref[ref_off[t]:ref_off[t + 1]]
        if np.array_equal(a, b):
            continue
        ids, gam = O.tile_gammas(oprep, means, t)
        gmap = dict(zip(ids.tolist(), gam.tolist()))
        ga, gb = np.array([gmap[i] for i in a]), np.array([gmap[i] for i in b])
        assert np.all(np.abs(ga - gb) <= 1e-12 * np.abs(gb) + 1e-300), f"tile {t}"
    out = vg().render(scene, cam, sort_by="gamma", prep=prep)
    gprep = O.prepare(scene, cam, sort_by="gamma")
    knife = device_knife_mask(gprep, scene, {}, out.n_contrib, prep.n_active())
    check_image(out.color, g[f"{name}_color"], gprep, scene, {}, f"{name} gamma color", knife=knife)
    fields = ("d_means", "d_scales", "d_rotations", "d_thetas", "d_colors", "d_background")
    dc = g[f"{name}_dcolor"]
    ref = {f: g[f"{name}_{f}"] for f in fields}
    knife_cap(int(knife.sum()), knife.size, f"{name} gamma backward")
    if knife.any():
        # threshold flips out of the upstream gradient on both sides (the
        # oracle is pinned to the reference's gamma render/backward)
        dc = dc * ~knife[..., None]
        g64 = O.backward(scene, cam, dc, prep=gprep)
        ref = {f: getattr(g64, f) for f in fields}
    gr = vg().backward(scene, cam, dc, sort_by="gamma", prep=prep)
    for f in fields:
        check_field(getattr(gr, f), ref[f], f"{name} gamma {f}")


def test_gamma_sort_long_lists_merge_path():
    """Tiles with lists longer than one 2048-entry shared-memory run take the
    global merge path; the result equals the oracle's stable gamma order."""
    from paper_2412_03378_b200 import configs
    cfg = configs.medium(n=20000, size=64, n_views=1)
    s = cfg.scene
    from types import SimpleNamespace
    scene = SimpleNamespace(means=s.means.astype(np.float64), scales=(s.scales * 6).astype(np.float32).astype(np.float64),
                            rotations=s.rotations.astype(np.float64), thetas=s.thetas.astype(np.float64),
                            colors=s.colors.astype(np.float64), background=np.zeros(3))
    cam = cfg.cameras[0]
    prep = vg().prepare(scene, cam, sort_by="gamma")
    prims, offs = prep.tile_lists_device()
    prims, offs = prims.cpu().numpy(), offs.cpu().numpy()
    oprep = O.prepare(scene, cam, key_dtype=np.float32, sort_by="gamma")
    assert np.array_equal(offs, oprep.tile_start)
    assert np.diff(offs).max() > 2 * 2048
    mism = np.flatnonzero(prims != oprep.pair_prim)
    assert mism.size <= 1e-4 * prims.size, mism.size


@pytest.mark.parametrize("name", ["mini_opaque", "tiny"])
def test_deterministic_backward_is_bitwise_reproducible(name):
    """deterministic=True (default of the drop-in backward): fixed-order sums
    (vg_det.cu), so repeated calls are bitwise identical -- the reference's
    thread-count invariance (grad.py:188-204) -- and agree with the
    atomic path within the parity tolerance."""
    scene, cam, d = load_case(name)
    rng = np.random.default_rng(3)
    dc = rng.uniform(-1, 1, (cam.height, cam.width, 3))
    a = vg().backward(scene, cam, dc)
    b = vg().backward(scene, cam, dc)
    fast = vg().backward(scene, cam, dc, deterministic=False)
    for f in GRAD_FIELDS + ["d_background"]:
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
        np.testing.assert_allclose(getattr(a, f), getattr(fast, f), rtol=1e-4,
                                   atol=1e-5 * max(1.0, float(np.abs(getattr(fast, f)).max())))
    assert np.array_equal(a.visible, fast.visible)


def test_deterministic_multiview_step_is_bitwise_reproducible():
    """The engine's multi-view step with deterministic=True: two runs give
    bitwise-identical flat gradient buffers and loss."""
    import torch
    from paper_2412_03378_b200 import configs
    from paper_2412_03378_b200.engine import Engine
    from paper_2412_03378_b200.multiview import ViewShardedStep
    cfg = configs.large(n=20000, width=160, height=96, n_views=4)
    eng = Engine(deterministic=True)
    ds = eng.upload(cfg.scene)
    targets = {v: torch.from_numpy(cfg.target(v, (96, 160, 3))).cuda() for v in range(4)}
    step = ViewShardedStep(eng, ds, cfg.cameras, targets)
    l1 = float(step())
    g1 = step.grads.flat.clone()
    l2 = float(step())
    g2 = step.grads.flat.clone()
    assert l1 == l2
    assert torch.equal(g1, g2)


@pytest.mark.parametrize("name", ["tiny", "ragged"])
def test_splat_mode_matches_reference(name):
    """mode='splat' (the EWA comparator): 3-sigma tile lists bit-exact, image
    and every gradient (incl. d_splat_opacities) against the reference's
    golden vectors (make_golden_splat.py); knife-edge pixels (alpha_raw at
    the cut or the clamp, T at the early stop) are taken out of the upstream
    gradient on both sides via the pinned splat oracle."""
    import os
    from types import SimpleNamespace
    from oracle import splat_oracle as SO
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "splat.npz"))
    scene, cam, d = load_case(name)
    scene = SimpleNamespace(means=scene.means, scales=scene.scales, rotations=scene.rotations,
                            thetas=scene.thetas, colors=scene.colors, background=scene.background,
                            splat_opacities=g[f"{name}_opac"])
    prep = vg().prepare(scene, cam, mode="splat")
    prims, offs = prep.tile_lists_device()
    assert np.array_equal(offs.cpu().numpy(), g[f"{name}_offsets"])
    sprep = SO.prepare(scene, cam, key_dtype=np.float32)
    assert np.array_equal(prims.cpu().numpy(), sprep.pair_prim)
    out = vg().render(scene, cam, mode="splat", prep=prep)
    # pixels whose float32 counts differ from the oracle's (each explained by
    # an entry at a threshold), plus alpha-clamp edges, with the splat alphas
    def splat_alphas(p, ids, rows, cols):
        raw, alpha, _, _, _, _, _ = SO._alphas(p, scene, ids, rows, cols, O.ALPHA_CUT, O.ALPHA_CLAMP)
        return raw, alpha
    knife = device_knife_mask(sprep, scene, {}, out.n_contrib, prep.n_active(), alphas=splat_alphas)
    knife_cap(int(knife.sum()), knife.size, f"{name} splat")
    # the image contract (1e-4 + 1e-3 |ref|) everywhere but on knife edges
    bad = image_mismatch(out.color, g[f"{name}_color"])
    assert not (bad & ~knife).any(), (np.argwhere(bad & ~knife)[:5],
                                      float(np.abs(out.color - g[f"{name}_color"]).max()))
    dc = g[f"{name}_dcolor"]
    fields = ("d_means", "d_scales", "d_rotations", "d_colors", "d_background", "d_splat_opacities")
    ref = {f: g[f"{name}_{f}"] for f in fields}
    if knife.any():
        dc = dc * ~knife[..., None]
        r64 = SO.backward(scene, cam, dc, prep=sprep)
        ref = {f: getattr(r64, f) for f in fields}
    gr = vg().backward(scene, cam, dc, mode="splat", prep=prep)
    for f in fields:
        check_field(getattr(gr, f), ref[f], f"{name} splat {f}")
    assert not np.any(gr.d_thetas)


def test_gpu_raymarch_matches_reference_quadrature():
    """The GPU ground-truth ray marcher (vg_raymarch) reproduces the
    reference's oracle.raymarch_image (golden: make_golden_io.py) on the
    reference's golden scene and a 40-primitive miniature of config 1."""
    import os
    from types import SimpleNamespace
    from paper_2412_03378_b200 import groundtruth
    from paper_2412_03378_b200.camera import Camera
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "raymarch.npz"))
    scene, cam, d = load_case("golden_scene")
    col, tf = groundtruth.raymarch_image(scene, cam)
    np.testing.assert_allclose(col, g["golden_color"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(tf, g["golden_T"], rtol=1e-5, atol=1e-6)
    t = np.load(os.path.join(os.path.dirname(__file__), "golden", "tiny.npz"))
    sel = g["mini_sel"]
    mscene = SimpleNamespace(means=t["means"][sel], scales=t["scales"][sel], rotations=t["rotations"][sel],
                             thetas=t["thetas"][sel], colors=t["colors"][sel], background=np.array([0.1, 0.2, 0.3]))
    fx, fy, cx, cy = g["mini_cam_f"]
    mcam = Camera(width=24, height=24, fx=fx, fy=fy, cx=cx, cy=cy, translation=np.array([0.0, 0.0, 3.0]))
    col, tf = groundtruth.raymarch_image(mscene, mcam)
    np.testing.assert_allclose(col, g["mini_color"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(tf, g["mini_T"], rtol=1e-5, atol=1e-6)


def test_analytic_render_matches_ground_truth_on_separated_scene():
    """Acceptance-style check (test_raster.py:146-152): for primitives that do
    not overlap along any ray the closed form is exact, so the rasterizer
    (alpha_cut=0, no early stop, no clamp) agrees with the GPU quadrature."""
    from types import SimpleNamespace
    from paper_2412_03378_b200 import groundtruth
    from paper_2412_03378_b200.camera import look_at
    means = np.array([[-0.6, -0.4, 0.0], [0.5, 0.3, 0.2], [0.0, 0.6, -0.3], [-0.2, -0.7, 0.4]])
    scene = SimpleNamespace(means=means, scales=np.full((4, 3), 0.12),
                            rotations=np.tile([1.0, 0.0, 0.0, 0.0], (4, 1)),
                            thetas=np.array([0.3, 0.6, 0.8, 0.45]),
                            colors=np.array([[0.9, 0.1, 0.1], [0.1, 0.8, 0.2], [0.2, 0.3, 0.9], [0.7, 0.7, 0.1]]),
                            background=np.array([0.05, 0.05, 0.1]))
    cam = look_at([0.0, 0.0, -3.0], [0, 0, 0], width=48, height=40, fov_x_deg=55.0)
    out = vg().render(scene, cam, alpha_cut=0.0, early_stop=None, alpha_clamp=1.0)
    col, tf = groundtruth.raymarch_image(scene, cam)
    assert np.max(np.abs(out.color - col)) < 1e-3
    assert np.max(np.abs(out.final_transmittance - tf)) < 1e-3


@pytest.mark.parametrize("mode", ["analytic", "splat"])
@pytest.mark.parametrize("sort_by", ["depth", "gamma"])
def test_single_and_empty_scenes_all_modes(mode, sort_by):
    """Degenerate sizes through every mode / order / reduction combination:
    one primitive (the depth sort's n == 1 path), an empty scene (background
    only, d_background = sum of d_color, grad.py:126-128)."""
    from types import SimpleNamespace
    from oracle import splat_oracle as SO
    cam = vg().look_at([0, 0, -3.0], [0, 0, 0], width=40, height=24, fov_x_deg=60.0)
    one = SimpleNamespace(means=np.array([[0.1, -0.05, 0.2]]), scales=np.array([[0.3, 0.2, 0.25]]),
                          rotations=np.array([[0.9, 0.1, 0.2, 0.3]]), thetas=np.array([0.6]),
                          colors=np.array([[0.8, 0.3, 0.1]]), splat_opacities=np.array([0.7]),
                          background=np.array([0.1, 0.2, 0.3]))
    rng = np.random.default_rng(5)
    dc = rng.uniform(-1, 1, (24, 40, 3))
    out = vg().render(one, cam, mode=mode, sort_by=sort_by)
    ref = (SO.render(one, cam) if mode == "splat" else O.render(one, cam)).color
    np.testing.assert_allclose(out.color, ref, rtol=1e-3, atol=1e-4)
    for det in (True, False):
        g = vg().backward(one, cam, dc, mode=mode, sort_by=sort_by, deterministic=det)
        rg = SO.backward(one, cam, dc) if mode == "splat" else O.backward(one, cam, dc)
        for f in ("d_means", "d_scales", "d_rotations", "d_colors", "d_background"):
            check_field(getattr(g, f), getattr(rg, f), f"one {mode} {sort_by} {det} {f}")
    empty = SimpleNamespace(means=np.zeros((0, 3)), scales=np.zeros((0, 3)), rotations=np.zeros((0, 4)),
                            thetas=np.zeros(0), colors=np.zeros((0, 3)), splat_opacities=np.zeros(0),
                            background=np.array([0.1, 0.2, 0.3]))
    out = vg().render(empty, cam, mode=mode, sort_by=sort_by)
    np.testing.assert_allclose(out.color, np.broadcast_to([0.1, 0.2, 0.3], (24, 40, 3)), atol=1e-7)
    g = vg().backward(empty, cam, dc, mode=mode, sort_by=sort_by)
    np.testing.assert_allclose(g.d_background, dc.reshape(-1, 3).sum(axis=0), rtol=1e-5)


@pytest.mark.parametrize("parallel", [False, True])
def test_tomography_deterministic_adjoint(parallel):
    """The tomography adjoint in deterministic mode (default of the drop-in):
    bitwise reproducible and equal to the atomic path within tolerance."""
    scene, cam, d = load_case("tiny")
    rng = np.random.default_rng(9)
    w = rng.uniform(0.1, 1.0, (cam.height, cam.width))
    a = vg().tomo_backward(scene, cam, w, parallel=parallel)
    b = vg().tomo_backward(scene, cam, w, parallel=parallel)
    f = vg().tomo_backward(scene, cam, w, parallel=parallel, deterministic=False)
    for k in ("d_means", "d_scales", "d_rotations", "d_thetas", "d_kappas"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
        np.testing.assert_allclose(getattr(a, k), getattr(f, k), rtol=1e-4,
                                   atol=1e-5 * max(1.0, float(np.abs(getattr(f, k)).max())))
    assert np.array_equal(a.visible, f.visible)


def test_host_fed_step_matches_device_step():
    """multiview.HostFedStep (double-buffered host uploads/downloads) returns,
    step by step, what the device-resident ViewShardedStep computes on the
    same scene -- also when the host scene changes between steps (slot reuse)."""
    import torch
    from paper_2412_03378_b200 import configs
    from paper_2412_03378_b200.engine import Engine
    from paper_2412_03378_b200.multiview import HostFedStep, ViewShardedStep
    cfg = configs.large(n=2000, width=96, height=64, n_views=3)
    s = cfg.scene
    eng = Engine(deterministic=True)
    ds = eng.upload(s)
    targets = {v: torch.from_numpy(cfg.target(v, (64, 96, 3))).cuda() for v in range(3)}
    step = ViewShardedStep(eng, ds, cfg.cameras, targets)
    host = {k: torch.from_numpy(np.ascontiguousarray(getattr(s, k))).float().pin_memory()
            for k in ("means", "scales", "rotations", "thetas", "colors")}
    if s.sh is not None:
        host["sh"] = torch.from_numpy(np.ascontiguousarray(s.sh)).float().pin_memory()
    htgt = {v: t.cpu().pin_memory() for v, t in targets.items()}
    ref_eng = Engine(deterministic=True)
    for k in range(4):
        host["means"][:, 0] += 0.001 * k            # a new scene each step
        ref_ds = ref_eng.upload(type("S", (), {n: (t.numpy() if hasattr(t, "numpy") else t)
                                               for n, t in host.items()} | {"background": s.background})())
        ref = ViewShardedStep(ref_eng, ref_ds, cfg.cameras, targets)
        ref_loss = float(ref())
        ref_g = ref.grads.flat.cpu().numpy().copy()
        if k == 0:
            fed = HostFedStep(step, host, htgt)
        fed.step()
        fed.drain()
        torch.cuda.synchronize()
        assert float(fed.loss_host) == ref_loss, k
        np.testing.assert_array_equal(fed.grads_host.numpy(), ref_g, err_msg=f"step {k}")
    # lookahead (prefetching) on a fixed scene: every step bitwise the same
    fed2 = HostFedStep(step, host, htgt, lookahead=True)
    for k in range(3):
        fed2.step()
    fed2.drain()
    torch.cuda.synchronize()
    assert float(fed2.loss_host) == ref_loss
    np.testing.assert_array_equal(fed2.grads_host.numpy(), ref_g)


def test_tomography_split_lists_pinhole():
    """Long per-tile lists (~950 pairs per tile) make the projector split each
    tile over several CTAs (forward partial images summed in split order,
    adjoint one thread per pair): image and adjoint against the float64
    oracle, the deterministic adjoint bitwise reproducible."""
    from paper_2412_03378_b200 import configs
    cfg = configs.medium(n=3000, size=64, n_views=1)
    scene = _f64_scene(cfg.scene)
    cam = cfg.cameras[0]
    prep = vg().tomo_prepare(scene, cam)
    assert prep.pair_count() / (prep.n_tiles_x * prep.n_tiles_y) > 512   # splits > 1 both ways
    img, inten = vg().tomo_forward(scene, cam, prep=prep, intensity=True)
    ref = O.tomo_forward(scene, cam)
    check_field(img, ref, "split tomo image")
    np.testing.assert_allclose(inten, np.exp(-ref), rtol=1e-4, atol=1e-6)
    w = np.random.default_rng(4).uniform(0.1, 1.0, (cam.height, cam.width))
    a = vg().tomo_backward(scene, cam, w)
    b = vg().tomo_backward(scene, cam, w)
    rg = O.tomo_backward(scene, cam, w)
    for f in ("d_means", "d_scales", "d_rotations", "d_thetas", "d_kappas"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
        check_field(getattr(a, f), getattr(rg, f), f"split tomo {f}")


def test_host_fed_step_kernel_download():
    """HostFedStep with the streaming-kernel gradient download (vg_copy_streaming)
    delivers the same bytes as the copy-engine download."""
    import torch
    from paper_2412_03378_b200 import configs
    from paper_2412_03378_b200.engine import Engine
    from paper_2412_03378_b200.multiview import HostFedStep, ViewShardedStep
    cfg = configs.large(n=2000, width=96, height=64, n_views=3)
    s = cfg.scene
    eng = Engine(deterministic=True)
    ds = eng.upload(s)
    targets = {v: torch.from_numpy(cfg.target(v, (64, 96, 3))).cuda() for v in range(3)}
    step = ViewShardedStep(eng, ds, cfg.cameras, targets)
    host = {k: torch.from_numpy(np.ascontiguousarray(getattr(s, k))).float().pin_memory()
            for k in ("means", "scales", "rotations", "thetas", "colors")}
    if s.sh is not None:
        host["sh"] = torch.from_numpy(np.ascontiguousarray(s.sh)).float().pin_memory()
    htgt = {v: t.cpu().pin_memory() for v, t in targets.items()}
    out = []
    for ctas in (0, 8):
        fed = HostFedStep(step, host, htgt, lookahead=True, download_ctas=ctas)
        for _ in range(3):
            fed.step()
        fed.drain()
        torch.cuda.synchronize()
        out.append((fed.grads_host.numpy().copy(), float(fed.loss_host)))
    np.testing.assert_array_equal(out[0][0], out[1][0])
    assert out[0][1] == out[1][1]


def test_integration_md_ctypes_stub_runs():
    """The ctypes binding shown in INTEGRATION.md section 3 (what a maintainer
    adds to the reference) runs as written and renders what render() renders."""
    import os
    import torch
    from paper_2412_03378_b200 import configs
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cfg = configs.tiny()
    scene, cam = cfg.scene, cfg.cameras[0]
    src = open(os.path.join(root, "INTEGRATION.md")).read()
    body = src[src.index("## 3. The ctypes binding"):]
    body = body[body.index("```python") + len("```python"):]
    body = body[:body.index("```")]
    cwd = os.getcwd()
    os.chdir(root)
    try:
        ns = {"scene": scene, "cam": cam}
        exec(compile(body, "INTEGRATION.md#3", "exec"), ns)
    finally:
        os.chdir(cwd)
    torch.cuda.synchronize()
    ref = vg().render(scene, cam)
    np.testing.assert_allclose(ns["color"].cpu().numpy(), ref.color, rtol=1e-6, atol=1e-6)


def test_parallel_beam_anisotropic_narrow_and_wide():
    """Parallel-beam projector and adjoint on rotated anisotropic Gaussians
    from sub-pixel to tile-spanning widths: exercises the row recurrence and
    its per-pixel fallback (anchors deep in a narrow tail), the tail skip and
    the moment-form adjoint with a non-zero shear term (P21) and centres
    inside and outside the tile."""
    rng = np.random.default_rng(23)
    n = 400
    from types import SimpleNamespace
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    scales = np.exp(rng.uniform(np.log(0.004), np.log(0.15), (n, 3)))
    scene = SimpleNamespace(means=rng.uniform(-1, 1, (n, 3)).astype(np.float32).astype(np.float64),
                            scales=scales.astype(np.float32).astype(np.float64),
                            rotations=q.astype(np.float32).astype(np.float64),
                            thetas=rng.uniform(0.05, 0.9, n).astype(np.float32).astype(np.float64),
                            colors=np.zeros((n, 3)), background=np.zeros(3))
    cam = vg().look_at([4.0 * np.sin(1.1), 0.7, 4.0 * np.cos(1.1)], [0, 0, 0], width=96, height=80,
                       fov_x_deg=30.0)
    img = vg().tomo_forward(scene, cam, parallel=True, extent=1.2)
    ref = O.tomo_forward(scene, cam, parallel=True, extent=1.2)
    check_field(img, ref, "anisotropic parallel image")
    w = rng.uniform(-1.0, 1.0, (80, 96))
    g = vg().tomo_backward(scene, cam, w, parallel=True, extent=1.2)
    rg = O.tomo_backward(scene, cam, w, parallel=True, extent=1.2)
    for f in ["d_means", "d_scales", "d_rotations", "d_thetas", "d_kappas"]:
        check_field(getattr(g, f), getattr(rg, f), f"anisotropic parallel {f}")
    assert np.array_equal(g.visible, rg.visible)


def _recon_golden():
    import os
    from types import SimpleNamespace
    from paper_2412_03378_b200.camera import Camera
    d = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "recon.npz"))
    projs = []
    for k in range(int(d["n_proj"])):
        w, h, fx, fy, cx, cy, zn = d[f"p{k}_cam"]
        cam = Camera(width=int(w), height=int(h), fx=fx, fy=fy, cx=cx, cy=cy, rotation=d[f"p{k}_rot"],
                     translation=d[f"p{k}_trans"], z_near=zn)
        projs.append(SimpleNamespace(camera=cam, image=d[f"p{k}_image"]))
    return d, projs


def test_voxelize_matches_reference():
    """tomo.voxelize on the GPU (vg_voxelize) against the reference's grid: the
    float64 oracle on the same float32-rounded inputs to float64 rounding, the
    reference's float64-input grid to float32 input precision."""
    from types import SimpleNamespace
    from paper_2412_03378_b200 import tomo
    d, _ = _recon_golden()
    f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
    scene = SimpleNamespace(means=f32(d["vox_means"]), scales=f32(d["vox_scales"]),
                            rotations=f32(d["vox_rotations"]), thetas=f32(d["vox_thetas"]),
                            colors=np.full((len(d["vox_thetas"]), 3), 0.5), background=np.zeros(3))
    grid = tomo.voxelize(scene, resolution=d["vox_values"].shape, bbox=(d["vox_bmin"], d["vox_bmax"]))
    ref32 = O.voxelize(scene.means, scene.scales, scene.rotations, scene.thetas, d["vox_values"].shape,
                       d["vox_bmin"], d["vox_bmax"])
    np.testing.assert_allclose(grid.values, ref32, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(grid.values, d["vox_values"], rtol=1e-5, atol=1e-6 * d["vox_values"].max())
    # flat (zero spacing) and reversed boxes, which tomo.voxelize accepts
    # unchecked: the device's index ranges are numpy's searchsorted on them
    for tag in ("flat", "reversed"):
        lo, hi = d[f"vox_{tag}_bmin"], d[f"vox_{tag}_bmax"]
        ref_v = d[f"vox_{tag}_values"]
        g2 = tomo.voxelize(scene, resolution=ref_v.shape, bbox=(lo, hi))
        o2 = O.voxelize(scene.means, scene.scales, scene.rotations, scene.thetas, ref_v.shape, lo, hi)
        np.testing.assert_allclose(g2.values, o2, rtol=1e-9, atol=1e-12, err_msg=tag)
        np.testing.assert_allclose(g2.values, ref_v, rtol=1e-5, atol=1e-6 * ref_v.max(), err_msg=tag)
    empty = tomo.voxelize(SimpleNamespace(means=np.zeros((0, 3)), scales=np.zeros((0, 3)),
                                          rotations=np.zeros((0, 4)), thetas=np.zeros(0),
                                          colors=np.zeros((0, 3)), background=np.zeros(3)),
                          resolution=(4, 6, 8))
    assert empty.values.shape == (4, 6, 8) and not empty.values.any()


def test_reconstruct_follows_reference():
    """tomo.reconstruct on the GPU against the reference's own run
    (make_golden_recon.py: six 24x24 cone-beam blob projections, L2, 16
    primitives, 24 iterations, seed 0): same initial draws and view order, the
    loss curve, the final primitives, the voxel grid and psnr/ssim_3d."""
    from paper_2412_03378_b200 import tomo
    from paper_2412_03378_b200.optim import TrainConfig
    d, projs = _recon_golden()
    ref = tomo.DensityGrid(d["ref_grid"], -np.ones(3), np.ones(3))
    cfg = TrainConfig(iterations=24, loss="l2", n_init=16, seed=0)
    scene, grid, rep = tomo.reconstruct(projs, cfg, resolution=20, reference=ref)
    scene2, _, rep2 = tomo.reconstruct(projs, cfg, resolution=20, reference=ref)
    assert rep2["losses"] == rep["losses"]          # deterministic adjoint (default)
    assert not rep["diverged"] and rep["final_count"] == 16 == scene.n
    # measured on B200: losses 1e-6 relative, primitives <= 1.5e-5, psnr 4e-6
    np.testing.assert_allclose(rep["losses"], d["losses"], rtol=1e-4)
    for k in ("means", "scales", "rotations", "thetas"):
        np.testing.assert_allclose(getattr(scene, k).cpu().numpy(), d[f"final_{k}"], rtol=1e-4, atol=1e-4,
                                   err_msg=k)
    np.testing.assert_allclose(grid.values, d["grid"], rtol=1e-4, atol=1e-4 * d["grid"].max())
    assert rep["psnr_3d"] == pytest.approx(float(d["psnr_3d"]), abs=1e-3)
    assert rep["ssim_3d"] == pytest.approx(float(d["ssim_3d"]), abs=1e-5)
    with pytest.raises(ValueError):
        tomo.reconstruct(projs[:1], cfg)


def test_reconstruct_mixed_loss_follows_reference():
    """tomo.reconstruct with the reference's default loss, mixed (0.8 L1 +
    0.2 D-SSIM, grad.py:338-358): the loss is formed on the device image by
    grad.loss_and_grad and pulled back through the explicit-gradient adjoint;
    loss curve, final primitives and voxel grid against the reference's own
    run (make_golden_recon.py), and two runs are bitwise identical
    (deterministic adjoint, the default)."""
    from paper_2412_03378_b200 import tomo
    from paper_2412_03378_b200.optim import TrainConfig
    d, projs = _recon_golden()
    ref = tomo.DensityGrid(d["ref_grid"], -np.ones(3), np.ones(3))
    cfg = TrainConfig(iterations=24, n_init=16, seed=0)
    assert cfg.loss.kind == "mixed"
    scene, grid, rep = tomo.reconstruct(projs, cfg, resolution=20, reference=ref)
    assert not rep["diverged"]
    np.testing.assert_allclose(rep["losses"], d["mixed_losses"], rtol=1e-4)
    for k in ("means", "scales", "rotations", "thetas"):
        np.testing.assert_allclose(getattr(scene, k).cpu().numpy(), d[f"mixed_final_{k}"], rtol=1e-4,
                                   atol=1e-4, err_msg=k)
    np.testing.assert_allclose(grid.values, d["mixed_grid"], rtol=1e-4, atol=1e-4 * d["mixed_grid"].max())
    assert rep["psnr_3d"] == pytest.approx(float(d["mixed_psnr_3d"]), abs=1e-3)
    scene2, _, rep2 = tomo.reconstruct(projs, cfg, resolution=20, reference=ref)
    assert rep2["losses"] == rep["losses"]
    for k in ("means", "scales", "rotations", "thetas"):
        assert np.array_equal(getattr(scene2, k).cpu().numpy(), getattr(scene, k).cpu().numpy()), k


def test_pipelined_step_is_stable_across_steps():
    """Repeated multi-view steps on identical inputs (three contexts, binning on
    the side stream, two alternating blend streams): atomic mode varies only by
    summation order, deterministic mode is bitwise identical step to step."""
    import torch
    from paper_2412_03378_b200 import configs
    from paper_2412_03378_b200.engine import Engine
    from paper_2412_03378_b200.multiview import ViewShardedStep
    cfg = configs.large(n=3000, width=96, height=64, n_views=7)
    targets = {v: torch.from_numpy(cfg.target(v, (64, 96, 3))).cuda() for v in range(7)}
    for det in (False, True):
        eng = Engine(deterministic=det)
        step = ViewShardedStep(eng, eng.upload(cfg.scene), cfg.cameras, targets)
        losses, grads = [], []
        for _ in range(5):
            losses.append(float(step()))
            grads.append(step.grads.flat.clone())
        for g in grads[1:]:
            if det:
                assert torch.equal(g, grads[0])
            else:
                torch.testing.assert_close(g, grads[0], rtol=1e-4, atol=1e-7)
        assert max(losses) - min(losses) <= 1e-12 * abs(losses[0])


def test_sh_gradient_matches_float64_central_differences():
    """SH-3 colour gradients against float64 central differences (the FD
    semantics of grad.fd_check, grad.py:420-467): L = sum_px w . colour over
    two views of the float64 oracle fed each view's SH-evaluated RGB, the
    analytic gradient from the device backward of w (d_means includes the
    colour's view-direction term, d_sh the per-view basis pull-back).  Smooth
    flags (no cut, no early stop, no clamp) so the differences see no
    threshold."""
    from types import SimpleNamespace
    from paper_2412_03378_b200 import configs
    rng = np.random.default_rng(31)
    n = 24
    f32 = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)  # noqa: E731
    means = f32(rng.uniform(-0.5, 0.5, (n, 3)))
    scales = f32(np.exp(rng.uniform(np.log(0.08), np.log(0.22), (n, 3))))
    q = rng.normal(size=(n, 4))
    rots = f32(q / np.linalg.norm(q, axis=1, keepdims=True))
    thetas = f32(rng.uniform(0.2, 0.8, n))
    sh = rng.normal(0.0, 0.3, (n, 16, 3))
    sh[:, 0, :] = rng.uniform(0.2, 0.9, (n, 3))
    sh = f32(sh)
    flags = dict(alpha_cut=0.0, early_stop=None, alpha_clamp=1.0)
    cams = [vg().look_at([0.4, 0.6, -3.0], [0, 0, 0], width=40, height=32, fov_x_deg=50.0),
            vg().look_at([-2.5, 0.3, -1.8], [0, 0, 0], width=40, height=32, fov_x_deg=50.0)]
    ws = [rng.uniform(-1, 1, (32, 40, 3)) for _ in cams]

    def oracle_loss(m, coef):
        tot = 0.0
        for cam, w in zip(cams, ws):
            d = m - O.cam_center(cam)
            d /= np.linalg.norm(d, axis=1, keepdims=True)
            rgb = np.einsum("nl,nlc->nc", configs.sh_basis(d), coef)
            sc = SimpleNamespace(means=m, scales=scales, rotations=rots, thetas=thetas, colors=rgb,
                                 background=np.zeros(3))
            tot += float(np.sum(O.render(sc, cam, **flags).color * w))
        return tot

    dev_scene = SimpleNamespace(means=means, scales=scales, rotations=rots, thetas=thetas, sh=sh,
                                colors=None, background=np.zeros(3))
    gm = np.zeros((n, 3))
    gsh = np.zeros((n, 16, 3))
    for cam, w in zip(cams, ws):
        g = vg().backward(dev_scene, cam, w, **flags)
        gm += np.asarray(g.d_means)
        gsh += np.asarray(g.d_sh).reshape(n, 16, 3)
    eps = 1e-5
    picks = rng.choice(n, 6, replace=False)
    for i in picks:
        for k in range(3):
            a, b = means.copy(), means.copy()
            a[i, k] += eps
            b[i, k] -= eps
            fd = (oracle_loss(a, sh) - oracle_loss(b, sh)) / (2 * eps)
            assert abs(gm[i, k] - fd) <= 1e-4 * np.abs(gm).max() + 1e-3 * abs(fd), (i, k, gm[i, k], fd)
        for l, ch in ((0, 0), (3, 1), (8, 2), (15, 0)):
            a, b = sh.copy(), sh.copy()
            a[i, l, ch] += eps
            b[i, l, ch] -= eps
            fd = (oracle_loss(means, a) - oracle_loss(means, b)) / (2 * eps)
            assert abs(gsh[i, l, ch] - fd) <= 1e-4 * np.abs(gsh).max() + 1e-3 * abs(fd), (i, l, ch, gsh[i, l, ch], fd)
    # the direction term matters at this scale: without it d_means misses
    # sum_v (I - d d^T)/|u| grad_b . (sh dRGB)
    assert np.abs(gm).max() > 0


# --- config 3: the full 64-view step against the per-view oracle ------------

_STEP64 = {}


def _oracle_view_job(v):
    """Worker (forked): view v of config 3 on the float64 oracle -- its
    seeded tile, the knife-edge pixels there (the device's counts against
    the oracle's), and the backward of the L2 residual against the seeded
    tile target (knife pixels excluded), as sparse rows.  Runs in a child
    process: numpy only."""
    from types import SimpleNamespace
    from paper_2412_03378_b200 import configs
    s, cams, means, sh = _STEP64["scene"], _STEP64["cams"], _STEP64["means"], _STEP64["sh"]
    t, dev_nc, dev_na = _STEP64["dev"][v]
    cam = cams[v]
    c = O.cam_center(cam)
    d = means - c
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    basis = configs.sh_basis(d)
    rgb = np.einsum("nl,nlc->nc", basis, sh)
    scene = SimpleNamespace(means=means, scales=s.scales.astype(np.float64),
                            rotations=s.rotations.astype(np.float64), thetas=s.thetas.astype(np.float64),
                            colors=rgb, background=np.zeros(3))
    prep = O.prepare(scene, cam, key_dtype=np.float32)
    ref = O.render(scene, cam, prep=prep, tiles=[t])
    ty, tx = divmod(t, prep.tiles_x)
    r0, c0 = ty * 16, tx * 16
    h, w = dev_nc.shape
    full_nc = np.zeros((cam.height, cam.width), dtype=np.int64)
    full_na = np.zeros((cam.height, cam.width), dtype=np.int64)
    full_nc[r0:r0 + h, c0:c0 + w] = dev_nc
    full_na[r0:r0 + h, c0:c0 + w] = dev_na
    knife = device_knife_mask(prep, scene, {}, full_nc, full_na, tiles=[t])
    rng = np.random.default_rng(1000 + v)
    tgt = rng.uniform(0.0, 1.0, (h, w, 3))
    keep = ~knife[r0:r0 + h, c0:c0 + w]
    r = (ref.color[r0:r0 + h, c0:c0 + w] - tgt) * keep[..., None]
    dc = np.zeros((cam.height, cam.width, 3))
    dc[r0:r0 + h, c0:c0 + w] = 2.0 * r / (3.0 * cam.width * cam.height)
    g = O.backward(scene, cam, dc, prep=prep, tiles=[t])
    rows = np.flatnonzero(g.visible | np.any(g.d_colors != 0, axis=1))
    out = {f: getattr(g, f)[rows] for f in ("d_means", "d_scales", "d_rotations", "d_thetas",
                                           "d_kappas", "d_colors")}
    out["d_means"] = out["d_means"] + _sh_dir_rows(means[rows], c, sh[rows], out["d_colors"])
    out["d_sh"] = basis[rows][:, :, None] * out["d_colors"][:, None, :]
    return dict(v=v, tile=t, knife=int((~keep).sum()), tgt=tgt, keep=keep, rows=rows, g=out,
                d_background=g.d_background, loss=float(np.sum(r * r)))


def _sh_dir_rows(means, centre, sh, d_rgb):
    """Numpy restatement of sh_direction_grad for the worker (no torch in a
    forked child): central differences of the float64 basis along each axis
    are not needed -- the basis is polynomial, so use its exact derivative by
    complex-step differentiation."""
    from paper_2412_03378_b200 import configs
    out = np.zeros_like(means)
    for k in range(3):
        m = means.astype(np.complex128)
        m[:, k] += 1e-30j
        d = m - centre
        d = d / np.sqrt(np.sum(d * d, axis=1, keepdims=True))
        rgb = np.einsum("nl,nlc->nc", configs.sh_basis(d), sh)
        out[:, k] = np.sum(rgb.imag * d_rgb, axis=1) / 1e-30
    return out


def _engine_lists(eng):
    """Tile offsets of an engine's last prepare (host int64)."""
    import torch
    from paper_2412_03378_b200 import _lib
    nt = ((eng.cam.width + 15) // 16) * ((eng.cam.height + 15) // 16)
    P = eng.pair_count()
    prims = torch.empty(max(P, 1), dtype=torch.int32, device=eng.device)
    offs = torch.empty(nt + 1, dtype=torch.int32, device=eng.device)
    _lib.check(eng.lib.vg_tile_lists(eng.ctx.handle, _lib.ptr(prims), _lib.ptr(offs), eng.stream()),
               "vg_tile_lists")
    return prims[:P].cpu().numpy(), offs.cpu().numpy().astype(np.int64)


def test_full_size_large_64_view_step_equals_sum_of_oracle_views():
    """BASELINE config 3 at full size: N=1M SH-3 Gaussians, all 64 views at
    1920x1080 through the production multi-view step (pipelined contexts,
    dual blend streams, fused L2, deferred float64 parameter chain, SH
    pull-back incl. the view-direction term).  Each view's target equals the
    device's own render except on one seeded tile per view (seeded values;
    knife-edge pixels keep the device colour), so the L2 gradient is zero
    outside those 64 tiles and the step's flat gradient must equal the sum of
    64 per-view float64 oracle backwards (raster.py:410-439, grad.py:107-259)
    on those tiles."""
    import multiprocessing as mp
    import torch
    from paper_2412_03378_b200 import configs
    from paper_2412_03378_b200.engine import Engine
    from paper_2412_03378_b200.multiview import ViewShardedStep
    cfg = configs.large()
    s = cfg.scene
    _STEP64.update(scene=s, cams=cfg.cameras, means=s.means.astype(np.float64), sh=s.sh.astype(np.float64))
    V = len(cfg.cameras)
    assert V == 64
    eng = Engine()
    ds = eng.upload(s)
    # the device forward of every view: its colour (the target outside the
    # sampled tile) and its counts on one seeded tile of at least median
    # list length
    colors, dev = [], {}
    for v, cam in enumerate(cfg.cameras):
        eng.prepare(ds, cam)
        color, _, ncon = eng.forward()
        nact = eng.n_active()
        _, offs = _engine_lists(eng)
        lens = np.diff(offs)
        cand = np.flatnonzero(lens >= np.median(lens[lens > 0]))
        t = int(np.random.default_rng(1000 + v).choice(cand))
        ty, tx = divmod(t, (cam.width + 15) // 16)
        blk = (slice(ty * 16, min(ty * 16 + 16, cam.height)), slice(tx * 16, min(tx * 16 + 16, cam.width)))
        dev[v] = (t, ncon[blk].cpu().numpy(), nact[blk].cpu().numpy())
        colors.append(color.clone())
    _STEP64["dev"] = dev
    ctx = mp.get_context("fork")
    with ctx.Pool(min(8, os.cpu_count() or 1)) as pool:
        res = pool.map(_oracle_view_job, range(V))
    targets = {}
    for v, cam in enumerate(cfg.cameras):
        tg = colors[v]
        r = res[v]
        ty, tx = divmod(r["tile"], (cam.width + 15) // 16)
        h, w = r["tgt"].shape[:2]
        blk = tg[ty * 16:ty * 16 + h, tx * 16:tx * 16 + w]
        keep = torch.from_numpy(r["keep"]).cuda()[..., None]
        blk.copy_(torch.where(keep, torch.from_numpy(r["tgt"]).float().cuda(), blk))
        targets[v] = tg
    step = ViewShardedStep(eng, ds, cfg.cameras, targets)
    loss = float(step())
    g = step.grads.to_scene_grads("analytic", torch_out=False)
    n = len(s.means)
    tot = {f: np.zeros((n,) + np.shape(res[0]["g"][f])[1:]) for f in res[0]["g"]}
    bg = np.zeros(3)
    ref_loss = 0.0
    for r in res:
        for f, a in r["g"].items():
            np.add.at(tot[f], r["rows"], a)
        bg += r["d_background"]
        ref_loss += r["loss"]
    knives = sum(r["knife"] for r in res)
    knife_cap(knives, 256 * V, "64-view step")
    assert abs(loss - ref_loss) <= 1e-4 * ref_loss
    for f in ("d_means", "d_scales", "d_rotations", "d_thetas", "d_kappas"):
        check_field(getattr(g, f), tot[f], f"64-view step {f}")
    check_field(np.asarray(g.d_sh).reshape(n, 48), tot["d_sh"].reshape(n, 48), "64-view step d_sh")
    check_field(g.d_background, bg, "64-view step d_background")


def test_deterministic_views_without_pairs_stay_reproducible():
    """Deterministic mode with views that bin no (tile, Gaussian) pair (the
    camera looks away; and the empty scene): their d_background / loss still
    go through the fixed-order per-tile sums, so a deferred multi-view step
    mixing them with ordinary views on the two blend streams is bitwise
    reproducible, and d_background equals the tile-order sum of d_color."""
    import torch
    from types import SimpleNamespace
    from paper_2412_03378_b200 import configs
    from paper_2412_03378_b200.engine import Engine
    from paper_2412_03378_b200.multiview import ViewShardedStep
    cfg = configs.large(n=3000, width=96, height=64, n_views=4)
    away = vg().look_at([0.0, 0.0, 30.0], [0.0, 0.0, 60.0], width=96, height=64, fov_x_deg=20.0)
    cams = [cfg.cameras[0], away, cfg.cameras[1], away, cfg.cameras[2]]
    targets = {v: torch.from_numpy(cfg.target(v, (64, 96, 3))).cuda() for v in range(len(cams))}
    eng = Engine(deterministic=True)
    step = ViewShardedStep(eng, eng.upload(cfg.scene), cams, targets)
    runs = []
    for _ in range(3):
        loss = float(step())
        runs.append((loss, step.grads.flat.clone()))
    for loss, g in runs[1:]:
        assert loss == runs[0][0] and torch.equal(g, runs[0][1])
    empty = SimpleNamespace(means=np.zeros((0, 3)), scales=np.zeros((0, 3)), rotations=np.zeros((0, 4)),
                            thetas=np.zeros(0), colors=np.zeros((0, 3)), background=np.array([0.1, 0.2, 0.3]))
    dc = np.random.default_rng(1).uniform(-1, 1, (64, 96, 3)).astype(np.float32)
    a = vg().backward(empty, away, dc)
    b = vg().backward(empty, away, dc)
    assert np.array_equal(a.d_background, b.d_background)
    np.testing.assert_allclose(a.d_background, dc.astype(np.float64).reshape(-1, 3).sum(axis=0), rtol=1e-5)


@pytest.mark.parametrize("loss", ["l2", "dssim"])
def test_device_fd_check(loss):
    """grad.fd_check on the device (grad.py:420-467): every scalar parameter
    of a small smooth scene, the device backward against five-point central
    differences of the device render's loss (float32 renders, so a float32
    step); the analytic and numeric derivatives agree.  Smooth losses only:
    the L1 term of 'mixed' has kinks at r = 0 that a float32-sized step
    straddles."""
    from types import SimpleNamespace
    rng = np.random.default_rng(12)
    n = 5
    q = rng.normal(size=(n, 4))
    scene = SimpleNamespace(means=rng.uniform(-0.4, 0.4, (n, 3)), scales=rng.uniform(0.12, 0.3, (n, 3)),
                            rotations=q / np.linalg.norm(q, axis=1, keepdims=True),
                            thetas=rng.uniform(0.2, 0.6, n), colors=rng.uniform(0.1, 0.9, (n, 3)),
                            background=np.array([0.1, 0.1, 0.2]))
    cam = vg().look_at([0.2, -0.3, -2.5], [0, 0, 0], width=32, height=32, fov_x_deg=45.0)
    target = rng.uniform(0, 1, (32, 32, 3))
    rep = vg().fd_check(scene, cam, target, vg().LossSpec.parse(loss))
    assert len(rep.records) == n * 14
    big = [r for r in rep.records if max(abs(r.analytic), abs(r.numeric)) > 1e-3 * max(
        abs(x.analytic) for x in rep.records)]
    frac = sum(r.within(2e-2) for r in big) / len(big)
    print(f"[fd_check {loss}] {len(big)} non-negligible records, {frac:.3f} within 2e-2, worst {rep.worst()}")
    assert frac >= 0.95


def test_hostio_round_trips():
    """The facade's pinned staging (hostio): float64 numpy -> float32 device
    equals numpy's float32 rounding; downloads are exact; non-contiguous and
    empty inputs; back-to-back transfers through the same staging buffer do
    not overwrite each other."""
    import torch
    from paper_2412_03378_b200 import hostio
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(7)
    a = rng.normal(size=(300, 7))
    t = hostio.to_device(a[:, ::2], dev, (300, 4))      # non-contiguous view
    assert np.array_equal(t.cpu().numpy(), a[:, ::2].astype(np.float32))
    outs = [hostio.to_device(np.full(1000, float(k)), dev, (1000,)) for k in range(5)]
    for k, o in enumerate(outs):
        assert bool((o == k).all())
    g = torch.randn(1234, device=dev)
    h = hostio.to_host(g)
    assert h.dtype == np.float64 and np.array_equal(h, g.double().cpu().numpy())
    i = torch.arange(77, dtype=torch.int32, device=dev)
    assert np.array_equal(hostio.to_host(i, np.int32), np.arange(77))
    assert hostio.to_device(np.zeros((0, 3)), dev, (0, 3)).shape == (0, 3)
    assert hostio.to_host(torch.zeros((0, 3), device=dev)).shape == (0, 3)
    assert hostio.all_finite(g) and not hostio.all_finite(g / 0.0)


def _deep_scene(n=5000, seed=11):
    """Thin, overlapping Gaussians: ~5000-entry tile lists walked to depths of
    1500-5000 before the early stop, i.e. several VG_SEG (1024) segments per
    tile for the segmented backward."""
    from types import SimpleNamespace
    rng = np.random.default_rng(seed)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return SimpleNamespace(means=rng.normal(0, 0.25, (n, 3)), scales=rng.uniform(0.25, 0.5, (n, 3)),
                           rotations=q, thetas=rng.uniform(0.002, 0.006, n),
                           colors=rng.uniform(0, 1, (n, 3)), background=np.array([0.2, 0.1, 0.3]))


_SEG_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
import test_parity_gpu as T
g = T._deep_engine_backward(np.load(sys.argv[2])["dc"], passes=1)[0]
np.savez(sys.argv[3], **g)
"""


def _segments(ctx):
    import ctypes
    import paper_2412_03378_b200._lib as L
    n, flag = ctypes.c_int64(), ctypes.c_int32()
    L.check(L.load().vg_debug_segments(ctx.handle, ctypes.byref(n), ctypes.byref(flag)),
            "vg_debug_segments")
    return int(flag.value), int(n.value)


def _deep_engine_backward(dc, passes=2, deterministic=False, sort_by="depth"):
    """Forward + explicit-gradient backward of the deep scene, `passes` times
    on one atomic-mode engine context; per pass the gradient fields and the
    context's segment plan (segmented flag, item count)."""
    import torch
    from paper_2412_03378_b200.engine import Engine
    s = _deep_scene()
    cam = vg().look_at([0, 0, -3.0], [0, 0, 0], width=40, height=36, fov_x_deg=40.0)
    eng = Engine(deterministic=deterministic, sort_by=sort_by)
    ds = eng.upload(s)
    eng.prepare(ds, cam)
    dct = torch.from_numpy(np.ascontiguousarray(dc, dtype=np.float32)).cuda()
    out = []
    for _ in range(passes):
        color, tfin, _ = eng.forward(counts=False)
        grads = eng.new_grads(ds)
        eng.backward(color, tfin, dct, grads)
        torch.cuda.synchronize()
        sg = grads.to_scene_grads("analytic", False)
        out.append(({f: np.array(getattr(sg, f), dtype=np.float64) for f in GRAD_FIELDS + ["d_background"]},
                    _segments(eng.ctx)))
    return [g for g, _ in out] if passes == 1 else out


def test_segmented_backward_deep_tiles(tmp_path):
    """Tiles walked past several VG_SEG boundaries.  The first atomic-mode
    forward on a context only records depth statistics; the next view's
    backward then splits this scene's deep tiles into (tile, segment) items
    that run as independent CTAs from the forward's boundary states.  Both
    passes against the oracle (parity contract); the segmented pass equal to
    the unsegmented one within float32 rounding, and to the backward of a
    library with segmentation off (VG_SEG_BWD=0, child process); the
    deterministic backward never segments (bitwise reproducible)."""
    import subprocess
    import sys
    s = _deep_scene()
    cam = vg().look_at([0, 0, -3.0], [0, 0, 0], width=40, height=36, fov_x_deg=40.0)
    dc = np.random.default_rng(5).uniform(-1, 1, (36, 40, 3))
    flags = dict(early_stop=O.EARLY_STOP_T, alpha_cut=O.ALPHA_CUT)
    dprep = vg().prepare(s, cam)
    out = vg().render(s, cam, prep=dprep)
    na = dprep.n_active()
    assert na.max() > 4 * 1024, "the scene must span several segments"
    prep = O.prepare(s, cam)
    knife = device_knife_mask(prep, s, flags, out.n_contrib, na)
    knife_cap(int(knife.sum()), knife.size, "deep backward")
    dck = dc * ~knife[..., None]
    ref = O.backward(s, cam, dck, prep=prep)
    (g1, p1), (g2, p2) = _deep_engine_backward(dck)
    assert p1 == (0, 0), "no statistics before the first forward"
    # segmented backward (bit 0) and deep-tile forward (bit 1)
    assert p2[0] == 3 and p2[1] > 2 * 9, p2
    for f in GRAD_FIELDS + ["d_background"]:
        check_field(g1[f], getattr(ref, f), f"deep unsegmented {f}")
        check_field(g2[f], getattr(ref, f), f"deep segmented {f}")
        np.testing.assert_allclose(g2[f], g1[f], rtol=1e-4, atol=1e-5 * max(1.0, float(np.abs(g1[f]).max())),
                                   err_msg=f)
    # a library with segmentation off, same upstream gradient
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    np.savez(str(tmp_path / "dc.npz"), dc=dck)
    env = dict(os.environ, VG_SEG_BWD="0")
    r = subprocess.run([sys.executable, "-c", _SEG_CHILD, root, str(tmp_path / "dc.npz"),
                        str(tmp_path / "unseg.npz")], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    unseg = np.load(str(tmp_path / "unseg.npz"))
    for f in GRAD_FIELDS + ["d_background"]:
        np.testing.assert_allclose(g2[f], unseg[f], rtol=1e-4,
                                   atol=1e-5 * max(1.0, float(np.abs(unseg[f]).max())), err_msg=f)
    # deterministic mode: never a segmented backward (the deep-tile forward,
    # bitwise equal to the regular one, from the second pass), reproducible
    (d1, q1), (d2, q2) = _deep_engine_backward(dck, deterministic=True)
    assert q1 == (0, 0) and q2 == (2, 0), (q1, q2)
    for f in GRAD_FIELDS + ["d_background"]:
        assert np.array_equal(d1[f], d2[f]), f
        check_field(d1[f], getattr(ref, f), f"deep det {f}")


_TAIL_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
import test_parity_gpu as T
flat, loss, _ = T._tail_step()
np.savez(sys.argv[2], flat=flat, loss=np.array(loss))
"""


def _tail_step(steps=2):
    """Two multi-view steps (three rotating contexts, two blend streams,
    atomic mode) of a small opaque scene; every context's later views are
    tail-bound (a 256 x 256 view has far fewer tiles than backward CTA slots).
    Returns the last step's flat gradient buffer, its loss and the per-context
    load-balance plans of the last views."""
    import torch
    from paper_2412_03378_b200 import configs
    from paper_2412_03378_b200.engine import Engine
    from paper_2412_03378_b200.multiview import ViewShardedStep
    cfg = configs.opaque(n=60000, size=256, n_views=6)
    eng = Engine(deterministic=False)
    ds = eng.upload(cfg.scene)
    targets = {v: torch.from_numpy(cfg.target(v, (256, 256, 3))).cuda() for v in range(6)}
    step = ViewShardedStep(eng, ds, cfg.cameras, targets)
    for _ in range(steps):
        loss = float(step())
    torch.cuda.synchronize()
    plans = [_segments(e.ctx) for e in step.engines]
    return step.grads.flat.cpu().numpy().astype(np.float64), loss, plans


def test_tail_bound_multiview_step_matches_unsegmented(tmp_path):
    """The production multi-view step with the load-balance paths engaged
    (deep-tile forward beside the regular launch on each context's side
    stream, segmented backward) equals the same step with them off
    (VG_SEG_BWD=0, child process) within float32 rounding."""
    import subprocess
    import sys
    flat, loss, plans = _tail_step()
    assert all(p[0] == 3 for p in plans), plans
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = str(tmp_path / "off.npz")
    env = dict(os.environ, VG_SEG_BWD="0")
    r = subprocess.run([sys.executable, "-c", _TAIL_CHILD, root, path], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    off = np.load(path)
    assert abs(loss - float(off["loss"])) <= 1e-6 * abs(float(off["loss"])), (loss, float(off["loss"]))
    np.testing.assert_allclose(flat, off["flat"], rtol=1e-4, atol=1e-5 * float(np.abs(off["flat"]).max()))


def test_segmented_backward_deep_tiles_gamma_order():
    """The load-balance paths on sort_by='gamma' lists (the same blend
    kernels over per-tile gamma-sorted lists): both engine passes -- the
    second with the deep-tile forward and the segmented backward -- against
    the oracle composited in gamma order."""
    s = _deep_scene()
    cam = vg().look_at([0, 0, -3.0], [0, 0, 0], width=40, height=36, fov_x_deg=40.0)
    dc = np.random.default_rng(6).uniform(-1, 1, (36, 40, 3))
    flags = dict(early_stop=O.EARLY_STOP_T, alpha_cut=O.ALPHA_CUT)
    dprep = vg().prepare(s, cam, sort_by="gamma")
    out = vg().render(s, cam, sort_by="gamma", prep=dprep)
    gprep = O.prepare(s, cam, sort_by="gamma")
    knife = device_knife_mask(gprep, s, flags, out.n_contrib, dprep.n_active())
    knife_cap(int(knife.sum()), knife.size, "deep gamma backward")
    dck = dc * ~knife[..., None]
    ref = O.backward(s, cam, dck, prep=gprep)
    (g1, p1), (g2, p2) = _deep_engine_backward(dck, sort_by="gamma")
    assert p1 == (0, 0) and p2[0] == 3, (p1, p2)
    for f in GRAD_FIELDS + ["d_background"]:
        check_field(g1[f], getattr(ref, f), f"deep gamma unsegmented {f}")
        check_field(g2[f], getattr(ref, f), f"deep gamma segmented {f}")
