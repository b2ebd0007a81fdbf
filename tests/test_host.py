"""Host-side logic of the facade, checked on CPU: reference-compatible
argument validation, loud failure without a GPU (no CPU fallback), the
synthetic configs, and the loss helper."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2412_03378_b200 as vg
from conftest import cuda_available, load_case
from paper_2412_03378_b200 import configs


def test_mode_and_sort_validation():
    scene, cam, _ = load_case("golden_scene")
    with pytest.raises(ValueError):
        vg.render(scene, cam, mode="hybrid")
    with pytest.raises(ValueError):
        vg.render(scene, cam, sort_by="nonsense")
    with pytest.raises(NotImplementedError):
        vg.render(scene, cam, tile_size=8)


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU path")
def test_no_cpu_fallback():
    scene, cam, _ = load_case("golden_scene")
    with pytest.raises(RuntimeError):
        vg.render(scene, cam)
    with pytest.raises(RuntimeError):
        vg.tomo_forward(scene, cam)
    with pytest.raises(RuntimeError):
        vg.render(scene, cam, mode="splat")
    with pytest.raises(RuntimeError):
        vg.render(scene, cam, sort_by="gamma")


def test_scene_container_mirrors_reference():
    s = vg.Scene(means=[[0, 0, 1]], scales=[[0.1] * 3], rotations=[[1, 0, 0, 0]], thetas=[0.5],
                 colors=[[1, 0, 0]], background=(0.1, 0.2, 0.3))
    assert len(s) == 1 and s.splat_opacities.shape == (1,)
    assert s.kappas()[0] == pytest.approx(-np.log1p(-0.99 * 0.5) * 10.0)
    c = s.copy()
    c.means[0, 0] = 5
    assert s.means[0, 0] == 0
    assert len(vg.Scene.empty()) == 0


def test_composite_pixel_semantics():
    # raster.py:442-454: two layers, early stop before an entry
    color, t = vg.composite_pixel([(0.5, (1, 0, 0)), (0.5, (0, 1, 0))], (0, 0, 0))
    assert np.allclose(color, [0.5, 0.25, 0.0]) and t == 0.25
    layers = [(0.9, (1, 0, 0))] * 6 + [(1 - 1e-12, (0, 1, 0))]
    color, t = vg.composite_pixel(layers, (0, 0, 0))
    assert color[1] == 0.0 and t == pytest.approx(1e-4, rel=1e-9)


def test_loss_helper():
    rng = np.random.default_rng(0)
    a, b = rng.uniform(size=(4, 4, 3)), rng.uniform(size=(4, 4, 3))
    v, g = vg.loss_and_grad(a, b, vg.LossSpec("l2"))
    assert v == pytest.approx(np.mean((a - b) ** 2))
    assert np.allclose(g, 2 * (a - b) / a.size)
    with pytest.raises(ValueError):
        vg.loss_and_grad(a, b, vg.LossSpec("huber"))


def test_configs_deterministic_and_shaped():
    a, b = configs.tiny(), configs.tiny()
    assert np.array_equal(a.scene.means, b.scene.means)
    s = a.scene
    assert s.means.dtype == np.float32 and s.means.shape == (1024, 3)
    assert np.all((s.thetas > 0) & (s.thetas < 1))
    cam = a.cameras[0]
    assert (cam.width, cam.height) == (64, 64)
    assert np.allclose(cam.center, [0, 0, -3])
    m = configs.medium(n=2000, size=32)
    assert len(m.cameras) == 8
    assert all(np.linalg.norm(c.center) == pytest.approx(5.0) for c in m.cameras)
    t = configs.tomography(n=500, size=32, n_views=6)
    assert t.parallel and len(t.cameras) == 6
    o = configs.opaque(n=1000, size=32, n_views=2)
    assert np.allclose(o.scene.scales[:, 2], 1e-3)


@pytest.mark.parametrize("name", ["rgb", "grey"])
@pytest.mark.parametrize("kind", ["l1", "l2", "dssim", "mixed:0.2", "mixed:0.7"])
def test_losses_match_reference_golden(name, kind):
    """grad.loss_and_grad for every loss kind (grad.py:338-358, the SSIM
    gradient of metrics.py:70-95) against the reference's own values
    (tests/golden/make_golden_loss.py), on numpy and on torch (float64)."""
    import os
    import torch
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "loss.npz"))
    a, b = g[f"{name}_a"], g[f"{name}_b"]
    key = kind.replace(":", "_").replace(".", "")
    spec = vg.LossSpec.parse(kind)
    v, d = vg.loss_and_grad(a, b, spec)
    assert v == pytest.approx(float(g[f"{name}_{key}_value"]), rel=1e-12, abs=1e-15)
    np.testing.assert_allclose(d, g[f"{name}_{key}_grad"], rtol=1e-10, atol=1e-15)
    vt, dt = vg.loss_and_grad(torch.from_numpy(a), torch.from_numpy(b), spec)
    assert vt == pytest.approx(v, rel=1e-12, abs=1e-15)
    np.testing.assert_allclose(dt.numpy(), d, rtol=1e-10, atol=1e-15)
    assert vg.loss_value(a, b, spec) == v


def test_loss_default_is_the_reference_default():
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "loss.npz"))
    assert vg.LossSpec().kind == str(g["default_kind"]) == "mixed"
    assert vg.LossSpec().lam == float(g["default_lam"])
    from paper_2412_03378_b200.optim import TrainConfig
    assert TrainConfig().loss.kind == "mixed"


def test_camera_helpers_and_scene_gaussian_match_reference():
    """Camera.pixel_directions / view_to_pixel / ray_through_pixel, look_at and
    Scene.gaussian (camera.py:50-99, raster.py:85-89) against the
    reference's own outputs (tests/golden/make_golden_camera.py)."""
    import os
    from paper_2412_03378_b200.camera import look_at
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "camera.npz"))
    cam = look_at([0.7, -1.1, -2.6], [0.1, 0.2, 0.0], up=(0.0, 1.0, 0.0), width=19, height=13,
                  fov_x_deg=47.0)
    np.testing.assert_array_equal(cam.rotation, g["R"])
    np.testing.assert_array_equal(cam.translation, g["t"])
    np.testing.assert_allclose(cam.pixel_directions(), g["dirs"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(cam.view_to_pixel(g["v"]), g["px"], rtol=1e-15, atol=1e-13)
    ray = cam.ray_through_pixel(4, 11)
    np.testing.assert_allclose(ray.origin, g["ray_o"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(ray.direction, g["ray_d"], rtol=0, atol=1e-15)
    s = vg.Scene(g["s_means"], g["s_scales"], g["s_rot"], g["s_thetas"], g["s_colors"], g["s_opac"])
    p = s.gaussian(2)
    got = np.concatenate([p.mean, p.scale, p.rotation, [p.theta], p.color, [p.splat_opacity]])
    np.testing.assert_array_equal(got, g["g"])


def test_bench_multi_gpu_launch_guard():
    """`bench.py --gpus N` outside torchrun launches N ranks itself; without N
    visible GPUs it reports that as a JSON error line instead of silently
    running one rank (bench.py main)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 2, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert "error" in line and "--gpus 2" in line["error"]
