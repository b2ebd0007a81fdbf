"""The N>1 path on CPU: two gloo ranks shard the views of a small scene,
each computes its views' gradients (float64 oracle standing in for the GPU
engine), accumulates them into one flat buffer and all-reduces it.  The
reduced buffer on every rank must equal the serial sum over all views, and
the per-primitive `visible` flags the OR over all views (so every rank's
GradAccum / densify inputs agree)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

N_VIEWS = 5


def _scene_and_cams():
    from types import SimpleNamespace

    from paper_2412_03378_b200 import configs
    cfg = configs.medium(n=60, size=24, n_views=N_VIEWS)
    s = cfg.scene
    scene = SimpleNamespace(means=s.means.astype(np.float64), scales=s.scales.astype(np.float64),
                            rotations=s.rotations.astype(np.float64),
                            thetas=s.thetas.astype(np.float64), colors=s.colors.astype(np.float64),
                            background=np.zeros(3))
    return cfg, scene


def _view_grads(cfg, scene, v):
    """Flat per-view gradient in the GradBuffers layout (float64)."""
    from oracle import volgauss_oracle as O
    cam = cfg.cameras[v]
    img = O.render(scene, cam)
    target = cfg.target(v, (cam.height, cam.width, 3)).astype(np.float64)
    loss, d_img = O.l2_loss_and_grad(img.color, target)
    g = O.backward(scene, cam, d_img)
    flat = np.concatenate([g.d_means.ravel(), g.d_scales.ravel(), g.d_rotations.ravel(),
                           g.d_thetas.ravel(), g.d_colors.ravel(), g.d_kappas.ravel(),
                           g.d_background.ravel()])
    return flat, loss * img.color.size, np.asarray(g.visible, dtype=np.uint8)


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    from paper_2412_03378_b200.multiview import shard, sharded_step
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    cfg, scene = _scene_and_cams()
    views = shard(N_VIEWS, world, rank)
    size = len(_view_grads(cfg, scene, 0)[0])
    flat = torch.zeros(size, dtype=torch.float64)
    loss = torch.zeros((), dtype=torch.float64)
    visible = torch.zeros(len(scene.means), dtype=torch.uint8)

    def view_fn(v, accumulate):
        g, l, vis = _view_grads(cfg, scene, v)
        if accumulate:
            flat.add_(torch.from_numpy(g))
            visible.copy_(torch.maximum(visible, torch.from_numpy(vis)))
        else:
            flat.copy_(torch.from_numpy(g))
            visible.copy_(torch.from_numpy(vis))
        loss.add_(l)

    sharded_step(views, view_fn, flat, loss, visible=visible)
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.append(flat.numpy(), float(loss)))
    np.save(os.path.join(out_dir, f"rank{rank}_visible.npy"), visible.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_covers_every_view_once():
    from paper_2412_03378_b200.multiview import shard
    for world in (1, 2, 3, 4, 8):
        got = sorted(v for r in range(world) for v in shard(64, world, r))
        assert got == list(range(64))
        sizes = [len(shard(64, world, r)) for r in range(world)]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


@pytest.mark.parametrize("world", [2, 3, 6])   # 6 > 5 views: one rank renders nothing
def test_gloo_allreduce_equals_serial_sum(tmp_path, world):
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       start_method="spawn", join=True)
    cfg, scene = _scene_and_cams()
    per_view = [_view_grads(cfg, scene, v) for v in range(N_VIEWS)]
    serial = sum(p[0] for p in per_view)
    serial_loss = sum(p[1] for p in per_view)
    serial_vis = np.max([p[2] for p in per_view], axis=0)
    assert 0 < serial_vis.sum() < len(serial_vis) or serial_vis.all()
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npy")
        np.testing.assert_allclose(got[:-1], serial, rtol=1e-12, atol=1e-14)
        assert got[-1] == pytest.approx(serial_loss, rel=1e-12)
        np.testing.assert_array_equal(np.load(tmp_path / f"rank{r}_visible.npy"), serial_vis)
