"""The N>1 step on the GPU: the production multi-view step
(multiview.ViewShardedStep) run as two ranks, and the NCCL exchange of the
C ABI (vg_allreduce_grads).

Only one GPU is available here, so the two-rank run puts both ranks on
cuda:0 with the gloo backend (the collective runs on the host between the
steps; no rank's kernel waits on another's): each rank renders its shard of
the views, and the reduced gradient, `visible` flags and loss must equal the
one-rank step over all views (the reference's per-view sum,
optim.py:367-378).  NCCL itself is exercised with a one-rank communicator
(NCCL refuses two ranks on one device)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import ROOT, cuda_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]

N_VIEWS = 5


def _setup(det):
    import torch
    from paper_2412_03378_b200 import configs
    from paper_2412_03378_b200.engine import Engine
    cfg = configs.large(n=4000, width=96, height=64, n_views=N_VIEWS)
    eng = Engine(deterministic=det)
    ds = eng.upload(cfg.scene)
    targets = {v: torch.from_numpy(cfg.target(v, (64, 96, 3))).cuda() for v in range(N_VIEWS)}
    return cfg, eng, ds, targets


def _rank(rank, world, port, out_dir, det):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2412_03378_b200.multiview import ViewShardedStep
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    cfg, eng, ds, targets = _setup(det)
    mine = {v: t for v, t in targets.items() if v % world == rank}
    step = ViewShardedStep(eng, ds, cfg.cameras, mine, world=world, rank=rank)
    assert step.views == sorted(mine)
    for _ in range(2):                       # the second step must start from clean accumulators
        loss = float(step())
    torch.cuda.synchronize()
    np.save(os.path.join(out_dir, f"flat{rank}.npy"), step.grads.flat.cpu().numpy())
    np.save(os.path.join(out_dir, f"vis{rank}.npy"), step.grads.visible.cpu().numpy())
    np.save(os.path.join(out_dir, f"loss{rank}.npy"), np.array([loss]))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("det", [False, True])
def test_view_sharded_step_two_ranks_equals_one_rank(tmp_path, det):
    import torch
    import torch.multiprocessing as mp
    from paper_2412_03378_b200.multiview import ViewShardedStep
    world = 2
    mp.start_processes(_rank, args=(world, _free_port(), str(tmp_path), det), nprocs=world,
                       start_method="spawn", join=True)
    cfg, eng, ds, targets = _setup(det)
    step = ViewShardedStep(eng, ds, cfg.cameras, targets)
    loss = float(step())
    ref = step.grads.flat.cpu().numpy().astype(np.float64)
    vis = step.grads.visible.cpu().numpy()
    torch.cuda.synchronize()
    assert vis.any() and not vis.all()
    scale = np.abs(ref).max()
    for r in range(world):
        got = np.load(tmp_path / f"flat{r}.npy").astype(np.float64)
        # the same per-view sums, added in another order (two partial sums)
        np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-6 * scale)
        np.testing.assert_array_equal(np.load(tmp_path / f"vis{r}.npy"), vis)
        assert float(np.load(tmp_path / f"loss{r}.npy")[0]) == pytest.approx(loss, rel=1e-12)
    # both ranks hold the same (reduced) buffer
    np.testing.assert_array_equal(np.load(tmp_path / "flat0.npy"), np.load(tmp_path / "flat1.npy"))


def test_nccl_allreduce_grads_single_rank_is_identity():
    """vg_allreduce_grads through a real NCCL communicator (one rank): the
    in-place sum / max over one rank leaves flat, visible and loss unchanged,
    and the step with the communicator equals the step without."""
    import torch
    from paper_2412_03378_b200 import _lib
    from paper_2412_03378_b200.multiview import NcclComm, ViewShardedStep
    assert _lib.load().vg_nccl_available() == 1
    comm = NcclComm(torch.device("cuda", 0))
    try:
        flat = torch.randn(1 << 20, device="cuda")
        vis = (torch.rand(1000, device="cuda") > 0.5).to(torch.uint8)
        loss = torch.tensor(3.25, dtype=torch.float64, device="cuda")
        f0, v0 = flat.clone(), vis.clone()
        comm.allreduce(flat, vis, loss)
        torch.cuda.synchronize()
        assert torch.equal(flat, f0) and torch.equal(vis, v0) and float(loss) == 3.25
        cfg, eng, ds, targets = _setup(True)
        a = ViewShardedStep(eng, ds, cfg.cameras, targets)
        la = float(a())
        ga = a.grads.flat.clone()
        b = ViewShardedStep(eng, ds, cfg.cameras, targets, comm=comm)
        lb = float(b())
        assert la == lb and torch.equal(ga, b.grads.flat)
    finally:
        comm.close()
