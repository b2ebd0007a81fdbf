"""Multi-view training step, sharded over GPUs.

Views are the natural unit of parallelism: every rank holds the full
Gaussian set (replicated in HBM), renders and back-propagates its own views,
accumulates their per-Gaussian gradients into one flat float32 buffer
(grad.GradBuffers), and a single NCCL all-reduce sums that buffer (and the
loss) across ranks -- the only data exchange of the step.  The reference
never batches views (optim.py:367-378); the reduced gradient equals the sum
of its per-view SceneGrads.

The step logic is written against two callables so the same code drives
the GPU engine (production, NCCL) and the float64 oracle (CPU gloo tests).
"""

from __future__ import annotations


def shard(n_views, world, rank):
    """Round-robin view assignment: rank r owns views r, r+world, ..."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return list(range(rank, n_views, world))


def reduce_across_ranks(flat, loss=None, group=None):
    """Sum the flat gradient buffer (and the loss scalar) over all ranks with
    one collective each; a no-op outside an initialised process group."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return
    if dist.get_world_size(group) == 1:
        return
    dist.all_reduce(flat, group=group)
    if loss is not None:
        dist.all_reduce(loss, group=group)


def sharded_step(views, view_fn, flat, loss, group=None, finish=None):
    """Run view_fn(view, accumulate) for this rank's views (the first one
    overwrites, the rest accumulate into `flat`), call finish() once (the
    deferred per-Gaussian parameter chain, if any), then all-reduce."""
    loss.zero_()
    if not views:
        flat.zero_()
    for j, v in enumerate(views):
        view_fn(v, j > 0)
    if finish is not None:
        finish()
    reduce_across_ranks(flat, loss, group)
    return loss


class ViewShardedStep:
    """One training step of the analytic rasterizer over a camera set, on
    this rank's share of the views (engine.Engine on the local GPU)."""

    def __init__(self, engine, dscene, cameras, targets, *, world=1, rank=0, tomography=False,
                 parallel=False, extent=1.6, group=None):
        import torch
        self.eng = engine
        self.ds = dscene
        self.cams = cameras
        self.targets = targets
        self.views = shard(len(cameras), world, rank)
        self.tomo = tomography
        self.parallel = parallel
        self.extent = extent
        self.group = group
        self.grads = engine.new_grads(dscene)
        self.ready = None
        self.loss = torch.zeros((), dtype=torch.float64, device=engine.device)

    def _view(self, v, accumulate):
        # every view defers the float64 parameter chain to one finalize pass;
        # the flat buffer is zeroed before the first view
        from ._lib import VG_DEFER
        if not accumulate:
            self.grads.zero_()
        accumulate = VG_DEFER
        if self.ready is not None and v in self.ready:
            # the target of this view is still streaming in on a copy stream
            self.eng.torch.cuda.current_stream(self.eng.device).wait_event(self.ready[v])
        eng, cam = self.eng, self.cams[v]
        if self.tomo:
            eng.prepare(self.ds, cam, tomo=True, parallel=self.parallel, extent=self.extent)
            img = eng.tomo_forward()
            eng.tomo_backward_l2(img, self.targets[v], self.grads, accumulate=accumulate,
                                 loss=self.loss)
        else:
            eng.prepare(self.ds, cam)
            color, tfin, _ = eng.forward()
            eng.backward_l2(color, tfin, self.targets[v], self.grads, accumulate=accumulate,
                            loss=self.loss)

    def __call__(self, dscene=None, targets=None, ready=None):
        """Run the step.  `ready` optionally maps view -> CUDA event that the
        view's target upload recorded (host->device copies overlap compute)."""
        if dscene is not None:
            self.ds = dscene
        if targets is not None:
            self.targets = targets
        self.ready = ready
        return sharded_step(self.views, self._view, self.grads.flat, self.loss, self.group,
                            finish=lambda: self.eng.finalize(self.grads, accumulate=True))
