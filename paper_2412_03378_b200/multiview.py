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


def reduce_across_ranks(flat, loss=None, group=None, visible=None, comm=None):
    """Sum the flat gradient buffer (and the loss scalar) over all ranks and
    OR the per-primitive `visible` flags (max of uint8), so every rank holds
    the gradient of all views and the same GradAccum / densify inputs.  With
    an NcclComm the three reductions run as one NCCL group through the C ABI
    (vg_allreduce_grads); otherwise through torch.distributed (any backend:
    gloo on CPU tests).  A no-op for one rank."""
    if comm is not None:
        comm.allreduce(flat, visible, loss)
        return
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return
    if dist.get_world_size(group) == 1:
        return
    dist.all_reduce(flat, group=group)
    if visible is not None:
        dist.all_reduce(visible, op=dist.ReduceOp.MAX, group=group)
    if loss is not None:
        dist.all_reduce(loss, group=group)


class NcclComm:
    """An NCCL communicator over the ranks of a torch.distributed group, owned
    by the C ABI (vg_nccl_comm_init); rank 0's unique id travels over the
    group (any backend).  allreduce() runs vg_allreduce_grads on the current
    CUDA stream: the step's only data exchange."""

    def __init__(self, device, group=None):
        import ctypes
        import torch
        import torch.distributed as dist
        from . import _lib
        self.torch = torch
        self.lib = _lib.load()
        self.device = torch.device(device)
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _lib.check(self.lib.vg_nccl_unique_id(uid), "vg_nccl_unique_id")
        if self.world > 1:
            box = [bytes(uid.raw)]
            dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0, group=group)
            uid = ctypes.create_string_buffer(box[0], 128)
        self.handle = ctypes.c_void_p()
        _lib.check(self.lib.vg_nccl_comm_init(ctypes.byref(self.handle), self.world, uid, self.rank,
                                              self.device.index or 0), "vg_nccl_comm_init")

    def allreduce(self, flat, visible=None, loss=None):
        from . import _lib
        st = self.torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(self.lib.vg_allreduce_grads(
            None, self.handle, _lib.ptr(flat), flat.numel(), _lib.ptr(visible),
            visible.numel() if visible is not None else 0, _lib.ptr(loss), st), "vg_allreduce_grads")

    def close(self):
        if self.handle:
            self.lib.vg_nccl_comm_destroy(self.handle)
            self.handle = None


def sharded_step(views, view_fn, flat, loss, group=None, finish=None, visible=None):
    """Run view_fn(view, accumulate) for this rank's views (the first one
    overwrites, the rest accumulate into `flat`), call finish() once (the
    deferred per-Gaussian parameter chain, if any), then all-reduce."""
    loss.zero_()
    if not views:
        flat.zero_()
        if visible is not None:
            visible.zero_()
    for j, v in enumerate(views):
        view_fn(v, j > 0)
    if finish is not None:
        finish()
    reduce_across_ranks(flat, loss, group, visible=visible)
    return loss


class ViewShardedStep:
    """One training step of the analytic rasterizer over a camera set, on
    this rank's share of the views.

    Three device contexts (engine.Engine) rotate over the views: the binning
    of the next views (projection, depth sort, span binning) runs on a
    high-priority side stream while earlier views blend, and consecutive
    views blend on two alternating streams so their kernels overlap (atomic
    mode).  The binning kernels are latency-bound and fill the issue slots
    the compute-bound blend kernels leave free, and the one host wait of the
    pipeline (the pair count that sizes the lists) happens while the GPU is
    busy.  Every context defers the float64 parameter chain, which runs once
    per step per context (vg_finalize_grads adds them into the same flat
    buffer)."""

    def __init__(self, engine, dscene, cameras, targets, *, world=1, rank=0, tomography=False,
                 parallel=False, extent=1.6, group=None, pipeline=True, contexts=None, comm=None):
        import torch
        from .engine import Engine
        self.torch = torch
        self.eng = engine
        self.engines = [engine]
        import os
        # contexts in flight: binning runs up to (contexts - 1) views ahead of the blend
        n_ctx = contexts if contexts is not None else int(os.environ.get("VG_CONTEXTS", "3"))
        for _ in range((max(2, n_ctx) if pipeline else 1) - 1):
            self.engines.append(Engine(engine.ctx.device, *engine.flags,
                                       deterministic=engine.deterministic, sort_by=engine.sort_by,
                                       mode=engine.mode))
        self.ds = dscene
        self.cams = cameras
        self.targets = targets
        self.views = shard(len(cameras), world, rank)
        self.tomo = tomography
        self.parallel = parallel
        self.extent = extent
        self.group = group
        self.comm = comm                            # NcclComm: the exchange through the C ABI
        self.grads = engine.new_grads(dscene)
        self.loss = torch.zeros((), dtype=torch.float64, device=engine.device)
        self.ready = None
        dev = engine.device
        # binning stream: high priority so its short CTAs interleave with the blend kernels
        import os
        prio = int(os.environ.get("VG_SIDE_PRIORITY", "-1"))
        overlap = pipeline and os.environ.get("VG_OVERLAP", "1") != "0"  # "0": serial A/B timing
        self.side = torch.cuda.Stream(device=dev, priority=prio) if overlap else None
        self.ev_binned = [torch.cuda.Event() for _ in self.engines]
        self.ev_free = [torch.cuda.Event() for _ in self.engines]
        # Odd views blend on a second stream, so consecutive views' blend kernels
        # overlap: a tile CTA whose warps finish at different depths (early
        # termination) or a short grid's tail no longer idles SMs.  Measured
        # (3 contexts): config 4 49.6 -> 34.5 ms/step, config 2 -5 %, config 5
        # -2.3 %, config 3 -0.4 %.  Deterministic contexts defer their per-view
        # d_background / loss sums per context (summed in view order, contexts
        # added in a fixed order), so they overlap too (VG_DUAL_BLEND=0: off).
        self.blend2 = (torch.cuda.Stream(device=dev)
                       if self.side is not None and os.environ.get("VG_DUAL_BLEND", "1") != "0"
                       else None)

    def _blend_stream(self, j):
        """Blend stream of the j-th view of the step: alternating when dual."""
        main = self.torch.cuda.current_stream(self.eng.device)
        return self.blend2 if (self.blend2 is not None and j % 2) else main

    def _bin(self, i, v):
        """Bin view v on context i (side stream when pipelining)."""
        eng = self.engines[i]
        kw = dict(tomo=True, parallel=self.parallel, extent=self.extent) if self.tomo else {}
        if self.side is None:
            eng.prepare(self.ds, self.cams[v], **kw)
            return
        with self.torch.cuda.stream(self.side):
            eng.prepare_async(self.ds, self.cams[v], **kw)
            eng.prepare_finish()                    # host waits for the pair count only
            self.ev_binned[i].record(self.side)

    def _blend(self, i, v, j=0):
        bs = self._blend_stream(j)
        if bs is self.blend2:
            with self.torch.cuda.stream(bs):
                self._blend_on(i, v)
        else:
            self._blend_on(i, v)

    def _blend_on(self, i, v):
        from ._lib import VG_DEFER
        eng = self.engines[i]
        main = self.torch.cuda.current_stream(eng.device)
        if self.side is not None:
            main.wait_event(self.ev_binned[i])
        if self.ready is not None and v in self.ready:
            # the target of this view is still streaming in on a copy stream
            main.wait_event(self.ready[v])
        if self.tomo:
            img = eng.tomo_forward()
            eng.tomo_backward_l2(img, self.targets[v], self.grads, accumulate=VG_DEFER,
                                 loss=self.loss)
        else:
            color, tfin, _ = eng.forward(counts=False)
            eng.backward_l2(color, tfin, self.targets[v], self.grads, accumulate=VG_DEFER,
                            loss=self.loss)
        if self.side is not None:
            self.ev_free[i].record(main)            # context i may be re-binned after this

    def _run_views(self):
        views = self.views
        self.grads.zero_()
        self._used = set()
        if not views:
            return
        ne = len(self.engines)
        self._used = set(range(min(ne, len(views))))
        if self.side is not None:
            # the scene (and zeroed buffers) come from the main stream
            self.side.wait_stream(self.torch.cuda.current_stream(self.eng.device))
        if self.blend2 is not None:
            self.blend2.wait_stream(self.torch.cuda.current_stream(self.eng.device))
        ahead = ne - 1                              # views binned ahead of the blend
        for j in range(min(ahead, len(views)) if ahead else 1):
            self._bin(j % ne, views[j])
        for j, v in enumerate(views):
            cur = j % ne
            if not ahead and j > 0:
                self._bin(cur, v)
            self._blend(cur, v, j)                  # enqueued before the host waits below
            nxt = j + ahead
            if ahead and nxt < len(views):
                i = nxt % ne
                if self.side is not None and nxt >= ne:
                    self.side.wait_event(self.ev_free[i])   # its previous view is done
                self._bin(i, views[nxt])
        if self.blend2 is not None:
            self.torch.cuda.current_stream(self.eng.device).wait_stream(self.blend2)

    def _finish(self):
        used = sorted(getattr(self, "_used", ()))
        if not used:
            return
        # one parameter-chain pass per step: the other contexts' deferred
        # accumulators are merged into the first one (in context order)
        first = self.engines[used[0]]
        for i in used[1:]:
            first.merge_deferred(self.engines[i])
        first.finalize(self.grads, accumulate=True)

    def __call__(self, dscene=None, targets=None, ready=None, grads=None, loss=None):
        """Run the step.  `ready` optionally maps view -> CUDA event that the
        view's target upload recorded (host->device copies overlap compute);
        grads / loss optionally redirect the outputs (double buffering)."""
        if dscene is not None:
            self.ds = dscene
        if targets is not None:
            self.targets = targets
        if grads is not None:
            self.grads = grads
        if loss is not None:
            self.loss = loss
        self.ready = ready
        self.loss.zero_()
        self._run_views()
        self._finish()
        reduce_across_ranks(self.grads.flat, self.loss, self.group, visible=self.grads.visible,
                            comm=self.comm)
        return self.loss


class HostFedStep:
    """A ViewShardedStep fed from pinned host memory: every step uploads the
    scene and this rank's targets and downloads the flat gradient buffer and
    the loss.  The device copies are double-buffered on two copy streams, so
    step k's uploads overlap step k-1's compute and its download overlaps
    step k+1's -- the host<->device traffic of a training loop whose data
    lives on the host, hidden behind the kernels.

        fed = HostFedStep(step, host_scene, host_targets)
        for k in range(K): fed.step()
        fed.drain()        # grads_host / loss_host hold the last step's results
    """

    def __init__(self, runner, host_scene, host_targets, lookahead=False, download_ctas=0):
        """download_ctas: 0 = copy engine, > 0 = a streaming kernel of that
        many CTAs, None = the kernel (8 CTAs) for gradient buffers of 64 MB
        and more, the copy engine below (config 3: kernel -2.7 ms per step;
        config 2's 26 MB: copy engine -0.1 ms)."""
        import torch
        from types import SimpleNamespace
        from .raster import DeviceScene
        self.torch = torch
        self.runner = runner
        dev = runner.eng.device
        self.host_scene = host_scene                    # name -> pinned tensor
        self.host_targets = host_targets                # view -> pinned tensor
        tmpl = runner.ds
        self.names = [k for k in ("means", "scales", "rotations", "thetas", "colors", "sh",
                                  "splat_opacities") if getattr(tmpl, k, None) is not None and k in host_scene]
        self.ds, self.tg, self.grads, self.loss = [], [], [], []
        for _ in range(2):
            fields = {k: getattr(tmpl, k).clone() for k in ("means", "scales", "rotations", "thetas")}
            for k in ("colors", "sh", "splat_opacities"):
                v = getattr(tmpl, k, None)
                fields[k] = v.clone() if v is not None else None
            self.ds.append(DeviceScene(SimpleNamespace(**fields, background=tmpl.background), dev.index))
            self.tg.append({v: torch.empty_like(t, device=dev) for v, t in host_targets.items()})
            self.grads.append(runner.eng.new_grads(self.ds[-1]))
            self.loss.append(torch.zeros((), dtype=torch.float64, device=dev))
        self.grads_host = torch.empty(self.grads[0].flat.shape, dtype=torch.float32).pin_memory()
        if download_ctas is None:
            download_ctas = 8 if self.grads_host.numel() * 4 >= (64 << 20) else 0
        self.loss_host = torch.empty((), dtype=torch.float64).pin_memory()
        self.up = torch.cuda.Stream(device=dev)
        self.down = torch.cuda.Stream(device=dev)
        E = torch.cuda.Event
        self.scene_up = [E(), E()]
        self.tgt_up = [{v: E() for v in host_targets} for _ in range(2)]
        self.computed = [E(), E()]
        self.downloaded = [E(), E()]
        self.k = 0
        # download_ctas > 0: the gradient download runs as a small streaming kernel
        # (evict-first loads) instead of a copy-engine transfer through L2, which
        # evicted the blend kernels' working set (config 3: -2.7 ms per step; the
        # same for uploads costs more than it saves)
        self.download_ctas = download_ctas
        self.lookahead = lookahead
        self.used = [False, False]
        self.staged = [False, False]

    def h2d_bytes(self):
        return sum(t.numel() * t.element_size() for k, t in self.host_scene.items() if k in self.names) + \
            sum(t.numel() * t.element_size() for t in self.host_targets.values())

    def d2h_bytes(self):
        return self.grads_host.numel() * 4 + 8

    def _upload(self, s):
        torch = self.torch
        if self.used[s]:
            self.up.wait_event(self.computed[s])       # slot s last read two steps ago
        with torch.cuda.stream(self.up):
            ds = self.ds[s]
            for name in self.names:
                dst = getattr(ds, name)
                dst.copy_(self.host_scene[name].view(dst.shape), non_blocking=True)
            self.scene_up[s].record(self.up)
            for v, t in self.host_targets.items():      # each view waits for its own target only
                self.tg[s][v].copy_(t, non_blocking=True)
                self.tgt_up[s][v].record(self.up)

    def step(self):
        """One step: upload (unless prefetched), run, download.  With
        lookahead, the NEXT step's inputs are read from the host buffers now
        (data-loader-style prefetch) so their upload overlaps this step."""
        torch = self.torch
        s = self.k % 2
        main = torch.cuda.current_stream(self.runner.eng.device)
        if not self.staged[s]:
            self._upload(s)
        self.staged[s] = False
        if self.lookahead:
            nxt = (self.k + 1) % 2
            self._upload(nxt)
            self.staged[nxt] = True
        main.wait_event(self.scene_up[s])
        if self.used[s]:
            main.wait_event(self.downloaded[s])        # gradients of step k-2 are out
        self.runner(self.ds[s], self.tg[s], ready=self.tgt_up[s], grads=self.grads[s],
                    loss=self.loss[s])
        self.computed[s].record(main)
        self.used[s] = True
        self.down.wait_event(self.computed[s])
        with torch.cuda.stream(self.down):
            if self.download_ctas > 0:
                from . import _lib
                g = self.grads[s].flat
                _lib.check(_lib.load().vg_copy_streaming(
                    _lib.ptr(self.grads_host), _lib.ptr(g), g.numel() * g.element_size(),
                    self.download_ctas, self.down.cuda_stream), "vg_copy_streaming")
            else:
                self.grads_host.copy_(self.grads[s].flat, non_blocking=True)
            self.loss_host.copy_(self.loss[s], non_blocking=True)
            self.downloaded[s].record(self.down)
        self.k += 1

    def drain(self):
        """Make the current stream wait for the last download (and any
        prefetched upload)."""
        cur = self.torch.cuda.current_stream(self.runner.eng.device)
        cur.wait_stream(self.down)
        cur.wait_stream(self.up)
