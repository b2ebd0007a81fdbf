"""Benchmark: Mpixels/s of the analytic rasterizer's forward+backward step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config large]
                    [--impl ours|reference] [--views V] [--no-e2e] [--no-cpu]

Workload (default `--config large`, BASELINE.json configs[2], the config the
north-star 1000x target is quoted on): N=1M Gaussians with SH-3 colour,
64 cameras at 1920x1080.  One step = every view of the config rendered
forward, L2 loss against a seeded target (fused into the backward blend),
backward, per-Gaussian finalize with gradient accumulation over the views,
and -- on N>1 GPUs -- one NCCL all-reduce of the flat gradient buffer.
Views are sharded round-robin over ranks, so total work is fixed ("strong").

`value` is device-timed with CUDA events (inputs resident in HBM), max over
ranks.  `e2e` runs the same step through the public engine API with the
scene and targets copied from pinned host memory and the gradients + loss
copied back inside the timed region.  `roofline` is for the dominant kernel
(measured live with CUDA events on the launch stream); its denominator is
the FP32 / MUFU throughput probed on this GPU at its live clock.
`cpu_baseline` is the float64 numpy oracle (a port of the reference path,
oracle/) on a bounded, seeded sample of tiles of view 0, all host cores.
`--impl reference` prints that CPU arm as the line itself.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpixels/sec fwd+bwd (render+grad)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="large",
                    choices=["tiny", "medium", "large", "opaque", "tomography"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--views", type=int, default=0, help="limit the number of views (0 = all)")
    ap.add_argument("--deterministic", action="store_true",
                    help="fixed-order gradient reductions (the drop-in backward's default)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-tiles", type=int, default=0, help="tiles in the CPU sample (0 = auto)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_config(name, views):
    from paper_2412_03378_b200 import configs
    cfg = configs.BY_NAME[name]()
    if views:
        cfg.cameras = cfg.cameras[:views]
    return cfg


# ---------------------------------------------------------------------------
# clocks sampled during the timed region


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's first sample takes ~0.1-0.5 s; wait for it so that
            # short timed regions are covered from their start
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0:
                time.sleep(0.01)
            self.lines.clear()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        # a timed region shorter than the 200 ms period may hold no sample: take
        # the next one (the clock right after the region)
        t0 = time.time()
        while not self.lines and time.time() - t0 < 1.0:
            time.sleep(0.01)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# GPU arm


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2412_03378_b200 import _lib
    from paper_2412_03378_b200.engine import Engine
    from paper_2412_03378_b200.multiview import ViewShardedStep, shard

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = load_config(args.config, args.views)
    tomo = cfg.tomography
    my_views = shard(len(cfg.cameras), ws, rank)
    eng = Engine(local, deterministic=args.deterministic)
    ds = eng.upload(cfg.scene)
    cams = cfg.cameras
    H, W = int(cams[0].height), int(cams[0].width)
    tshape = (H, W) if tomo else (H, W, 3)
    targets = {v: torch.from_numpy(cfg.target(v, tshape)).to(dev) for v in my_views}
    runner = ViewShardedStep(eng, ds, cams, targets, world=ws, rank=rank, tomography=tomo,
                             parallel=cfg.parallel, extent=cfg.extent)
    grads = runner.grads
    loss = runner.loss

    def step(scene_dev, tgts, gbuf=None):
        return runner(scene_dev, tgts)

    for _ in range(args.warmup):
        step(ds, targets, grads)
    torch.cuda.synchronize()

    fp32_peak = mufu_peak = None
    import ctypes
    fp, mu = ctypes.c_double(), ctypes.c_double()
    if _lib.load().vg_probe_peaks(local, ctypes.byref(fp), ctypes.byref(mu)) == 0:
        fp32_peak, mufu_peak = fp.value, mu.value

    # --- timed region (device time, CUDA events on the launch stream)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    l0 = sum(e.launches() for e in runner.engines)
    st = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        step(ds, targets, grads)
    e1.record(st)
    torch.cuda.synchronize()
    ms_total = e0.elapsed_time(e1)
    launches = sum(e.launches() for e in runner.engines) - l0
    clk = clocks.stop()
    # per-kernel breakdown: a separate pass with per-launch events (vg_profile),
    # outside the timed region; consecutive views' blends run on one stream
    # here, so each launch's event interval is its own (in the timed steps
    # they alternate over two streams and overlap)
    blend2, runner.blend2 = runner.blend2, None
    for e in runner.engines:
        e.ctx.profile(True)
    for _ in range(args.steps):
        step(ds, targets, grads)
    torch.cuda.synchronize()
    runner.blend2 = blend2
    prof = {}
    for e in runner.engines:
        for k, (ms, cnt) in e.ctx.profile_read().items():
            a, b = prof.get(k, (0.0, 0))
            prof[k] = (a + ms, b + cnt)
        e.ctx.profile(False)
    loss_val = float(loss) / (len(cams) * math.prod(tshape))
    if ws > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t)
        if ws > 1:
            dist.barrier()
    ms_step = ms_total / args.steps
    px_step = len(cams) * H * W
    value = px_step / (ms_step * 1e-3) / 1e6

    # --- end to end: host buffers in, host buffers out
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, cfg, eng, my_views, tshape, dev, ws, step, runner)

    result = None
    if rank == 0:
        kernels = {k: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps}
                   for k, v in prof.items() if v[1]}
        roof = build_roofline(prof, args.steps, eng, ds, cams, my_views, tomo, cfg,
                              fp32_peak, mufu_peak, args.config)
        result = {
            "metric": METRIC, "value": round(value, 3), "unit": "Mpixels/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Philox, BASELINE.json config shapes/distributions)",
            "config": {"workload": cfg.description,
                       "views_per_step": len(cams), "pixels_per_step": px_step,
                       "gaussians": len(cfg.scene), "parallelism": f"views sharded over {ws} GPU(s)",
                       "l2_flush": "inputs larger than L2 (scene + SH coefficients > 126 MB)",
                       "gradient_reduction": "deterministic (fixed order)" if args.deterministic
                       else "atomic"},
            "e2e": e2e, "gpu_launches": launches, "clocks": clk, "kernels": kernels,
            "roofline": roof, "loss": loss_val,
        }
    return result


def run_e2e(args, cfg, eng, my_views, tshape, dev, ws, step, runner):
    """The step through the public host-fed API (multiview.HostFedStep): the
    scene and this rank's targets uploaded from pinned host memory and the
    flat gradient buffer + loss downloaded, every step, double-buffered so the
    copies overlap the neighbouring steps' kernels."""
    import torch
    from paper_2412_03378_b200.multiview import HostFedStep
    s = cfg.scene
    host = {k: torch.from_numpy(np.ascontiguousarray(getattr(s, k))).pin_memory()
            for k in ("means", "scales", "rotations", "thetas", "colors")}
    if s.sh is not None:
        host["sh"] = torch.from_numpy(np.ascontiguousarray(s.sh)).pin_memory()
    htgt = {v: torch.from_numpy(cfg.target(v, tshape)).pin_memory() for v in my_views}
    fed = HostFedStep(runner, host, htgt, lookahead=True, download_ctas=None)
    for _ in range(max(1, args.warmup)):
        fed.step()
    fed.drain()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        fed.step()
    fed.drain()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t)
    px = len(cfg.cameras) * int(cfg.cameras[0].height) * int(cfg.cameras[0].width)
    return {"value": round(px / (ms * 1e-3) / 1e6, 3), "unit": "Mpixels/s",
            "h2d_bytes_per_step": int(fed.h2d_bytes()), "d2h_bytes_per_step": int(fed.d2h_bytes()),
            "ms_per_step": round(ms, 3),
            "api": "multiview.HostFedStep(lookahead=True): every step uploads its scene + targets and downloads grads + loss, double-buffered and overlapped with compute (gradient buffers >= 64 MB by an 8-CTA streaming kernel); the timed region holds K uploads and K downloads"}


def build_roofline(prof, steps, eng, ds, cams, my_views, tomo, cfg, fp32_peak, mufu_peak, cfg_name):
    """Roofline of the dominant blend kernel from this run's CUDA-event times.

    The blend kernels are neither HBM- nor tensor-core-bound (ncu: DRAM
    throughput ~3%, no MMA); they are instruction-issue-bound (no single pipe
    saturated), so the roofline is the SM issue rate, 148 SMs x 4 schedulers
    x 1 warp-instruction / clock at the live clock.
    Algorithmic units, counted in an untimed pass over this rank's views:
    render -- V = visible (entry, 64-pixel warp block) pairs, what the
    backward walks (one warp iteration each), plus A = active pair-pixels
    and L = live pair-pixels; tomography -- the binned
    (tile, Gaussian) pairs, one thread walking the tile's 256 pixels each.
    achieved = (ncu warp instructions per unit of the profiled view of this
    config, profiles/traffic.json) x units per step / the kernel's CUDA-event
    time per step."""
    import torch
    kinds = ("tomo_fwd", "tomo_bwd") if tomo else ("render_fwd", "render_bwd")
    dom = max(kinds, key=lambda k: prof.get(k, (0, 0))[0])
    ms, cnt = prof.get(dom, (0.0, 0))
    if not cnt:
        return None
    tr = load_traffic(cfg_name, dom) or {}
    pv = tr.get("view", 0)
    A = L = U = 0.0
    U_prof = None
    for v in my_views if pv in my_views else list(my_views) + [pv]:
        if tomo:
            eng.prepare(ds, cams[v], tomo=True, parallel=cfg.parallel, extent=cfg.extent)
            u = eng.pair_count()
        else:
            eng.prepare(ds, cams[v])
            _, _, nc = eng.forward()
            u = eng.visible_pairs()
        if v == pv:
            U_prof = u
        if v in my_views:
            U += u
            if not tomo:
                A += float(eng.n_active().double().sum())
                L += float(nc.double().sum())
    torch.cuda.synchronize()
    t = ms * 1e-3 / steps                       # seconds per step in this kernel
    launch_s = t / max(cnt / steps, 1.0)        # average duration of one launch
    unit = "binned pairs" if tomo else "visible pairs"
    out = {"kernel": dom, "unit_of_work": unit, "units_per_step": U,
           "ms_per_step": ms / steps, "launches_per_step": cnt / steps,
           "ns_per_unit": t / U * 1e9 if U else None,
           "traffic": tr.get("bytes_per_launch"),
           "traffic_source": f"profiles/traffic.json[{cfg_name}] (ncu --set full, dram read + write per launch)",
           "timing_note": "kernel time from a profiling pass with the blends of consecutive views on one "
                          "stream (in the timed steps they alternate over two streams and overlap)"}
    if not tomo:
        out.update(visible_pair_pixels_per_step=64.0 * U, active_pair_pixels_per_step=A,
                   live_pair_pixels_per_step=L)
    if tr.get("bytes_per_launch"):
        hbm = measured_hbm_gbs()
        gbs = tr["bytes_per_launch"] / launch_s / 1e9
        out["hbm_check"] = {"achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm if hbm else None,
                            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)"}
    if tr.get("warp_instructions_per_launch") and U_prof and mufu_peak:
        f_clk = mufu_peak / (148 * 16)          # live SM clock from the MUFU probe (16 ex2/clk/SM)
        issue_peak = 148 * 4 * f_clk
        ipu = tr["warp_instructions_per_launch"] / U_prof
        ach = ipu * U / t
        f_issue = ach / issue_peak
        out.update(bound="issue", achieved=ach / 1e9, peak=issue_peak / 1e9,
                   unit="G warp-instructions/s", frac=f_issue,
                   warp_instructions_per_unit=ipu,
                   peak_source="148 SMs x 4 issue/clk at the live clock (vg_probe_peaks MUFU loop / 16)",
                   ncu_pipes_pct={k: tr.get(k) for k in ("issue_active_pct", "xu_pipe_pct", "fma_pipe_pct",
                                                          "alu_pipe_pct", "lsu_pipe_pct", "occupancy_pct")})
        # the busiest pipe: ncu's pipe / issue utilisation ratio scaled to the live issue rate
        ia = tr.get("issue_active_pct") or 0.0
        if ia > 0:
            fr = {"issue": f_issue}
            for name, key in (("fma pipe", "fma_pipe_pct"), ("xu (MUFU) pipe", "xu_pipe_pct"),
                              ("alu pipe", "alu_pipe_pct")):
                if tr.get(key) is not None:
                    fr[name] = f_issue * tr[key] / ia
            out["pipe_fracs"] = fr
            top = max(fr, key=fr.get)
            if top != "issue":
                out.update(bound=top, frac=fr[top],
                           frac_note=f"{top} utilisation = live issue fraction x ncu {top} / issue-active")
    return out


def measured_hbm_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6650.0  # the profiling recipe's fallback


def load_traffic(config, kernel):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(config, {}).get(kernel)
    except (OSError, ValueError, AttributeError):
        return None


# ---------------------------------------------------------------------------
# CPU arm: float64 numpy oracle (port of the reference path) on sampled tiles


def cpu_sample(cfg, n_tiles_target, seed=0, budget_s=25.0):
    """Fwd+bwd Mpx/s of the oracle on a seeded sample of tiles of view 0,
    using every host core; the per-view preprocessing cost is prorated."""
    from oracle import volgauss_oracle as O
    threads = os.cpu_count() or 1
    s = cfg.scene
    cam = cfg.cameras[0]
    from types import SimpleNamespace
    scene = SimpleNamespace(means=s.means.astype(np.float64), scales=s.scales.astype(np.float64),
                            rotations=s.rotations.astype(np.float64), thetas=s.thetas.astype(np.float64),
                            colors=s.colors.astype(np.float64), background=np.zeros(3))
    t0 = time.perf_counter()
    if cfg.tomography:
        prep = O.tomo_prepare(scene, cam, cfg.parallel, cfg.extent)
    else:
        prep = O.prepare(scene, cam)
    t_prep = time.perf_counter() - t0
    n_all = prep.tiles_x * prep.tiles_y
    rng = np.random.default_rng(seed)
    order = rng.permutation(n_all)
    H, W = cam.height, cam.width
    tshape = (H, W) if cfg.tomography else (H, W, 3)
    target = cfg.target(0, tshape).astype(np.float64)
    done_px = 0
    t_work = 0.0
    used = []
    for start in range(0, n_all, max(threads, 8)):
        chunk = [int(t) for t in order[start:start + max(threads, 8)]]
        t1 = time.perf_counter()
        if cfg.tomography:
            img = O.tomo_forward(scene, cam, prep=prep, threads=threads, tiles=chunk)
            mask = _tile_mask(prep, chunk, H, W)
            O.tomo_backward(scene, cam, 2 * (img - target) * mask / (H * W), prep=prep,
                            threads=threads, tiles=chunk)
        else:
            img = O.render(scene, cam, prep=prep, threads=threads, tiles=chunk)
            mask = _tile_mask(prep, chunk, H, W)[..., None]
            O.backward(scene, cam, 2 * (img.color - target) * mask / (H * W * 3), prep=prep,
                       tiles=chunk, threads=threads)
        t_work += time.perf_counter() - t1
        used += chunk
        done_px += sum(_tile_px(prep, t, H, W) for t in chunk)
        if (n_tiles_target and len(used) >= n_tiles_target) or t_work > budget_s:
            break
    frac = done_px / (H * W)
    t_eff = t_work + t_prep * frac
    return {"value": done_px / t_eff / 1e6, "unit": "Mpixels/s", "cores": threads, "kind": "port",
            "sample": (f"{len(used)} seeded-random 16x16 tiles ({done_px} px) of view 0 of "
                       f"{cfg.name}, fwd+bwd, float64 numpy oracle/ (port of raster/grad"
                       f"{'/tomo' if cfg.tomography else ''}.py); per-view prepare "
                       f"{t_prep:.1f}s prorated by pixel fraction"),
            "seconds": round(t_eff, 2)}


def _tile_px(prep, t, H, W):
    ty, tx = divmod(t, prep.tiles_x)
    return min(16, H - ty * 16) * min(16, W - tx * 16)


def _tile_mask(prep, tiles, H, W):
    m = np.zeros((H, W))
    for t in tiles:
        ty, tx = divmod(t, prep.tiles_x)
        m[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16] = 1.0
    return m


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    cfg = load_config(args.config, args.views)
    samples = []
    for i in range(args.warmup + args.steps):
        warm = i < args.warmup
        r = cpu_sample(cfg, 8 if warm else (args.cpu_tiles or 64), seed=i,
                       budget_s=3.0 if warm else 12.0)
        if not warm:
            samples.append(r)
    val = statistics.mean(r["value"] for r in samples)
    ms_step = len(cfg.cameras) * cfg.cameras[0].height * cfg.cameras[0].width / (val * 1e6) * 1e3
    return {"metric": METRIC, "value": round(val, 6), "unit": "Mpixels/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Philox, BASELINE.json config shapes/distributions)",
            "impl": "reference",
            "config": {"workload": cfg.description, "views_per_step": len(cfg.cameras)},
            "cpu_baseline": {k: samples[-1][k] for k in ("unit", "cores", "kind", "sample")} | {"value": round(val, 6)},
            "e2e": {"value": round(val, 6), "unit": "Mpixels/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    if args.impl == "reference":
        res = run_reference(args)
        if res is not None:
            print(json.dumps(res))
        return
    res = run_gpu(args)
    ws, rank, _ = dist_env()
    if rank == 0:
        if not args.no_cpu and ws == 1:
            cfg = load_config(args.config, args.views)
            res["cpu_baseline"] = cpu_sample(cfg, args.cpu_tiles or 0, budget_s=15.0)
        print(json.dumps(res))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
