"""Benchmark: Mpixels/s of the analytic rasterizer's forward+backward step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config large]
                    [--impl ours|reference] [--views V] [--no-e2e] [--no-cpu]

`--gpus N` (N > 1) outside torchrun re-runs itself as N ranks under
torch.distributed.run (127.0.0.1); under torchrun the ranks come from
RANK / LOCAL_RANK / WORLD_SIZE.  Each rank renders its share of the views
and one NCCL group per step (vg_allreduce_grads through the C ABI) sums the
gradients, ORs `visible` and sums the loss.

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
copied back inside the timed region.  `roofline` is for the dominant kernel:
its SURVEY 8(d) algorithmic FP32 / MUFU work (counted per step: evaluated
and live pair-pixels x the canonical per-unit costs) over its time in an
isolated serial pass (CUDA events on the launch stream), against the FP32 /
MUFU throughput probed on this GPU at its live clock; `roofline.issue` keeps
the issue-slot view (ncu warp instructions per unit).
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
    ap.add_argument("--no-facade", action="store_true",
                    help="skip the drop-in facade leg (numpy render + backward of one view)")
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
    from paper_2412_03378_b200.multiview import NcclComm, ViewShardedStep, shard

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
        # the step's gradient exchange: one NCCL group through the C ABI
        # (vg_allreduce_grads) on the step's stream
        comm = NcclComm(dev)
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
                             parallel=cfg.parallel, extent=cfg.extent, comm=comm)
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
    # per-kernel breakdown: a separate, fully serial pass (one context, one
    # stream, no side-stream binning: VG_OVERLAP=0) with per-launch events
    # (vg_profile), outside the timed region, so every launch's event interval
    # is that kernel alone; in the timed steps binning and consecutive views'
    # blends overlap, so these times sum to more than the step
    serial = ViewShardedStep(eng, ds, cams, targets, world=ws, rank=rank, tomography=tomo,
                             parallel=cfg.parallel, extent=cfg.extent, pipeline=False)
    serial()
    torch.cuda.synchronize()
    eng.ctx.profile(True)
    for _ in range(args.steps):
        serial()
    torch.cuda.synchronize()
    prof = dict(eng.ctx.profile_read())
    eng.ctx.profile(False)
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
        kernels["_note"] = ("isolated: a serial pass (one context, one stream, VG_OVERLAP=0 equivalent) "
                            "timed per launch with CUDA events; the timed steps overlap binning and "
                            "consecutive views' blends, so these sum to more than ms_per_step")
        roof = build_roofline(prof, args.steps, eng, ds, cams, my_views, tomo, cfg,
                              fp32_peak, mufu_peak, args.config)
        result = {
            "metric": METRIC, "value": round(value, 3), "unit": "Mpixels/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "collective": ("NCCL all-reduce of the flat gradient buffer + visible OR + loss, one group "
                           "per step via vg_allreduce_grads") if ws > 1 else None,
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
    if comm is not None:
        torch.cuda.synchronize()
        comm.close()
    return result


def run_facade(args, cfg):
    """The drop-in path a reference user calls (optim.py:379-386): numpy
    scene in, prep = prepare(scene, cam); render(prep=prep); the L2 loss
    gradient on the host (numpy float64, like the reference);
    backward(prep=prep) -> float64 numpy SceneGrads.  One view of the
    config per step with RGB colour (the reference Scene has no SH);
    host<->device copies, float64<->float32 conversions and the per-call
    context all inside the timed region (wall clock around synchronised
    calls: the facade returns host arrays, so it synchronises anyway)."""
    import torch
    import paper_2412_03378_b200 as vgm
    from paper_2412_03378_b200 import configs as C
    s = cfg.scene
    scene = vgm.Scene(s.means.astype(np.float64), s.scales.astype(np.float64),
                      s.rotations.astype(np.float64), s.thetas.astype(np.float64),
                      s.colors.astype(np.float64))
    cam = cfg.cameras[0]
    H, W = int(cam.height), int(cam.width)
    target = cfg.target(0, (H, W, 3)).astype(np.float64)
    stages = {"prepare": 0.0, "render": 0.0, "loss": 0.0, "backward": 0.0}

    def once(acc):
        t0 = time.perf_counter()
        prep = vgm.prepare(scene, cam)
        t1 = time.perf_counter()
        out = vgm.render(scene, cam, prep=prep)
        t2 = time.perf_counter()
        _, d_img = vgm.loss_and_grad(out.color, target, vgm.LossSpec("l2"))
        t3 = time.perf_counter()
        g = vgm.backward(scene, cam, d_img, prep=prep, deterministic=False)
        torch.cuda.synchronize()
        t4 = time.perf_counter()
        if acc:
            for k, a, b in (("prepare", t0, t1), ("render", t1, t2), ("loss", t2, t3), ("backward", t3, t4)):
                stages[k] += b - a
        return g
    for _ in range(max(1, args.warmup)):
        once(False)
    n = max(1, args.steps)
    t0 = time.perf_counter()
    for _ in range(n):
        g = once(True)
    ms = (time.perf_counter() - t0) * 1e3 / n
    del g
    h2d = 14 * 8 * len(scene) + 3 * 8 * H * W
    d2h = (3 + 1) * 8 * H * W + 4 * H * W + 16 * 8 * len(scene)
    return {"value": round(H * W / (ms * 1e-3) / 1e6, 3), "unit": "Mpixels/s", "ms_per_view": round(ms, 3),
            "stages_ms": {k: round(v * 1e3 / n, 3) for k, v in stages.items()},
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "api": "prepare / render(prep=) / loss_and_grad (numpy) / backward(prep=, deterministic=False), "
                   "float64 numpy in and out, one view of the config with RGB colour"}


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


# SURVEY 8(d) / BASELINE.md section 4: canonical FP32 instructions and MUFU ops
# per unit of the blend kernels.  Render: per evaluated pair-pixel E (an entry
# evaluated at a pixel: 64 per (entry, 8x8 warp block) pair the kernel walks)
# plus extra FP32 per live pair-pixel L (sum of n_contrib).  Tomography: per
# binned pair-pixel B (pairs x 256): cone-beam forward 16 + 2, adjoint 45 + 2;
# parallel-beam forward 9 + 1.  The parallel-beam adjoint has no 8(d) figure:
# the parallel-beam forward's (every binned pair-pixel's Gaussian evaluated
# once) is used as its lower bound.
COSTS = {"render_fwd": {"fp32_per_E": 21, "mufu_per_E": 3, "fp32_per_L": 5},
         "render_bwd": {"fp32_per_E": 24, "mufu_per_E": 4, "fp32_per_L": 46},
         "tomo_fwd": {"fp32_per_E": 16, "mufu_per_E": 2, "fp32_per_L": 0},
         "tomo_bwd": {"fp32_per_E": 45, "mufu_per_E": 2, "fp32_per_L": 0}}
COSTS_PARALLEL = {"tomo_fwd": {"fp32_per_E": 9, "mufu_per_E": 1, "fp32_per_L": 0},
                  "tomo_bwd": {"fp32_per_E": 9, "mufu_per_E": 1, "fp32_per_L": 0,
                               "note": "no SURVEY 8(d) figure for the parallel-beam adjoint: the "
                                       "parallel-beam forward's per-B cost used as a lower bound"}}


def build_roofline(prof, steps, eng, ds, cams, my_views, tomo, cfg, fp32_peak, mufu_peak, cfg_name):
    """Roofline of the blend kernels (the dominant one first).

    Algorithmic: the kernels are FP32-issue / SFU bound (no
    tensor cores: a per-pixel exponential chain; ncu DRAM throughput ~3 %).
    Work per step is counted in an untimed pass over this rank's views:
    E = evaluated pair-pixels (64 x the (entry, warp block) pairs each kernel
    walks: the forward's culled set from a counting forward, the backward's
    forward-visible set), L = live pair-pixels (sum n_contrib), A = active
    pair-pixels (sum n_active); tomography: B = 256 x binned pairs.  FP32 =
    fp32_per_E E + fp32_per_L L, MUFU = mufu_per_E E (COSTS); the peaks are
    probed on this GPU at its live clock (vg_probe_peaks: scalar FFMA lane
    ops/s = 148 x 128 x f, MUFU ex2/s = 148 x 16 x f); t* = max(FP32 /
    P_fp32, MUFU / P_mufu) and frac = t* / t, t the kernel's time per step
    in the isolated (serial) pass.  `issue` keeps the issue-slot view (ncu
    warp instructions per unit of the profiled view, profiles/traffic.json).
    """
    import torch
    kinds = ("tomo_fwd", "tomo_bwd") if tomo else ("render_fwd", "render_bwd")
    dom = max(kinds, key=lambda k: prof.get(k, (0, 0))[0])
    if not prof.get(dom, (0, 0))[1]:
        return None
    tr_all = {k: load_traffic(cfg_name, k) or {} for k in kinds}
    pv = tr_all[dom].get("view", 0)
    A = L = 0.0
    U = {"fwd": 0.0, "bwd": 0.0}
    U_prof = None
    for v in my_views if pv in my_views else list(my_views) + [pv]:
        if tomo:
            eng.prepare(ds, cams[v], tomo=True, parallel=cfg.parallel, extent=cfg.extent)
            uf = ub = float(eng.pair_count())
        else:
            eng.prepare(ds, cams[v])
            _, _, nc = eng.forward()
            ub = float(eng.visible_pairs())
            na = eng.n_active()
            a_v, l_v = float(na.double().sum()), float(nc.double().sum())
            uf = float(eng.forward_stats()[0])
        if v == pv:
            U_prof = ub
        if v in my_views:
            U["fwd"] += uf
            U["bwd"] += ub
            if not tomo:
                A += a_v
                L += l_v
    torch.cuda.synchronize()
    px_per_unit = 256.0 if tomo else 64.0
    clock_mhz = mufu_peak / (148 * 16) / 1e6 if mufu_peak else None
    blend = {}
    for k in kinds:
        ms, cnt = prof.get(k, (0.0, 0))
        if not cnt:
            continue
        t = ms * 1e-3 / steps
        units = U["fwd" if k.endswith("fwd") else "bwd"]
        E = px_per_unit * units
        c = (COSTS_PARALLEL if tomo and cfg.parallel else COSTS)[k]
        fp32 = c["fp32_per_E"] * E + c["fp32_per_L"] * (0.0 if tomo else L)
        mufu = c["mufu_per_E"] * E
        alg = {"kernel": k, "ms_per_step": ms / steps, "launches_per_step": cnt / steps,
               "unit": "binned pair-pixels B (256 x binned pairs)" if tomo else
                       "evaluated pair-pixels E (64 x walked (entry, 8x8 block) pairs)",
               "E_per_step": E, "L_per_step": None if tomo else L,
               "fp32_per_E": c["fp32_per_E"], "fp32_per_L": c["fp32_per_L"], "mufu_per_E": c["mufu_per_E"],
               "cost_note": c.get("note"),
               "fp32_instr_per_step": fp32, "mufu_ops_per_step": mufu,
               "p_fp32_per_s": fp32_peak, "p_mufu_per_s": mufu_peak, "sm_clock_mhz_probed": clock_mhz}
        if fp32_peak and mufu_peak:
            t_fp, t_mu = fp32 / fp32_peak, mufu / mufu_peak
            t_star = max(t_fp, t_mu)
            alg.update(t_fp32_ms=t_fp * 1e3, t_mufu_ms=t_mu * 1e3, t_star_ms=t_star * 1e3,
                       bound="fp32" if t_fp >= t_mu else "mufu", frac=t_star / t)
        blend[k] = alg
    dalg = blend[dom]
    tr = tr_all[dom]
    ms, cnt = prof[dom]
    t = ms * 1e-3 / steps
    launch_s = t / max(cnt / steps, 1.0)
    out = {"kernel": dom, "bound": dalg.get("bound"), "frac": dalg.get("frac"),
           "achieved": (dalg["fp32_instr_per_step"] if dalg.get("bound") == "fp32" else dalg["mufu_ops_per_step"]) / t / 1e12
           if dalg.get("bound") else None,
           "peak": ((fp32_peak if dalg.get("bound") == "fp32" else mufu_peak) or 0) / 1e12,
           "unit": "T FP32 lane-instr/s" if dalg.get("bound") == "fp32" else "T MUFU ops/s",
           "traffic": tr.get("bytes_per_launch"),
           "traffic_source": f"profiles/traffic.json[{cfg_name}] (ncu --set full, dram read + write per launch)",
           "timing": "isolated serial pass (VG_OVERLAP=0 equivalent), CUDA events on the launch stream",
           "algorithmic": dalg, "blend_kernels": blend,
           "A_active_pair_pixels_per_step": None if tomo else A}
    if tr.get("bytes_per_launch"):
        hbm = measured_hbm_gbs()
        gbs = tr["bytes_per_launch"] / launch_s / 1e9
        out["hbm_check"] = {"achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm if hbm else None,
                            "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)"}
    if tr.get("warp_instructions_per_launch") and U_prof and mufu_peak:
        f_clk = mufu_peak / (148 * 16)          # live SM clock from the MUFU probe (16 ex2/clk/SM)
        issue_peak = 148 * 4 * f_clk
        ipu = tr["warp_instructions_per_launch"] / U_prof
        ach = ipu * U["fwd" if dom.endswith("fwd") else "bwd"] / t
        out["issue"] = {"achieved": ach / 1e9, "peak": issue_peak / 1e9, "unit": "G warp-instructions/s",
                        "frac": ach / issue_peak, "warp_instructions_per_unit": ipu,
                        "unit_of_work": "binned pairs" if tomo else "visible (entry, 8x8 block) pairs",
                        "peak_source": "148 SMs x 4 issue/clk at the live clock",
                        "ncu_pipes_pct": {k: tr.get(k) for k in ("issue_active_pct", "xu_pipe_pct",
                                                                  "fma_pipe_pct", "alu_pipe_pct",
                                                                  "lsu_pipe_pct", "occupancy_pct")}}
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
                       f"{t_prep:.1f}s prorated by pixel fraction"
                       + ("; SH-3 colour replaced by its DC band (the reference has RGB colour only; "
                          "the SH evaluation is < 0.1 % of the CPU work)" if getattr(s, "sh", None) is not None
                          else "")),
            "host_cpu": cpu_model(),
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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return f"{line.split(':', 1)[1].strip()} ({os.cpu_count()} logical CPUs)"
    except OSError:
        pass
    return f"unknown ({os.cpu_count()} logical CPUs)"


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
    # NOT timed: the whole step would take hours on the CPU; this is the step's
    # pixel count at the sampled rate
    ms_step = len(cfg.cameras) * cfg.cameras[0].height * cfg.cameras[0].width / (val * 1e6) * 1e3
    return {"metric": METRIC, "value": round(val, 6), "unit": "Mpixels/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 1),
            "ms_per_step_extrapolated": True,
            "ms_per_step_note": ("extrapolated: the step's pixels at the rate measured on the sampled tiles "
                                 "(cpu_baseline.sample); a full config-3 step would take hours on the host"),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Philox, BASELINE.json config shapes/distributions)",
            "impl": "reference", "host_cpu": cpu_model(),
            "config": {"workload": cfg.description, "views_per_step": len(cfg.cameras)},
            "cpu_baseline": {k: samples[-1][k] for k in ("unit", "cores", "kind", "sample")} | {"value": round(val, 6)},
            "e2e": {"value": round(val, 6), "unit": "Mpixels/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def launch_ranks(n):
    """`--gpus N` (N > 1) outside torchrun: re-run this command as N ranks
    under torch.distributed.run on this node (one process per GPU, NCCL);
    rank 0 prints the line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} but only {have} CUDA device(s) visible"}))
            sys.exit(2)
        launch_ranks(args.gpus)
    ws, _, _ = dist_env()
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; running {ws} rank(s)", file=sys.stderr)
    if args.impl == "reference":
        res = run_reference(args)
        if res is not None:
            print(json.dumps(res))
        return
    res = run_gpu(args)
    ws, rank, _ = dist_env()
    if rank == 0:
        if not args.no_facade and ws == 1 and args.config != "tomography":
            res["facade"] = run_facade(args, load_config(args.config, args.views))
        if not args.no_cpu and ws == 1:
            cfg = load_config(args.config, args.views)
            res["cpu_baseline"] = cpu_sample(cfg, args.cpu_tiles or 0, budget_s=15.0)
        print(json.dumps(res))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
