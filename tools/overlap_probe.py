"""Device-step time of config 3 with / without the per-launch profiling events
(vg_profile) -- they change how the side-stream binning interleaves with the
main-stream blends."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import load_config  # noqa: E402
from paper_2412_03378_b200.engine import Engine  # noqa: E402
from paper_2412_03378_b200.multiview import ViewShardedStep  # noqa: E402


def timed(fn, steps=5, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


cfg = load_config(sys.argv[2] if len(sys.argv) > 2 else "large", None)
dev = torch.device("cuda", 0)
eng = Engine(0)
ds = eng.upload(cfg.scene)
cams = cfg.cameras
H, W = int(cams[0].height), int(cams[0].width)
shape = (H, W) if cfg.tomography else (H, W, 3)
targets = {v: torch.from_numpy(cfg.target(v, shape)).to(dev) for v in range(len(cams))}
runner = ViewShardedStep(eng, ds, cams, targets, tomography=cfg.tomography, parallel=cfg.parallel,
                         extent=cfg.extent)
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for prof in (False, True):
    for e in runner.engines:
        e.ctx.profile(prof)
    print(tag, "profile" if prof else "plain  ", "%.2f ms" % timed(lambda: runner(ds, targets)))
