"""Runs many multi-view steps of a config on identical inputs and checks that
the loss and the gradient norm stay put (atomic-order noise only): a guard
against stream-ordering hazards in the pipelined, dual-stream step."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import load_config  # noqa: E402
from paper_2412_03378_b200.engine import Engine  # noqa: E402
from paper_2412_03378_b200.multiview import ViewShardedStep  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "large"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
det = len(sys.argv) > 3 and sys.argv[3] == "det"
cfg = load_config(name, None)
eng = Engine(0, deterministic=det)
ds = eng.upload(cfg.scene)
cams = cfg.cameras
H, W = int(cams[0].height), int(cams[0].width)
shape = (H, W) if cfg.tomography else (H, W, 3)
targets = {v: torch.from_numpy(cfg.target(v, shape)).cuda() for v in range(len(cams))}
step = ViewShardedStep(eng, ds, cams, targets, tomography=cfg.tomography, parallel=cfg.parallel,
                       extent=cfg.extent)
losses, norms, first = [], [], None
for k in range(steps):
    loss = float(step())
    g = step.grads.flat
    norms.append(float(g.double().norm()))
    losses.append(loss)
    if det:
        if first is None:
            first = g.clone()
        elif not torch.equal(first, g):
            print(f"{name} det: step {k} gradients differ bitwise")
            sys.exit(1)
rl = (max(losses) - min(losses)) / abs(losses[0])
rn = (max(norms) - min(norms)) / norms[0]
print(f"{name}{' det' if det else ''}: {steps} steps, loss spread {rl:.2e}, grad-norm spread {rn:.2e}")
sys.exit(0 if rl < 1e-6 and rn < 1e-4 else 1)
