"""Run one multi-view step of a config through the product step
(multiview.ViewShardedStep) -- for ncu captures.

    python tools/profile_view.py --config large --views 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="large")
    ap.add_argument("--views", type=int, default=3)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--deterministic", action="store_true")
    args = ap.parse_args()
    import torch
    from paper_2412_03378_b200 import configs
    from paper_2412_03378_b200.engine import Engine
    from paper_2412_03378_b200.multiview import ViewShardedStep
    cfg = configs.BY_NAME[args.config]()
    cams = cfg.cameras[:args.views]
    eng = Engine(deterministic=args.deterministic)
    ds = eng.upload(cfg.scene)
    H, W = cams[0].height, cams[0].width
    shape = (H, W) if cfg.tomography else (H, W, 3)
    targets = {v: torch.from_numpy(cfg.target(v, shape)).cuda() for v in range(len(cams))}
    step = ViewShardedStep(eng, ds, cams, targets, tomography=cfg.tomography,
                           parallel=cfg.parallel, extent=cfg.extent)
    for s in range(args.steps):
        loss = step()
        torch.cuda.synchronize()
        print(f"step {s}: loss {float(loss):.6f} launches {eng.launches()}")


if __name__ == "__main__":
    main()
