"""Run a few views of a config through the engine (for ncu / nsight captures).

    python tools/profile_view.py --config large --views 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="large")
    ap.add_argument("--views", type=int, default=2)
    ap.add_argument("--tomo", action="store_true")
    args = ap.parse_args()
    import torch
    from paper_2412_03378_b200 import configs
    from paper_2412_03378_b200.engine import Engine
    cfg = configs.BY_NAME[args.config]()
    eng = Engine()
    ds = eng.upload(cfg.scene)
    grads = eng.new_grads(ds)
    H, W = cfg.cameras[0].height, cfg.cameras[0].width
    shape = (H, W) if cfg.tomography else (H, W, 3)
    for v in range(args.views):
        cam = cfg.cameras[v % len(cfg.cameras)]
        tgt = torch.from_numpy(cfg.target(v, shape)).cuda()
        if cfg.tomography:
            eng.prepare(ds, cam, tomo=True, parallel=cfg.parallel, extent=cfg.extent)
            img = eng.tomo_forward()
            loss = eng.tomo_backward_l2(img, tgt, grads, accumulate=v > 0)
        else:
            eng.prepare(ds, cam)
            color, tfin, _ = eng.forward()
            loss = eng.backward_l2(color, tfin, tgt, grads, accumulate=v > 0)
        torch.cuda.synchronize()
        print(f"view {v}: loss {float(loss):.6f} pairs {eng.ctx.launches()}")


if __name__ == "__main__":
    main()
