"""Where does the host-fed (e2e) step lose time against the device step?
Times config 3 with: device-resident inputs; HostFedStep with lookahead; and
HostFedStep variants with the scene / target uploads or the download dropped."""
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import load_config  # noqa: E402
from paper_2412_03378_b200.engine import Engine  # noqa: E402
from paper_2412_03378_b200.multiview import HostFedStep, ViewShardedStep  # noqa: E402


def timed(fn, steps=6, warm=3):
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


class Variant(HostFedStep):
    def __init__(self, *a, scene=True, tgt=True, down=True, **k):
        super().__init__(*a, **k)
        self.v_scene, self.v_tgt, self.v_down = scene, tgt, down
        if not scene:
            self.names = []
        if not tgt:
            self.host_targets_saved = self.host_targets
        if not down:
            self.grads_host = self.grads_host[:1]
            self.grads_dev_view = True

    def step(self):
        if self.v_down:
            return super().step()
        # same as HostFedStep.step without the gradient download
        torch_ = torch
        s = self.k % 2
        main = torch_.cuda.current_stream(self.runner.eng.device)
        if not self.staged[s]:
            self._upload(s)
        self.staged[s] = False
        if self.lookahead:
            nxt = (self.k + 1) % 2
            self._upload(nxt)
            self.staged[nxt] = True
        main.wait_event(self.scene_up[s])
        self.runner(self.ds[s], self.tg[s], ready=self.tgt_up[s], grads=self.grads[s], loss=self.loss[s])
        self.computed[s].record(main)
        self.used[s] = True
        self.k += 1

    def _upload(self, s):
        if not self.v_tgt:
            with torch.cuda.stream(self.up):
                for name in self.names:
                    dst = getattr(self.ds[s], name)
                    dst.copy_(self.host_scene[name].view(dst.shape), non_blocking=True)
                self.scene_up[s].record(self.up)
                for v in self.host_targets:
                    self.tgt_up[s][v].record(self.up)
            return
        super()._upload(s)


def main():
    cfg = load_config(sys.argv[1] if len(sys.argv) > 1 else "large", None)
    dev = torch.device("cuda", 0)
    eng = Engine(0)
    ds = eng.upload(cfg.scene)
    cams = cfg.cameras
    H, W = int(cams[0].height), int(cams[0].width)
    views = range(len(cams))
    htgt = {v: torch.from_numpy(cfg.target(v, (H, W, 3))).pin_memory() for v in views}
    targets = {v: t.to(dev) for v, t in htgt.items()}
    runner = ViewShardedStep(eng, ds, cams, targets)
    s = cfg.scene
    host = {k: torch.from_numpy(np.ascontiguousarray(getattr(s, k))).pin_memory()
            for k in ("means", "scales", "rotations", "thetas", "colors")}
    if s.sh is not None:
        host["sh"] = torch.from_numpy(np.ascontiguousarray(s.sh)).pin_memory()
    print("device step        %.2f ms" % timed(lambda: runner(ds, targets)))
    for name, kw in [("fed lookahead", {}), ("fed no downloads", dict(down=False)),
                     ("fed no uploads", dict(scene=False, tgt=False)),
                     ("fed no copies", dict(scene=False, tgt=False, down=False)),
                     ("fed kernel dl 8", dict(download_ctas=8)),
                     ("fed kernel dl 4", dict(download_ctas=4)),
                     ("fed kernel dl 2", dict(download_ctas=2))]:
        fed = Variant(runner, host, htgt, lookahead=True, **kw)

        def f():
            fed.step()
        ms = timed(f)
        fed.drain()
        print("%-18s %.2f ms" % (name, ms))
    print("device step again  %.2f ms" % timed(lambda: runner(ds, targets)))
    # raw copy bandwidth
    big = torch.empty(htgt[0].numel() * 16, dtype=torch.float32).pin_memory()
    dbig = torch.empty_like(big, device=dev)
    ms = timed(lambda: dbig.copy_(big, non_blocking=True), 3, 1)
    print("H2D %.1f GB/s" % (big.numel() * 4 / ms / 1e6))
    ms = timed(lambda: big.copy_(dbig, non_blocking=True), 3, 1)
    print("D2H %.1f GB/s" % (big.numel() * 4 / ms / 1e6))


if __name__ == "__main__":
    main()
