"""Host<->device transfer variants for the drop-in facade (float64 numpy in
and out, float32 on the device): which is fastest on this box.

    python tools/facade_probe.py
"""
import time

import numpy as np
import torch


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


def main():
    a = np.random.default_rng(0).uniform(size=(1920 * 1080 * 3,))
    dev = torch.device("cuda", 0)
    pin = torch.empty(a.shape, dtype=torch.float64).pin_memory()
    pin32 = torch.empty(a.shape, dtype=torch.float32).pin_memory()
    g = torch.from_numpy(a).to(dev)
    g32 = g.float()
    res = {
        "up: host astype f32 + H2D": t(lambda: torch.from_numpy(a.astype(np.float32)).to(dev)),
        "up: H2D f64 (pageable) + GPU cast": t(lambda: torch.from_numpy(a).to(dev).float()),
        "up: memcpy to pinned f64 + H2D + cast": t(lambda: (pin.numpy().__setitem__(slice(None), a), pin.to(dev, non_blocking=True).float())),
        "down: D2H f32 + host astype f64": t(lambda: g32.cpu().numpy().astype(np.float64)),
        "down: GPU cast f64 + D2H (pageable)": t(lambda: g32.double().cpu().numpy()),
        "down: D2H f32 into pinned + astype": t(lambda: (pin32.copy_(g32), pin32.numpy().astype(np.float64))),
        "down: GPU f64 into pinned + copy": t(lambda: (pin.copy_(g32.double()), pin.numpy().copy())),
        "isfinite host": t(lambda: np.isfinite(a).all()),
        "isfinite gpu": t(lambda: bool(torch.isfinite(g32).all())),
        "l2 numpy 5-pass": t(lambda: (lambda r: (float(np.mean(r * r)), 2.0 * r / r.size))(a - a[::-1])),
        "l2 numpy vdot": t(lambda: (lambda r: (float(np.vdot(r, r)) / r.size, np.multiply(r, 2.0 / r.size, out=r)))(a - a[::-1])),
    }
    for k, v in res.items():
        print(f"{v:8.2f} ms  {k}")


if __name__ == "__main__":
    main()
