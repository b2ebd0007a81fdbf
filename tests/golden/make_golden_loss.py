"""Generate tests/golden/loss.npz by running the REFERENCE photometric losses
(volgauss 0.1.0 grad.loss_and_grad / loss_value, metrics.ssim) themselves.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src:. \\
        python tests/golden/make_golden_loss.py

Cases: a seeded 23x31x3 colour pair and a 17x20 grey pair (unit range, the
second correlated with the first so SSIM is far from 0), every loss kind
(l1, l2, dssim, mixed with lam 0.2 and 0.7): value and dL/d(image).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from volgauss import grad, metrics  # noqa: E402  (reference)


def main():
    rng = np.random.default_rng(42)
    out = {}
    for name, shape in (("rgb", (23, 31, 3)), ("grey", (17, 20))):
        a = rng.uniform(0.0, 1.0, shape)
        b = np.clip(0.7 * a + 0.3 * rng.uniform(0.0, 1.0, shape), 0.0, 1.0)
        out[f"{name}_a"], out[f"{name}_b"] = a, b
        out[f"{name}_ssim"] = np.array(metrics.ssim(a, b))
        for kind in ("l1", "l2", "dssim", "mixed:0.2", "mixed:0.7"):
            spec = grad.LossSpec.parse(kind)
            v, g = grad.loss_and_grad(a, b, spec)
            key = kind.replace(":", "_").replace(".", "")
            out[f"{name}_{key}_value"] = np.array(v)
            out[f"{name}_{key}_grad"] = g
            assert abs(grad.loss_value(a, b, spec) - v) < 1e-12
    out["default_kind"] = np.array(grad.LossSpec().kind)
    out["default_lam"] = np.array(grad.LossSpec().lam)
    np.savez_compressed(os.path.join(HERE, "loss.npz"), **out)
    print("loss.npz:", {k: float(v) for k, v in out.items() if k.endswith("_value")})


if __name__ == "__main__":
    sys.exit(main())
