"""Shared fixtures.  `gpu`-marked tests need a B200 and the built extension;
everything else runs on CPU (oracle pins, host logic, ABI load checks,
gloo multi-process tests)."""

from __future__ import annotations

import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_case(name):
    """Golden case -> (scene, camera, data dict).  Scene/camera are plain
    namespaces with the reference attribute names."""
    from paper_2412_03378_b200.camera import Camera
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    d = {k: z[k] for k in z.files}
    w, h = (int(v) for v in d["cam_wh"])
    fx, fy, cx, cy, zn = (float(v) for v in d["cam_f"])
    cam = Camera(width=w, height=h, fx=fx, fy=fy, cx=cx, cy=cy, rotation=d["cam_R"],
                 translation=d["cam_t"], z_near=zn)
    if "means" in d:
        scene = SimpleNamespace(means=d["means"], scales=d["scales"], rotations=d["rotations"],
                                thetas=d["thetas"], colors=d["colors"], background=d["background"])
    else:
        scene = SimpleNamespace(means=np.zeros((0, 3)), scales=np.zeros((0, 3)),
                                rotations=np.zeros((0, 4)), thetas=np.zeros(0),
                                colors=np.zeros((0, 3)), background=d["background"])
    return scene, cam, d


def case_flags(d):
    es = float(d["flag_early_stop"])
    return dict(early_stop=None if es < 0 else es, alpha_cut=float(d["flag_alpha_cut"]))


def golden_lists(d, prefix="tiles"):
    p, o = d[f"{prefix}_prims"], d[f"{prefix}_offsets"]
    return [p[o[t]:o[t + 1]] for t in range(len(o) - 1)]


RASTER_CASES = ["tiny", "tiny_nostop", "golden_scene", "ragged", "early_stop", "lone_zero_theta",
                "lone_transmittance", "behind", "centre_tile", "mini_opaque"]
TOMO_CASES = ["tiny", "ragged", "tomo_unit"]


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture
def golden():
    return load_case
