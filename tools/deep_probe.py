"""Load-balance probe of the forward blend on one view (profiling build,
-DVG_CTA_LOG=1): per-CTA span / residency and per-warp walk / staging cycles
of a training forward.  VG_FWD_GRID=k (profiling build) launches only the k
longest-list tiles, e.g. k = 148 runs the heaviest tiles alone, one per SM.

    LIBP=build/prof/libvolgauss_b200_prof.so VG_FWD_GRID=148 CFG=opaque python tools/deep_probe.py
"""
import os, sys, json
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import numpy as np
from paper_2412_03378_b200 import _lib as L
L.LIB_PATH = os.environ.get("LIBP") or __import__("paper_2412_03378_b200.build", fromlist=["build"]).build(profile=True)
import torch
from paper_2412_03378_b200 import configs
from paper_2412_03378_b200.engine import Engine
from walk_stats import cta_stats
cfg = getattr(configs, os.environ.get("CFG", "opaque"))()
eng = Engine()
ds = eng.upload(cfg.scene)
cam = cfg.cameras[0]
eng.prepare(ds, cam)
H, W = cam.height, cam.width
nt = ((H + 15) // 16) * ((W + 15) // 16)
color, tfin, ncon = eng.forward()
na = eng.n_active().cpu().numpy()
pad = np.zeros((((H + 15) // 16) * 16, ((W + 15) // 16) * 16), np.int64); pad[:H, :W] = na
d_tile = pad.reshape(pad.shape[0] // 16, 16, pad.shape[1] // 16, 16).transpose(0, 2, 1, 3).reshape(nt, 256).max(1)
ref = color.clone()
log = torch.zeros(16 * nt, dtype=torch.int64, device="cuda")
L.check(eng.lib.vg_debug_cta_log(eng.ctx.handle, L.ptr(log), nt), "log")
k = min(int(os.environ.get("VG_FWD_GRID", nt)), nt)
c2, t2, _ = eng.forward(counts=False); torch.cuda.synchronize()
st = cta_stats(log[:16 * k], k, d_tile)
same = bool(torch.equal(c2, ref)) if k == nt else None
print(json.dumps({"lib": os.path.basename(L.LIB_PATH), "grid": k, "same_as_counting_fwd": same, "fwd": st}))
