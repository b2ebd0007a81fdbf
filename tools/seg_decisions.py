"""Per-view load-balance decisions of one engine context over a config's
first 16 views (vg_debug_segments: bit 0 segmented backward, bit 1 deep-tile
forward).  python tools/seg_decisions.py opaque
"""
import sys, ctypes
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import torch
from paper_2412_03378_b200 import configs, _lib as L
from paper_2412_03378_b200.engine import Engine
cfg = getattr(configs, sys.argv[1])()
eng = Engine(); ds = eng.upload(cfg.scene)
H, W = cfg.cameras[0].height, cfg.cameras[0].width
out = []
for v in range(min(16, len(cfg.cameras))):
    eng.prepare(ds, cfg.cameras[v])
    c, t, _ = eng.forward(counts=False)
    g = eng.new_grads(ds)
    tgt = torch.from_numpy(cfg.target(v, (H, W, 3))).cuda()
    eng.backward_l2(c, t, tgt, g)
    torch.cuda.synchronize()
    n, f = ctypes.c_int64(), ctypes.c_int32()
    L.check(L.load().vg_debug_segments(eng.ctx.handle, ctypes.byref(n), ctypes.byref(f)), "seg")
    out.append(f.value)
print(sys.argv[1], "decisions (bit0 seg bwd, bit1 deep fwd):", out)
