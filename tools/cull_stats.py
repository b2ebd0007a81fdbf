"""Forward culling statistics for a few views (debug entry point)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2412_03378_b200 import _lib, configs
    from paper_2412_03378_b200.engine import Engine
    name = sys.argv[1] if len(sys.argv) > 1 else "large"
    cfg = configs.BY_NAME[name]()
    eng = Engine()
    ds = eng.upload(cfg.scene)
    lib = _lib.load()
    fn = lib.vg_debug_forward_stats
    fn.restype = C.c_int
    for v in range(3):
        cam = cfg.cameras[v]
        eng.prepare(ds, cam)
        color, tfin, nc = eng.forward()
        na = eng.n_active()
        out = (C.c_ulonglong * 4)()
        fn(eng.ctx.handle, C.c_void_p(color.data_ptr()), C.c_void_p(tfin.data_ptr()),
           C.c_void_p(nc.data_ptr()), out, C.c_void_p(torch.cuda.current_stream().cuda_stream))
        A = float(na.double().sum()); L = float(nc.double().sum())
        proc, vis, tot = out[0], out[1], out[2]
        print(f"{name} view {v}: pairs {eng_pairs(eng)} warp-entries walked {tot} processed {proc} "
              f"({proc/tot:.3f}) visible {vis} ({vis/max(proc,1):.3f} of processed); "
              f"A/px-entries {A:.3e} L {L:.3e} processed px {64*proc:.3e}")


def eng_pairs(eng):
    import ctypes
    o = ctypes.c_int64()
    eng.lib.vg_pair_count(eng.ctx.handle, ctypes.byref(o))
    return o.value


if __name__ == "__main__":
    main()
