"""Per-view walk statistics and load balance of the blend kernels
(diagnostic, one GPU): how deep each tile / warp block must walk its list
before every pixel stops, against what the CTA stages (whole batches) and
what the culling evaluates; and, from the per-CTA launch log of the profiling
build (build(profile=True), -DVG_CTA_LOG=1), each blend launch's span, mean
resident CTAs per SM and its longest CTAs.

    python tools/walk_stats.py [large|opaque|medium] [--views 0,1]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BATCH = 256


STRIDE = 16  # uint64 per CTA (VG_CTA_LOG_STRIDE)


def cta_stats(log, nt, d_tile):
    full = log.cpu().numpy().reshape(nt, STRIDE)
    ct = full[:, :3]
    t0 = ct[:, 0].min()
    st, en = (ct[:, 0] - t0) / 1e3, (ct[:, 1] - t0) / 1e3  # us
    sm = ct[:, 2] >> 32
    tile = ct[:, 2] & 0xffffffff
    dur = en - st
    span = en.max()
    sm_end = np.array([en[sm == k].max() if (sm == k).any() else 0 for k in range(148)])
    order = np.argsort(-dur)
    out = {
        "span_us": round(float(span), 1),
        "sum_cta_us": round(float(dur.sum()), 1),
        "mean_resident": round(float(dur.sum() / span / 148), 2),
        "cta_dur_pct_us(50,90,99,100)": [round(float(x), 1) for x in np.percentile(dur, [50, 90, 99, 100])],
        "longest(tile,depth,start,dur)": [(int(tile[i]), int(d_tile[tile[i]]), round(float(st[i]), 1),
                                           round(float(dur[i]), 1)) for i in order[:4]],
        "sm_end_pct_us(0,10,50,90,100)": [round(float(x), 1) for x in np.percentile(sm_end, [0, 10, 50, 90, 100])],
        "last_cta_start_us": round(float(st.max()), 1),
        "corr_dur_depth": round(float(np.corrcoef(dur, d_tile[tile])[0, 1]), 3),
    }
    walk, stage = full[:, 3:7].astype(np.float64), full[:, 7:11].astype(np.float64)
    if walk.any():
        # forward: per-warp cycles walking chunks / staging (incl. its barrier), longest CTAs
        out["longest_warp_cycles(walk[4],stage[4])"] = [
            (int(tile[i]), [int(x) for x in walk[i]], [int(x) for x in stage[i]]) for i in order[:3]]
        tot = walk.sum(1) + 1e-9
        out["walk_max_over_mean"] = round(float(np.mean(walk.max(1) / (tot / 4))), 3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="opaque")
    ap.add_argument("--views", default="0")
    a = ap.parse_args()
    import torch
    from paper_2412_03378_b200 import _lib as L, build
    L.LIB_PATH = build.build(profile=True)  # before the first load
    from paper_2412_03378_b200 import _lib, configs
    from paper_2412_03378_b200.engine import Engine
    cfg = getattr(configs, a.config)()
    eng = Engine()
    ds = eng.upload(cfg.scene)
    for v in [int(x) for x in a.views.split(",")]:
        cam = cfg.cameras[v]
        eng.prepare(ds, cam)
        color, tfin, ncon = eng.forward()
        na = eng.n_active().cpu().numpy()
        nc = ncon.cpu().numpy()
        H, W = na.shape
        th, tw = (H + 15) // 16, (W + 15) // 16
        pad = np.zeros((th * 16, tw * 16), np.int64)
        pad[:H, :W] = na
        tiles = pad.reshape(th, 16, tw, 16).transpose(0, 2, 1, 3).reshape(th * tw, 256)
        d_tile = tiles.max(1)
        blocks = pad.reshape(th, 2, 8, tw, 2, 8).transpose(0, 3, 1, 4, 2, 5).reshape(th * tw, 4, 64)
        d_block = blocks.max(2)
        staged = np.minimum(np.ceil(d_tile / BATCH) * BATCH, d_tile + BATCH)  # upper bound
        proc, vis, tot = eng.forward_stats()
        nt = th * tw
        log = torch.zeros(STRIDE * nt, dtype=torch.int64, device="cuda")
        _lib.check(eng.lib.vg_debug_cta_log(eng.ctx.handle, _lib.ptr(log), nt), "vg_debug_cta_log")
        color, tfin, _ = eng.forward(counts=False)  # the training forward (deep tiles when tail-bound)
        torch.cuda.synchronize()
        cta = {"fwd": cta_stats(log, nt, d_tile)}
        log.zero_()
        grads = eng.new_grads(ds)
        tgt = torch.rand(H, W, 3, device="cuda")
        eng.backward_l2(color, tfin, tgt, grads)
        torch.cuda.synchronize()
        cta["bwd"] = cta_stats(log, nt, d_tile)
        _lib.check(eng.lib.vg_debug_cta_log(eng.ctx.handle, None, 0), "vg_debug_cta_log")
        pairs = eng.pair_count()
        out = {
            "config": a.config, "view": v, "pixels": H * W, "tiles": th * tw,
            "pairs_total": pairs,
            "depth_tile_sum": int(d_tile.sum()),
            "depth_block_sum": int(d_block.sum()),
            "staged_upper": int(staged.sum()),
            "walked_per_warp (fwd stats)": tot,
            "evaluated (entry, warp)": proc,
            "visible (entry, warp)": vis,
            "n_contrib_sum": int(nc.sum()),
            "n_active_sum": int(na.sum()),
            "depth_tile_pct": [int(x) for x in np.percentile(d_tile, [10, 50, 90, 99])],
            "block_over_tile_depth": float(d_block.sum() / max(4 * d_tile.sum(), 1)),
            "evaluated_over_walked": proc / max(tot, 1),
            "visible_over_evaluated": vis / max(proc, 1),
            "cta": cta,
        }
        print(json.dumps(out))


if __name__ == "__main__":
    main()
