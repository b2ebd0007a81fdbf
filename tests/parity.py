"""Parity helpers shared by the GPU tests: the tolerance contract and the
threshold-flip attribution.

Contract (BASELINE.json north star): images and gradients agree with the
float64 reference within 1e-4 absolute + 1e-3 relative in float32.  For
gradient fields the absolute term is 1e-4 of the field's largest entry
(1e-4 * max|ref|, no floor: fields of 1e-4..1e-3 such as config 1's L2
gradients are held to 1e-8..1e-7), because a float32 pipeline cannot resolve
1e-4 absolute on fields whose entries reach 1e2-1e3 and a fixed 1e-4 would
wave through fields that are themselves that small.  Pixels that exceed
the tolerance are accepted only when the oracle shows a threshold
knife-edge there (alpha_raw within CUT_BAND_REL of alpha_cut or CLAMP_BAND of
alpha_clamp, or the transmittance in front of an entry within float32 reach of
early_stop), where float32 and float64 may legitimately decide differently;
at most 0.1 % of the compared pixels may be knife edges (knife_cap).
"""

from __future__ import annotations

import numpy as np

from oracle import volgauss_oracle as O

ATOL = 1e-4
RTOL = 1e-3
# Threshold knife-edge bands: how close the float64 reference may sit to a
# threshold for the float32 device to decide the other way.  The device's
# alpha_raw agrees with the reference to ~1e-6 relative (images agree to
# ~1e-7), so: alpha_raw within 1e-5 relative of alpha_cut, within 1e-7 of the
# clamp (exp(-e) ~ 0.01 there), T within float32 reach of early_stop
# (stop_knife).
CUT_BAND_REL = 1e-5
CLAMP_BAND = 1e-7
# when a list, every check appends its measured margins here
# (tools/parity_report.py runs the GPU parity tests with it set)
RECORD = None


def _record(what, **st):
    if RECORD is not None:
        RECORD.append(dict(check=what, **st))


def image_mismatch(gpu, ref):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    bad = np.abs(gpu - ref) > ATOL + RTOL * np.abs(ref)
    if bad.ndim == 3:
        bad = bad.any(axis=2)
    return bad


def pixel_is_flip(prep, scene, row, col, flags):
    """True when the oracle's ray at (row, col) has a threshold knife-edge."""
    cut = flags.get("alpha_cut", O.ALPHA_CUT)
    stop = flags.get("early_stop", O.EARLY_STOP_T)
    clamp = flags.get("alpha_clamp", O.ALPHA_CLAMP)
    O._attach(prep, scene)
    t = (row // O.TILE) * prep.tiles_x + col // O.TILE
    ids = prep.tile_ids(t)
    if ids.size == 0:
        return False
    terms = O.ray_terms(prep, ids, np.array([row]), np.array([col]))
    raw, alpha, _ = O.clamp_cut(terms["e"], cut, clamp)
    before, active, _, _, _ = O.front_to_back(alpha, stop)
    raw, before, active = raw[:, 0], before[:, 0], active[:, 0]
    # entries that matter: the active prefix plus the first inactive one
    upto = min(int(active.sum()) + 1, len(raw))
    raw, before = raw[:upto], before[:upto]
    return bool(near_threshold(raw, before, cut, clamp, stop).any())


def near_threshold(raw, before, cut, clamp, stop):
    """Entries whose alpha_raw or transmittance-in-front sits within the
    knife-edge bands of alpha_cut / alpha_clamp / early_stop."""
    near = np.abs(raw - clamp) < CLAMP_BAND
    if cut > 0:
        near |= np.abs(raw - cut) < CUT_BAND_REL * cut
    if stop is not None and stop > 0:
        near |= stop_knife(before, stop)
    return near


def stop_knife(before, stop):
    """Transmittance within float32 reach of the early-stop threshold.  The
    device compares against stop * (1 - 2^-20) so that exact products of
    clamped alphas (e.g. (1-0.99)^2, a hair above 1e-4 in float64) decide like
    the reference; those exact cases are therefore not knife-edges."""
    return ((before >= stop * (1 - 3e-6)) & (before < stop)) | \
        ((before > stop * (1 + 1e-12)) & (before <= stop * (1 + 2e-6)))


# at most this fraction of an image's pixels may be threshold knife-edges
# (excluded from a check); at least KNIFE_MIN_PX pixels are always allowed
KNIFE_FRAC = 1e-3
KNIFE_MIN_PX = 2


def knife_cap(n_knife, n_px, what):
    """Report and cap the knife-edge pixels of one check."""
    print(f"[parity] {what}: {n_knife} knife-edge pixels of {n_px} ({n_knife / max(n_px, 1):.2e})")
    _record(what, kind="knife", knife_px=int(n_knife), pixels=int(n_px))
    assert n_knife <= max(KNIFE_MIN_PX, KNIFE_FRAC * n_px), \
        f"{what}: {n_knife}/{n_px} knife-edge pixels exceed {KNIFE_FRAC:.0e}"


def check_image(gpu, ref, prep, scene, flags, what, max_flips=None, n_px=None, knife=None):
    """Images within 1e-4 + 1e-3 |ref|; out-of-tolerance pixels must be
    knife-edges -- of `knife` (device_knife_mask) when given, else of the
    oracle's ray (pixel_is_flip) -- at most KNIFE_FRAC of the pixels (n_px:
    the pixels actually compared, default the whole image)."""
    bad = image_mismatch(gpu, ref)
    rows, cols = np.nonzero(bad)
    if knife is not None:
        unexplained = [(r, c) for r, c in zip(rows, cols) if not knife[r, c]]
    else:
        unexplained = [(r, c) for r, c in zip(rows, cols) if not pixel_is_flip(prep, scene, r, c, flags)]
    assert not unexplained, (
        f"{what}: {len(unexplained)} pixels outside tolerance without a threshold flip, "
        f"e.g. {unexplained[:5]}; max err {np.max(np.abs(np.asarray(gpu) - np.asarray(ref)))}")
    knife_cap(len(rows), bad.size if n_px is None else n_px, what)
    err = np.abs(np.asarray(gpu, dtype=np.float64) - np.asarray(ref, dtype=np.float64))
    u = err / (ATOL + RTOL * np.abs(np.asarray(ref, dtype=np.float64)))
    if u.ndim == 3:
        u = u.max(axis=2)
    _record(what, kind="image", usage=float(u[~bad].max()) if (~bad).any() else 0.0,
            max_err=float(err.max()), knife_px=len(rows), pixels=int(bad.size if n_px is None else n_px))
    if max_flips is not None:
        assert len(rows) <= max_flips, f"{what}: {len(rows)} threshold-flip pixels"
    return len(rows)


def check_field(gpu, ref, what, rtol=RTOL, atol=ATOL):
    """|gpu - ref| <= atol * max|ref| + rtol * |ref| entrywise (an all-zero
    reference field must be matched exactly)."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert gpu.shape == ref.shape, (what, gpu.shape, ref.shape)
    if ref.size == 0:
        return
    scale = float(np.max(np.abs(ref)))
    err = np.abs(gpu - ref)
    lim = atol * scale + rtol * np.abs(ref)
    bad = err > lim
    if RECORD is not None:
        _record(what, kind="field", atol=atol, rtol=rtol, **field_stats(gpu, ref))
    assert not bad.any(), (f"{what}: {int(bad.sum())}/{bad.size} entries out of tolerance; "
                           f"worst err {float(err.max()):.3e} (scale {scale:.3e}) at "
                           f"{np.unravel_index(int(np.argmax(err - lim)), err.shape)}")


def field_stats(gpu, ref):
    """Measured agreement of one field (tools/parity_report.py)."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if ref.size == 0:
        return dict(max_err=0.0, max_ref=0.0, err_over_max=0.0, max_rel=0.0, usage=0.0)
    err = np.abs(gpu - ref)
    mref = float(np.max(np.abs(ref)))
    big = (np.abs(ref) >= 1e-2 * mref) & (ref != 0)
    lim = ATOL * mref + RTOL * np.abs(ref)
    usage = float(np.max(np.where(lim > 0, err / np.where(lim > 0, lim, 1.0), np.where(err > 0, np.inf, 0.0))))
    return dict(max_err=float(err.max()), max_ref=mref,
                err_over_max=float(err.max() / mref) if mref > 0 else float(err.max()),
                max_rel=float(np.max(err[big] / np.abs(ref[big]))) if big.any() else 0.0,
                usage=usage)


def image_stats(gpu, ref, knife=None):
    """Image agreement against 1e-4 + 1e-3 |ref| per pixel; knife-edge pixels
    are counted and excluded from `usage`."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    err = np.abs(gpu - ref)
    u = err / (ATOL + RTOL * np.abs(ref))
    if knife is None:
        if u.ndim == 3:
            u = u.max(axis=2)
        k = np.zeros(u.shape, dtype=bool)
    else:
        k = np.asarray(knife, dtype=bool)
        if u.ndim == k.ndim + 1:
            u = u.max(axis=-1)
    npx = u.size
    return dict(max_err=float(err.max()) if err.size else 0.0,
                max_ref=float(np.abs(ref).max()) if ref.size else 0.0,
                usage=float(u[~k].max()) if (~k).any() else 0.0,
                usage_all=float(u.max()) if u.size else 0.0,
                out_of_tol=int((u > 1).sum()), out_of_tol_not_knife=int(((u > 1) & ~k).sum()),
                knife_px=int(k.sum()), knife_frac=float(k.sum() / max(npx, 1)), pixels=int(npx))


# running totals of device_knife_mask (diagnostics for the parity report)
STATS = dict(pixels=0, n_contrib_flips=0, n_active_flips=0, clamp_edges=0)

# wide bands: a count mismatch must sit at least this close to a threshold to
# count as a float32/float64 flip rather than a device error
WIDE_CUT_REL = 1e-4
WIDE_STOP_REL = 1e-4


def device_knife_mask(prep, scene, flags, dev_ncontrib, dev_nactive, tiles=None, alphas=None):
    """(H, W) bool: the pixels where the float32 device provably decided a
    threshold differently from the float64 oracle -- its per-pixel n_contrib
    (active entries with alpha > 0) or n_active (entries with T in front >=
    early_stop) differ from the oracle's -- plus pixels with an entry within
    CLAMP_BAND of the alpha clamp (alpha = min(alpha_raw, clamp) is
    continuous there, so no count reveals a flip of its gradient gate).
    Every count mismatch must be explained by an entry within the wide bands
    of alpha_cut / early_stop on the oracle's ray (else it is a device error
    and the assertion fails).  `alphas(prep, ids, rows, cols)` overrides the
    analytic alpha (splat mode)."""
    cut = flags.get("alpha_cut", O.ALPHA_CUT)
    stop = flags.get("early_stop", O.EARLY_STOP_T)
    clamp = flags.get("alpha_clamp", O.ALPHA_CLAMP)
    O._attach(prep, scene)
    H, W = prep.height, prep.width
    mask = np.zeros((H, W), dtype=bool)
    unexplained = []
    for t in (range(prep.tiles_x * prep.tiles_y) if tiles is None else tiles):
        ids = prep.tile_ids(t)
        if ids.size == 0:
            continue
        r0, c0, h, w, rows, cols = O._tile_box(prep, t)
        if alphas is None:
            terms = O.ray_terms(prep, ids, rows, cols)
            raw, alpha, _ = O.clamp_cut(terms["e"], cut, clamp)
        else:
            raw, alpha = alphas(prep, ids, rows, cols)
        before, active, _, _, n_act = O.front_to_back(alpha, stop)
        n_con = (active & (alpha > 0)).sum(axis=0)
        dn_c = np.asarray(dev_ncontrib[r0:r0 + h, c0:c0 + w]).reshape(-1)
        dn_a = np.asarray(dev_nactive[r0:r0 + h, c0:c0 + w]).reshape(-1)
        # alpha_cut = 0: the reference counts alpha ~ 1e-300 (below float32
        # range) as a contribution, so n_contrib is not a decision record;
        # no early stop: every entry is active
        flip = np.zeros(dn_c.shape, dtype=bool)
        if cut > 0:
            flip |= dn_c != n_con
        if stop is not None and stop > 0:
            flip |= dn_a != n_act
        STATS["pixels"] += dn_c.size
        STATS["n_contrib_flips"] += int((dn_c != n_con).sum()) if cut > 0 else 0
        STATS["n_active_flips"] += int((dn_a != n_act).sum()) if (stop is not None and stop > 0) else 0
        relevant = np.arange(len(ids))[:, None] <= np.maximum(n_act, dn_a)[None, :]
        near_clamp = ((np.abs(raw - clamp) < CLAMP_BAND) & relevant).any(axis=0)
        if flip.any():
            wide = np.zeros_like(raw, dtype=bool)
            if cut > 0:
                wide |= np.abs(raw - cut) < WIDE_CUT_REL * cut
            if stop is not None and stop > 0:
                wide |= np.abs(before - stop) < WIDE_STOP_REL * stop
            ok = (wide & relevant).any(axis=0)
            bad = flip & ~ok
            if bad.any():
                k = int(np.flatnonzero(bad)[0])
                unexplained.append((r0 + k // w, c0 + k % w))
        STATS["clamp_edges"] += int((near_clamp & ~flip).sum())
        mask[r0:r0 + h, c0:c0 + w] = (flip | near_clamp).reshape(h, w)
    assert not unexplained, (f"count mismatches away from any threshold at {unexplained[:5]} "
                             f"({len(unexplained)} tiles): a device decision error, not a flip")
    return mask


def knife_edge_mask(prep, scene, flags, tiles=None):
    """(H, W) bool: pixels whose oracle ray has a threshold knife-edge within
    its active prefix (plus the first inactive entry)."""
    cut = flags.get("alpha_cut", O.ALPHA_CUT)
    stop = flags.get("early_stop", O.EARLY_STOP_T)
    clamp = flags.get("alpha_clamp", O.ALPHA_CLAMP)
    O._attach(prep, scene)
    H, W = prep.height, prep.width
    mask = np.zeros((H, W), dtype=bool)
    for t in (range(prep.tiles_x * prep.tiles_y) if tiles is None else tiles):
        ids = prep.tile_ids(t)
        if ids.size == 0:
            continue
        r0, c0, h, w, rows, cols = O._tile_box(prep, t)
        terms = O.ray_terms(prep, ids, rows, cols)
        raw, alpha, _ = O.clamp_cut(terms["e"], cut, clamp)
        before, active, _, _, n_act = O.front_to_back(alpha, stop)
        k = np.arange(len(ids))[:, None]
        relevant = k <= n_act[None, :]
        near = near_threshold(raw, before, cut, clamp, stop)
        mask[r0:r0 + h, c0:c0 + w] = (near & relevant).any(axis=0).reshape(h, w)
    return mask
