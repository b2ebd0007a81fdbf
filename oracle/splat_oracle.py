"""CPU float64 oracle for mode="splat", the EWA 3DGS comparator of the
reference: screen-space Gaussian alpha
opacity * exp(-maha / 2) with the dilated EWA covariance, the same
compositing as the analytic path, and the backward through the EWA
projection.

TEST INFRASTRUCTURE ONLY (see volgauss_oracle.py's header): a numpy
restatement of `raster.py:154-209, 332-372` (splat branches) and
`grad.py:107-213, 262-302` (paths relative to the reference's
`pkg/src/volgauss/`), pinned against golden vectors the reference itself
produced (tests/golden/make_golden_splat.py, tests/test_oracle_pins.py).
The product package never imports it.
"""

from __future__ import annotations

import numpy as np

from .volgauss_oracle import (ALPHA_CLAMP, ALPHA_CUT, BASE_RADIUS_SIGMA, EARLY_STOP_T, SCALE_FLOOR,
                              TILE, Grads, Image, Prepared, _rotmat_quat_jac, _tile_box, floored,
                              front_to_back, quat_to_rotmat, sandwich, tile_pairs)


def prepare(scene, cam, key_dtype=np.float64, tile=TILE):
    """raster.prepare(mode='splat'): EWA projection (raster.py:175-209), the
    3-sigma bin radius of the dilated covariance (raster.py:154-172, splat
    branch) and the conic (raster.py:212-219)."""
    means = np.asarray(scene.means, dtype=np.float64).reshape(-1, 3)
    n = len(means)
    scales = np.asarray(scene.scales, dtype=np.float64).reshape(n, 3)
    rot = quat_to_rotmat(np.asarray(scene.rotations, dtype=np.float64).reshape(n, 4)) if n else np.zeros((0, 3, 3))
    s = floored(scales)
    Rc = np.asarray(cam.rotation, dtype=np.float64)
    tc = np.asarray(cam.translation, dtype=np.float64)
    v = means @ Rc.T + tc
    valid = v[:, 2] > cam.z_near
    z = np.where(valid, v[:, 2], 1.0)
    lim_x = 1.3 * (0.5 * cam.width / cam.fx)
    lim_y = 1.3 * (0.5 * cam.height / cam.fy)
    x, y = v[:, 0], v[:, 1]
    cx_ratio = np.clip(x / z, -lim_x, lim_x)
    cy_ratio = np.clip(y / z, -lim_y, lim_y)
    J = np.zeros((n, 2, 3))
    J[:, 0, 0] = cam.fx / z
    J[:, 1, 1] = cam.fy / z
    J[:, 0, 2] = -cam.fx * cx_ratio / z
    J[:, 1, 2] = -cam.fy * cy_ratio / z
    U = J @ Rc
    sigma = sandwich(rot, s * s) if n else np.zeros((0, 3, 3))
    cov2d = np.einsum("nij,njk,nlk->nil", U, sigma, U)
    cov2d[:, 0, 0] += 0.3
    cov2d[:, 1, 1] += 0.3
    mean2d = np.stack([cam.fx * x / z + cam.cx, cam.fy * y / z + cam.cy], axis=1)
    m = 0.5 * (cov2d[:, 0, 0] + cov2d[:, 1, 1])
    det = cov2d[:, 0, 0] * cov2d[:, 1, 1] - cov2d[:, 0, 1] * cov2d[:, 1, 0]
    radius = BASE_RADIUS_SIGMA * np.sqrt(m + np.sqrt(np.maximum(m * m - det, 0.0)))
    lam = np.empty_like(cov2d)
    lam[:, 0, 0] = cov2d[:, 1, 1]
    lam[:, 1, 1] = cov2d[:, 0, 0]
    lam[:, 0, 1] = -cov2d[:, 0, 1]
    lam[:, 1, 0] = -cov2d[:, 1, 0]
    lam /= det[:, None, None]
    depth = v[:, 2].copy()
    tx_n, ty_n, (pt, pp, start) = tile_pairs(valid, mean2d, radius, cam.width, cam.height,
                                             depth.astype(key_dtype), tile)
    prep = Prepared(cam.width, cam.height, tx_n, ty_n, valid, depth, mean2d, radius, np.zeros(n),
                    None, rot, None, pt, pp, start, False, 0.0, cam)
    prep.splat = dict(v=v, z=z, U=U, sigma=sigma, lam=lam, cx_ratio=cx_ratio, cy_ratio=cy_ratio,
                      clamped_x=np.abs(x / z) > lim_x, clamped_y=np.abs(y / z) > lim_y)
    return prep


def _alphas(prep, scene, ids, rows, cols, alpha_cut, alpha_clamp):
    """raster._tile_alphas, splat branch (raster.py:353-372)."""
    px = np.stack([cols + 0.5, rows + 0.5], axis=1)
    dlt = px[None, :, :] - prep.mean2d[ids][:, None, :]
    lam = prep.splat["lam"][ids]
    maha = np.einsum("kpi,kij,kpj->kp", dlt, lam, dlt)
    falloff = np.exp(-0.5 * maha)
    opac = np.asarray(scene.splat_opacities, dtype=np.float64).reshape(-1)[ids]
    raw = opac[:, None] * falloff
    alpha = np.minimum(raw, alpha_clamp)
    if alpha_cut > 0.0:
        cut = alpha < alpha_cut
        alpha = np.where(cut, 0.0, alpha)
    else:
        cut = np.zeros(alpha.shape, dtype=bool)
    return raw, alpha, cut, dlt, falloff, lam, opac


def render(scene, cam, *, early_stop=EARLY_STOP_T, alpha_cut=ALPHA_CUT, alpha_clamp=ALPHA_CLAMP,
           prep=None):
    """raster.render(mode='splat')."""
    if prep is None:
        prep = prepare(scene, cam)
    H, W = cam.height, cam.width
    colors = np.asarray(scene.colors, dtype=np.float64).reshape(-1, 3)
    bg = np.asarray(scene.background, dtype=np.float64)
    out_c, out_t = np.empty((H, W, 3)), np.empty((H, W))
    out_n, out_a = np.zeros((H, W), np.int32), np.zeros((H, W), np.int32)
    for t in range(prep.tiles_x * prep.tiles_y):
        r0, c0, h, w, rows, cols = _tile_box(prep, t)
        ids = prep.tile_ids(t)
        if ids.size == 0:
            out_c[r0:r0 + h, c0:c0 + w] = bg
            out_t[r0:r0 + h, c0:c0 + w] = 1.0
            continue
        _, alpha, _, _, _, _, _ = _alphas(prep, scene, ids, rows, cols, alpha_cut, alpha_clamp)
        _, active, weight, t_final, n_act = front_to_back(alpha, early_stop)
        col = np.einsum("kp,kc->pc", weight, colors[ids]) + t_final[:, None] * bg
        out_c[r0:r0 + h, c0:c0 + w] = col.reshape(h, w, 3)
        out_t[r0:r0 + h, c0:c0 + w] = t_final.reshape(h, w)
        out_n[r0:r0 + h, c0:c0 + w] = (active & (alpha > 0)).sum(axis=0).reshape(h, w)
        out_a[r0:r0 + h, c0:c0 + w] = n_act.reshape(h, w)
    return Image(out_c, out_t, out_n, out_a)


def backward(scene, cam, d_color, *, d_transmittance=None, early_stop=EARLY_STOP_T,
             alpha_cut=ALPHA_CUT, alpha_clamp=ALPHA_CLAMP, prep=None):
    """grad.backward(mode='splat') (grad.py:107-213) and
    _splat_projection_backward (grad.py:262-302).  Returns Grads with an
    extra d_splat_opacities field (d_thetas / d_kappas stay zero)."""
    n = len(np.asarray(scene.means).reshape(-1, 3))
    grads = Grads.zeros(n)
    grads.d_splat_opacities = np.zeros(n)
    d_color = np.asarray(d_color, dtype=np.float64)
    if n == 0:
        grads.d_background = d_color.reshape(-1, 3).sum(axis=0)
        return grads
    if prep is None:
        prep = prepare(scene, cam)
    colors = np.asarray(scene.colors, dtype=np.float64).reshape(-1, 3)
    bg = np.asarray(scene.background, dtype=np.float64)
    g_lam = np.zeros((n, 2, 2))
    d_mean2d = np.zeros((n, 2))
    for t in range(prep.tiles_x * prep.tiles_y):            # fixed tile order
        r0, c0, h, w, rows, cols = _tile_box(prep, t)
        dc = d_color[r0:r0 + h, c0:c0 + w].reshape(-1, 3)
        ids = prep.tile_ids(t)
        if ids.size == 0:
            grads.d_background += dc.sum(axis=0)
            continue
        raw, alpha, cut, dlt, falloff, lam, opac = _alphas(prep, scene, ids, rows, cols, alpha_cut,
                                                           alpha_clamp)
        before, active, weight, t_final, _ = front_to_back(alpha, early_stop)
        dot = np.einsum("pc,kc->kp", dc, colors[ids])
        dt = dc @ bg
        if d_transmittance is not None:
            dt = dt + d_transmittance[r0:r0 + h, c0:c0 + w].reshape(-1)
        acc = np.cumsum(dot * weight, axis=0)
        behind = (acc[-1] - acc) + (dt * t_final)[None, :]
        d_alpha = np.where(active, dot * before - behind / (1.0 - alpha), 0.0)
        live = ~cut & (raw < alpha_clamp)
        d_raw = np.where(live, d_alpha, 0.0)
        grads.d_colors[ids] += np.einsum("kp,pc->kc", weight, dc)
        grads.d_background += dc.T @ t_final
        grads.visible[ids] |= (active & (alpha > 0)).any(axis=1)
        grads.d_splat_opacities[ids] += np.einsum("kp,kp->k", d_raw, falloff)
        d_maha = -0.5 * falloff * (d_raw * opac[:, None])
        g_lam[ids] += np.einsum("kp,kpi,kpj->kij", d_maha, dlt, dlt)
        d_mean2d[ids] += -2.0 * np.einsum("kp,kpi->ki", d_maha, np.einsum("kij,kpj->kpi", lam, dlt))
    return projection_backward(scene, prep, g_lam, d_mean2d, grads)


def projection_backward(scene, prep, g_lam, d_mean2d, grads):
    """_splat_projection_backward (grad.py:262-302)."""
    cam = prep.camera
    c = prep.splat
    scales = np.asarray(scene.scales, dtype=np.float64).reshape(-1, 3)
    quats = np.asarray(scene.rotations, dtype=np.float64).reshape(-1, 4)
    s = floored(scales)
    live_scale = scales >= SCALE_FLOOR
    lam, U, sigma, z = c["lam"], c["U"], c["sigma"], c["z"]
    x, y = c["v"][:, 0], c["v"][:, 1]
    Rc = np.asarray(cam.rotation, dtype=np.float64)
    g_cov = -np.einsum("nij,njk,nkl->nil", lam, g_lam, lam)
    d_sigma = np.einsum("nji,njk,nkl->nil", U, g_cov, U)
    g_cov_sym = g_cov + np.transpose(g_cov, (0, 2, 1))
    d_u = np.einsum("nij,njk,nkl->nil", g_cov_sym, U, sigma)
    d_j = np.einsum("nij,kj->nik", d_u, Rc)
    fx, fy = cam.fx, cam.fy
    rx, ry = c["cx_ratio"], c["cy_ratio"]
    ox, oy = ~c["clamped_x"], ~c["clamped_y"]
    dj00, dj02, dj11, dj12 = d_j[:, 0, 0], d_j[:, 0, 2], d_j[:, 1, 1], d_j[:, 1, 2]
    du, dv_ = d_mean2d[:, 0], d_mean2d[:, 1]
    dv = np.zeros((len(s), 3))
    dv[:, 0] = dj02 * (-fx / z ** 2) * ox + du * fx / z
    dv[:, 1] = dj12 * (-fy / z ** 2) * oy + dv_ * fy / z
    dv[:, 2] = (dj00 * (-fx / z ** 2) + dj11 * (-fy / z ** 2)
                + dj02 * (fx * rx / z ** 2 + (fx * x / z ** 3) * ox)
                + dj12 * (fy * ry / z ** 2 + (fy * y / z ** 3) * oy)
                + du * (-fx * x / z ** 2) + dv_ * (-fy * y / z ** 2))
    valid = prep.valid
    dv[~valid] = 0.0
    grads.d_means += dv @ Rc
    d_sigma[~valid] = 0.0
    rot = prep.rot
    a = np.einsum("nji,njk,nkl->nil", rot, d_sigma, rot)
    grads.d_scales += np.einsum("nii->ni", a) * (2.0 * s) * live_scale
    d_rot = np.einsum("nij,njk->nik", d_sigma + np.transpose(d_sigma, (0, 2, 1)), rot * (s * s)[:, None, :])
    nq = np.linalg.norm(quats, axis=1, keepdims=True)
    qh = quats / nq
    dqh = np.einsum("nij,nqij->nq", d_rot, _rotmat_quat_jac(qh))
    grads.d_rotations += (dqh - qh * np.einsum("nq,nq->n", qh, dqh)[:, None]) / nq
    return grads
