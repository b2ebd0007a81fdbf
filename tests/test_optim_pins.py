"""Pin the training-step oracle (oracle/optim_oracle.py) against the golden
vectors the reference's own optim.Trainer.step / GradAccum /
densify_and_prune produced (tests/golden/make_golden_optim.py).  CPU only."""

from __future__ import annotations

import os
from types import SimpleNamespace

import numpy as np

from oracle import optim_oracle as OO

HERE = os.path.dirname(os.path.abspath(__file__))


def golden():
    return dict(np.load(os.path.join(HERE, "golden", "optim.npz")))


def start(d):
    scene = SimpleNamespace(means=d["means"].copy(), scales=d["scales"].copy(),
                            rotations=d["rotations"].copy(), thetas=d["thetas"].copy(),
                            colors=d["colors"].copy())
    cfg = OO.TrainConfig(iterations=int(d["iterations"]), max_primitives=int(d["max_primitives"]))
    extent = float(d["extent"])
    return scene, cfg, extent, OO.Trainer(scene, cfg, extent), OO.GradAccum(len(scene.means))


def grads_of(d, it):
    return SimpleNamespace(**{k: d[f"g{it}_{k}"] for k in
                              ("d_means", "d_scales", "d_rotations", "d_thetas", "d_colors", "visible")})


def test_trainer_steps_match_reference_bitwise():
    d = golden()
    scene, cfg, extent, tr, acc = start(d)
    for it in range(3):
        g = grads_of(d, it)
        acc.update(g)
        tr.step(g, it)
        for k in ("means", "scales", "rotations", "thetas", "colors"):
            assert np.array_equal(getattr(scene, k), d[f"s{it}_{k}"]), (it, k)
        assert np.array_equal(tr.color_raw, d[f"s{it}_color_raw"])
        for name, opt in tr.opts.items():
            assert np.array_equal(opt.m, d[f"s{it}_{name}_m"]), (it, name)
            assert np.array_equal(opt.v, d[f"s{it}_{name}_v"]), (it, name)
    assert np.array_equal(acc.norm_sum, d["accum_norm"])
    assert np.array_equal(acc.count, d["accum_count"])


def test_densify_and_prune_matches_reference():
    d = golden()
    scene, cfg, extent, tr, acc = start(d)
    for it in range(3):
        g = grads_of(d, it)
        acc.update(g)
        tr.step(g, it)
    rng = np.random.Generator(np.random.Philox(key=11))
    split, clone, prune = OO.densify_and_prune(scene, tr, acc, cfg, extent, rng)
    kinds, parents = d["d_event_kinds"], d["d_event_parents"]
    assert np.array_equal(np.flatnonzero(split), parents[kinds == 0])
    assert np.array_equal(np.flatnonzero(clone), parents[kinds == 1])
    assert np.array_equal(np.flatnonzero(prune), parents[kinds == 2])
    for k in ("means", "scales", "rotations", "thetas", "colors"):
        np.testing.assert_allclose(getattr(scene, k), d[f"d_{k}"], rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(tr.color_raw, d["d_color_raw"], rtol=1e-14, atol=1e-15)
    for name, opt in tr.opts.items():
        assert np.array_equal(opt.m, d[f"d_{name}_m"]) and np.array_equal(opt.v, d[f"d_{name}_v"])


def test_divergence_raises():
    d = golden()
    scene, cfg, extent, tr, acc = start(d)
    g = grads_of(d, 0)
    g.d_thetas = g.d_thetas.copy()
    g.d_thetas[5] = np.nan
    try:
        tr.step(g, 0)
    except FloatingPointError as e:
        assert "density" in str(e) and "primitive 5" in str(e)
    else:
        raise AssertionError("non-finite update must raise")
