"""Scene / camera text and PFM I/O (paper_2412_03378_b200/sceneio.py) against
files the reference's own sceneio wrote (tests/golden/make_golden_io.py,
make_golden.py's golden_render.pfm): byte-identical output, exact round
trips, reference error behaviour.  CPU only."""

from __future__ import annotations

import os

import numpy as np
import pytest

from paper_2412_03378_b200 import sceneio

G = os.path.join(os.path.dirname(__file__), "golden")


def test_scene_text_round_trips_byte_for_byte(tmp_path):
    scene, cams = sceneio.load_scene(os.path.join(G, "io_scene.txt"))
    assert len(scene) == 7 and set(cams) == {"front", "side"}
    assert cams["front"].z_near == 0.02 and cams["side"].width == 33
    out = tmp_path / "s.txt"
    sceneio.save_scene(out, scene, cams)
    assert out.read_bytes() == open(os.path.join(G, "io_scene.txt"), "rb").read()


def test_camera_text_round_trips_byte_for_byte(tmp_path):
    cam = sceneio.load_camera(os.path.join(G, "io_camera.txt"))
    out = tmp_path / "c.txt"
    sceneio.save_camera(out, cam)
    assert out.read_bytes() == open(os.path.join(G, "io_camera.txt"), "rb").read()


def test_pfm_matches_reference_bytes(tmp_path):
    img = sceneio.read_pfm(os.path.join(G, "golden_render.pfm"))
    ref = np.load(os.path.join(G, "golden_scene.npz"))["color"]
    np.testing.assert_array_equal(img, ref.astype(np.float32).astype(np.float64))
    out = tmp_path / "g.pfm"
    sceneio.write_pfm(out, ref)
    assert out.read_bytes() == open(os.path.join(G, "golden_render.pfm"), "rb").read()
    grey = np.arange(12, dtype=float).reshape(3, 4)
    sceneio.write_pfm(tmp_path / "g1.pfm", grey)
    np.testing.assert_array_equal(sceneio.read_pfm(tmp_path / "g1.pfm"), grey)


def test_format_errors_name_line_and_field(tmp_path):
    bad = tmp_path / "bad.txt"
    bad.write_text("volgauss scene v1\nprimitive\nmean 1 2\n")
    with pytest.raises(sceneio.FormatError, match="line 3: field 'mean' needs 3 values"):
        sceneio.load_scene(bad)
    bad.write_text("volgauss scene v1\ntheta 0.5\n")
    with pytest.raises(sceneio.FormatError, match="before any 'primitive'"):
        sceneio.load_scene(bad)
    bad.write_text("not a scene\n")
    with pytest.raises(sceneio.FormatError, match="line 1"):
        sceneio.load_scene(bad)
    bad.write_text("volgauss scene v1\ncamera c\nwidth 2.5\nend\n")
    with pytest.raises(sceneio.FormatError, match="must be integer"):
        sceneio.load_scene(bad)
    with pytest.raises(ValueError):
        sceneio.write_pfm(tmp_path / "x.pfm", np.zeros((2, 2, 2)))


def test_density_grid_files_match_reference(tmp_path):
    """save_density_grid writes the reference's bytes (tests/golden/io_grid.*,
    written by tomo.save_density_grid); load_density_grid reads them back."""
    from paper_2412_03378_b200 import sceneio
    from paper_2412_03378_b200.tomo import DensityGrid
    gold = os.path.join(G, "io_grid")
    values = np.load(os.path.join(G, "io_grid_values.npy"))
    g = sceneio.load_density_grid(gold)
    assert g.values.shape == (5, 6, 7)
    assert np.array_equal(g.values, values.astype(np.float32).astype(np.float64))
    base = str(tmp_path / "grid")
    sceneio.save_density_grid(base, DensityGrid(values, g.bbox_min, g.bbox_max))
    for ext in (".raw", ".txt"):
        assert open(base + ext, "rb").read() == open(gold + ext, "rb").read(), ext
    with open(base + ".txt", "w") as f:
        f.write("something else\n")
    with pytest.raises(ValueError):
        sceneio.load_density_grid(base)
