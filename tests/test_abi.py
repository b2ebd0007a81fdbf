"""CPU-side checks of the C ABI: the in-tree shared library loads, exports
every symbol include/volgauss_b200.h declares, and fails cleanly (VG_ECUDA,
no crash) when no GPU is present.  No compute calls."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT, cuda_available

HEADER = os.path.join(ROOT, "include", "volgauss_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|int64_t|size_t|const char\*)\s+(vg_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ["vg_prepare", "vg_render_forward", "vg_render_backward", "vg_tomo_forward",
                 "vg_tomo_backward", "vg_tile_lists", "vg_create", "vg_destroy", "vg_last_error",
                 "vg_allreduce_grads"]:
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_2412_03378_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libvolgauss_b200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_lib.EXPORTS)
    assert _lib.load().vg_abi_version() == _lib.ABI_VERSION


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU error path")
def test_create_without_gpu_reports_error():
    from paper_2412_03378_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    lib = _lib.load()
    h = ctypes.c_void_p()
    rc = lib.vg_create(ctypes.byref(h), 0)
    assert rc == _lib.VG_ECUDA
    assert b"device" in lib.vg_last_error()


def test_sass_targets_sm100a():
    """The library carries sm_100a SASS (and the blend kernels use MUFU)."""
    import shutil
    import subprocess
    from paper_2412_03378_b200 import _lib
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(_lib.LIB_PATH) or not os.path.exists(tool):
        pytest.skip("library or cuobjdump unavailable")
    out = subprocess.run([tool, "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
