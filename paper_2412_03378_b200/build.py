"""Build the sm_100a shared library `libvolgauss_b200.so` in-tree with nvcc.

Each translation unit is compiled to an object under build/ (in parallel),
then linked into paper_2412_03378_b200/libvolgauss_b200.so with the CUDA
runtime linked statically.  Used by __graft_entry__.build() and by
`python -m paper_2412_03378_b200.build`.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "csrc")
LIB = os.path.join(PKG, "libvolgauss_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
          "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
# translation units: (object, source, extra flags).  Preprocess rounds like
# numpy float64 (no FMA contraction); vg_blend.cu is split in two units so
# the forward kernel gets its own ptxas register-usage level (vg_blend.cu).
UNITS = [("vg_preprocess", "vg_preprocess.cu", ["-fmad=false"]), ("vg_radix", "vg_radix.cu", []),
         ("vg_span", "vg_span.cu", ["-Xptxas", "-regUsageLevel=6"]),  # place kernels -1.5 %
         ("vg_gamma", "vg_gamma.cu", []),
         ("vg_blend_fwd", "vg_blend.cu", ["-DVG_TU=1", "-Xptxas", "-regUsageLevel=6"]),
         ("vg_blend", "vg_blend.cu", ["-DVG_TU=2"]), ("vg_splat", "vg_splat.cu", []),
         ("vg_finalize", "vg_finalize.cu", []), ("vg_capi", "vg_capi.cu", []), ("vg_probe", "vg_probe.cu", []),
         ("vg_optim", "vg_optim.cu", []), ("vg_det", "vg_det.cu", []), ("vg_raymarch", "vg_raymarch.cu", []),
         ("vg_voxel", "vg_voxel.cu", []), ("vg_comm", "vg_comm.cu", [])]
SOURCES = sorted({src for _, src, _ in UNITS})


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _newer(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False, ptxas_verbose=False, debug=False, profile=False):
    """Compile and link the library.  debug=True builds the checking variant
    (-DVG_DEBUG: index asserts that trap, warp-schedule jitter, guarded and
    poisoned context buffers; tools/debug_checks.py) into
    build/debug/libvolgauss_b200_debug.so, loaded with VG_LIB=<path>;
    profile=True the variant with the per-CTA launch log (-DVG_CTA_LOG=1,
    vg_debug_cta_log; tools/walk_stats.py) into build/prof/."""
    build_dir, lib_path = BUILD, LIB
    variant = []
    if debug:
        build_dir = os.path.join(ROOT, "build", "debug")
        lib_path = os.path.join(build_dir, "libvolgauss_b200_debug.so")
        variant = ["-DVG_DEBUG"]
    elif profile:
        build_dir = os.path.join(ROOT, "build", "prof")
        lib_path = os.path.join(build_dir, "libvolgauss_b200_prof.so")
        variant = ["-DVG_CTA_LOG=1"]
    os.makedirs(build_dir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    headers.append(os.path.join(ROOT, "include", "volgauss_b200.h"))
    cc = nvcc()
    jobs = []
    for obj, src, extra in UNITS:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, obj + ".o")
        if force or _newer(o, [s] + headers):
            cmd = [cc] + ARCH + COMMON + extra + variant + ["-c", s, "-o", o]
            if ptxas_verbose:
                cmd += ["-Xptxas", "-v"]
            jobs.append((src, cmd))

    def run(job):
        src, cmd = job
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stdout}\n{r.stderr}")
        return src, r.stderr

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as pool:
        for src, err in pool.map(run, jobs):
            if verbose and err.strip():
                print(f"--- {src}\n{err}")
    objs = [os.path.join(build_dir, obj + ".o") for obj, _, _ in UNITS]
    if force or jobs or _newer(lib_path, objs):
        tmp = lib_path + ".tmp"
        cmd = [cc] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv, ptxas_verbose="-v" in sys.argv,
                debug="--debug" in sys.argv))
