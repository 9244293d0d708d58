"""Build the in-tree CUDA library ``libkinoptik_b200.so`` for sm_100a.

Plain nvcc, one object per translation unit (compiled in parallel), linked
into a shared library next to this file so it travels with the repo snapshot
to the GPU box.  No torch extension machinery: the boundary is the C ABI in
``include/kinoptik_b200.h``, loaded with ctypes.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libkinoptik_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC]

SOURCES = ["kop_kernels.cu", "kop_collision.cu", "kop_tree.cu", "kop_traj.cu", "kop_aux.cu", "kop_terms.cu",
           "kop_capi.cu"]
HEADERS = ["kop_check.cuh", "kop_chain.h", "kop_lie.cuh", "kop_lane.cuh", "kop_beam.cuh", "kop_collision.cuh", "kop_kernels.cuh", "kop_tree.cuh", "kop_traj.cuh", "kop_terms.cuh"]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


# checking builds (csrc/kop_check.cuh): same sources, extra defines, own objects,
# libraries under variants/ (shipped to the GPU box with the repo snapshot)
VARIANTS = {"poison": ["-DKOP_SMEM_POISON"], "jitter": ["-DKOP_JITTER"]}
VARIANT_DIR = os.path.join(ROOT, "variants")


def variant_lib(name: str) -> str:
    return os.path.join(VARIANT_DIR, f"libkinoptik_b200_{name}.so")


def build_variants(verbose: bool = False, force: bool = False) -> list:
    """Build every checking variant (tests/test_gpu_checks.py), concurrently (separate object dirs)."""
    with ThreadPoolExecutor(max_workers=len(VARIANTS)) as ex:
        return list(ex.map(lambda name: build(verbose=verbose, force=force, variant=name), VARIANTS))


def build_all(verbose: bool = False, force: bool = False) -> list:
    """The library and every checking variant, all translation units compiling at once."""
    with ThreadPoolExecutor(max_workers=1 + len(VARIANTS)) as ex:
        jobs = [ex.submit(build, verbose, False, force)] + \
               [ex.submit(build, verbose, False, force, name) for name in VARIANTS]
        return [j.result() for j in jobs]


def build(verbose: bool = False, ptxas_info: bool = False, force: bool = False, variant: str | None = None,
          defines: list | None = None) -> str:
    """The library (variant None) or a variant build: VARIANTS[variant] or the given -D defines
    (instrumented / A-B builds, e.g. -DKOP_TRAJ_PROFILE) into variants/."""
    extra = list(defines) if defines is not None else (VARIANTS[variant] if variant else [])
    obj_dir = os.path.join(ROOT, "build", f"obj_{variant}") if variant else OBJ
    lib_path = variant_lib(variant) if variant else LIB
    os.makedirs(obj_dir, exist_ok=True)
    os.makedirs(os.path.dirname(lib_path), exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "kinoptik_b200.h")]
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(obj_dir, src.replace(".cu", ".o"))
        if force or _stale(o, [s] + hdrs):
            cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", s, "-o", o]
            if ptxas_info:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append((src, cmd))

    def run(job):
        src, cmd = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, r

    with ThreadPoolExecutor(max_workers=max(1, len(jobs))) as ex:
        for src, r in ex.map(run, jobs):
            if verbose or r.returncode != 0 or ptxas_info:
                sys.stderr.write(r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed on {src}")
    objs = [os.path.join(obj_dir, s.replace(".cu", ".o")) for s in SOURCES]
    if force or jobs or _stale(lib_path, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib_path, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return lib_path


if __name__ == "__main__":
    print(build(verbose=True, ptxas_info="-v" in sys.argv, force="-f" in sys.argv))
    if "--variants" in sys.argv:
        print(build_variants(verbose=True, force="-f" in sys.argv))
