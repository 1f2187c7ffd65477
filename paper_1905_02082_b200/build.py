"""Builds the CUDA extension in-tree: nvcc for sm_100a only, one object per
.cu (compiled in parallel), linked into paper_1905_02082_b200/librefusion_b200.so.

-fmad=false keeps every double expression rounded as written, which is what
makes allocation, integration, carving and sampling bit-identical to the CPU
oracle ("Arithmetic contract")."""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "librefusion_b200.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fno-fast-math", "-Xptxas", "-warn-spills"]
SOURCES = ["rf_capi.cu", "rf_track.cu", "rf_volume.cu", "rf_raycast.cu", "rf_synth.cu", "rf_mesh.cu", "rf_eval.cu"]


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, defines=(), variant: str | None = None) -> str:
    """Default build -> librefusion_b200.so. A `variant` (tuning experiments,
    selected at run time with RF_LIB_PATH) builds with extra -D defines into
    _variants/lib<variant>.so."""
    build_dir = BUILD if not variant else os.path.join(HERE, "_variants", "obj_" + variant)
    lib = LIB if not variant else os.path.join(HERE, "_variants", f"lib{variant}.so")
    os.makedirs(build_dir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h", ".inc"))]
    headers.append(os.path.join(os.path.dirname(HERE), "include", "refusion_b200.h"))
    jobs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(build_dir, src.replace(".cu", ".o"))
        if _stale(o, [s] + headers) or variant:
            jobs.append([NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0 or verbose:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
        return r.stderr

    with cf.ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(build_dir, s.replace(".cu", ".o")) for s in SOURCES]
    if jobs or not os.path.exists(lib):
        run([NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lcudart"])
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    variant = args[args.index("--variant") + 1] if "--variant" in args else None
    defines = [a[2:] for a in args if a.startswith("-D")]
    print(build(verbose="-v" in args, defines=defines, variant=variant))
